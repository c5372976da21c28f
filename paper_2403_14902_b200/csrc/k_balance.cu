// K6: data-aware tile scheduling for classifier hops whose cost follows the input size
// (Laminar's data-aware load balancing).
//
// The paper's Laminar router sends each piece of work to the worker with the lowest monitored
// load, where the load is estimated proactively from a heuristic -- "input size as a reasonable
// proxy for execution cost ... for vision models, it is the input image/frame size" (PAPER.md:
// 876-878) -- instead of round-robin.  On the GPU the workers of a classifier
// hop are the persistent K4 CTAs.  For an AREA crop the work per tuple is proportional to its bbox
// area w*h (every source pixel of the box is read and summed), so:
//   K6a  the estimated cost of every 32-position chunk of the hop's input = sum of w*h (one warp
//        per chunk, grid-stride);
//   K6b  one CTA scans the chunk costs and cuts the input into bal_ctas contiguous position ranges
//        of equal estimated cost: CTA c starts at the first chunk k whose exclusive prefix
//        cost X_k satisfies X_k * G >= c * A (A = total, G = CTAs).  Each CTA's load is at most
//        A / G plus one chunk; ranges start on 32-position boundaries, so every verdict word of
//        the hop has exactly one writer.
// K4 then walks its range in 128-tuple tiles (the last one ragged).  Both kernels resolve the hop
// on the device like K4 and exit unless it is an AREA linear head.  The schedule never changes
// which tuples pass, only which SM evaluates them.
#include <algorithm>

#include "hydro_internal.cuh"

using namespace hydro;

namespace {

struct HopIn {
  const uint32_t* list_in;
  uint32_t base, count;
  bool area;
};

__device__ __forceinline__ HopIn resolve_hop(const ClsParams& p) {
  HopIn r{nullptr, p.range_base, 0u, false};
  const DevState* st = p.st;
  int pred;
  if (p.dispatch) {
    const int h = st->sched[p.hop];
    if (h < 0 || h >= st->n_pred) return r;
    pred = st->order[h];
    if (h == 0) {
      r.list_in = p.sel0;
      r.count = p.sel0 ? *p.sel0_count : p.range_n;
    } else {
      r.list_in = p.lists + static_cast<uint64_t>(h) * p.list_stride;
      r.count = p.counts[h];
    }
  } else {
    pred = p.explicit_pred;
    r.list_in = p.list_in;
    r.count = p.list_in ? *p.count_in : p.range_n;
  }
  r.area = st->kind[pred] == kLinear && p.preds[pred].crop_mode == HYDRO_CROP_AREA;
  return r;
}

__global__ void hydro_balance_cost_kernel(ClsParams p) {
  const HopIn hi = resolve_hop(p);
  // (a hop with >= kBalRangeTilesPerCta tiles per CTA runs round-robin tiles: no ranges needed)
  if (!hi.area || hi.count >= kBalRangeTilesPerCta * kTileM * static_cast<uint32_t>(p.bal_ctas)) return;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t n_chunks = (hi.count + 31u) / 32u;
  const uint32_t warps = gridDim.x * (blockDim.x / 32u);
  for (uint32_t k = blockIdx.x * (blockDim.x / 32u) + threadIdx.x / 32u; k < n_chunks; k += warps) {
    const uint32_t pos = 32u * k + lane;
    uint32_t area = 0;
    if (pos < hi.count) {
      const uint32_t idx = hi.list_in ? __ldg(hi.list_in + pos) : hi.base + pos;
      const uint64_t bb = __ldg(p.bbox + idx);
      const int x0 = static_cast<int>(bb & 0xFFFF), y0 = static_cast<int>((bb >> 16) & 0xFFFF);
      const int x1 = static_cast<int>((bb >> 32) & 0xFFFF), y1 = static_cast<int>((bb >> 48) & 0xFFFF);
      area = static_cast<uint32_t>(max(x1 - x0, 1)) * static_cast<uint32_t>(max(y1 - y0, 1));  // input size w*h
    }
    const uint32_t sum = __reduce_add_sync(0xFFFFFFFFu, area);
    if (lane == 0) p.bal_chunks[k] = sum;
  }
}

constexpr int kBalThreads = 1024;

__global__ void __launch_bounds__(kBalThreads) hydro_balance_bounds_kernel(ClsParams p) {
  const HopIn hi = resolve_hop(p);
  // (a hop with >= kBalRangeTilesPerCta tiles per CTA runs round-robin tiles: no ranges needed)
  if (!hi.area || hi.count >= kBalRangeTilesPerCta * kTileM * static_cast<uint32_t>(p.bal_ctas)) return;
  __shared__ unsigned long long warp_tot[kBalThreads / 32];
  const uint32_t G = static_cast<uint32_t>(p.bal_ctas);
  const uint32_t n_chunks = (hi.count + 31u) / 32u;
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  // thread t owns chunks [k0, k1)
  const uint32_t k0 = static_cast<uint32_t>((static_cast<uint64_t>(n_chunks) * t) / kBalThreads);
  const uint32_t k1 = static_cast<uint32_t>((static_cast<uint64_t>(n_chunks) * (t + 1)) / kBalThreads);
  unsigned long long mine = 0;
  for (uint32_t k = k0; k < k1; ++k) mine += p.bal_chunks[k];
  // block exclusive scan of the per-thread sums (64-bit)
  unsigned long long incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= static_cast<uint32_t>(d)) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = warp_tot[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, w, d);
      if (lane >= static_cast<uint32_t>(d)) w += v;
    }
    warp_tot[lane] = w;  // inclusive prefix over warps
  }
  __syncthreads();
  const unsigned long long total = warp_tot[kBalThreads / 32 - 1];
  unsigned long long x = incl - mine + (warp > 0 ? warp_tot[warp - 1] : 0ull);  // exclusive prefix of chunk k0
  if (t == 0) {
    p.bal_bounds[0] = 0;
    p.bal_bounds[G] = hi.count;
  }
  if (total == 0) {  // empty input: every range is empty
    for (uint32_t c = 1 + t; c < G; c += kBalThreads) p.bal_bounds[c] = 0;
    return;
  }
  // chunk k (exclusive prefix x, inclusive x') is the first chunk of CTA c for every c with
  // x_prev * G < c * A <= x * G; written here as: chunk k+1 starts CTA c for x * G < c * A <= x' * G
  for (uint32_t k = k0; k < k1; ++k) {
    const unsigned long long xn = x + p.bal_chunks[k];
    unsigned long long c_lo = (x * G) / total + 1, c_hi = (xn * G) / total;
    if (c_hi > G - 1) c_hi = G - 1;
    for (unsigned long long c = c_lo; c <= c_hi; ++c)
      p.bal_bounds[c] = min(32u * (k + 1u), hi.count);
    x = xn;
  }
}

}  // namespace

void hydro_balance_launch(const ClsParams& c, uint64_t max_positions, int num_sms, cudaStream_t stream) {
  const uint64_t chunks = (max_positions + 31) / 32;
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((chunks + 7) / 8, 4ull * num_sms)));
  hydro_balance_cost_kernel<<<grid, 256, 0, stream>>>(c);
  hydro_balance_bounds_kernel<<<1, kBalThreads, 0, stream>>>(c);
}
