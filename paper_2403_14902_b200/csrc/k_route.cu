// K1: route kernel (evaluate a run of cheap predicates), K2: compaction / emit, K5: statistics
// fold + rank + order, weight re-layout.
//
// K1 evaluates a maximal run of cheap predicates (LABEL_EQ, HASH) in the device-resident order
// on the still-alive positions of a routing batch and writes a verdict bitmap plus the survivors
// per 2048-position segment, accumulating the per-predicate in / pass / cycle counters the eddy
// folds.  K2 then drops the failing tuples at once (eager
// materialization): an order-preserving compaction of the hop's input
// positions into the next alive list, or the emitted (id, bbox) rows (the query's projection,
// PAPER.md:44, 277).  K2 runs after every evaluator (K1 or the classifier K4).
//
// K5 folds the counters: S <- gamma*S + delta (R4), s = S_pass/S_in,
// c = S_cost/S_in, key = c/(1-s), stable order by (key, id)
// (R1, R2).
#include <cuda_fp16.h>

#include <type_traits>

#include "hydro_internal.cuh"

using namespace hydro;

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;

__device__ __forceinline__ bool hash_pass(const PredDev& pd, uint64_t id, uint64_t bb) {
  int units = pd.units;
  if (pd.units_per_area > 0) {
    int w = static_cast<int>((bb >> 32) & 0xFFFF) - static_cast<int>(bb & 0xFFFF);
    int h = static_cast<int>((bb >> 48) & 0xFFFF) - static_cast<int>((bb >> 16) & 0xFFFF);
    int area = max(w, 1) * max(h, 1);
    units = max((area + pd.units_per_area - 1) / pd.units_per_area, 1);
  }
  uint32_t h = static_cast<uint32_t>(splitmix64(id ^ pd.seed) >> 32);
  for (int r = 0; r < units; ++r) h = fmix32(h + static_cast<uint32_t>(r));
  uint64_t T = (id >= pd.drift_id) ? pd.thr1 : pd.thr0;
  return static_cast<uint64_t>(h) < T;
}

// Compacted HASH evaluation: thread tid hashes compact entries tid + 256 q, q < M (M independent
// chains); the fail bits come back as one ballot word per 32 entries in s_vw.
template <int M>
__device__ __forceinline__ void hash_compacted(const PredDev& pd, const uint64_t* buf, uint32_t n, int tid, int lane,
                                               int warp, uint32_t* s_vw) {
  const bool one_thr = pd.thr0 == pd.thr1;
  const int units = pd.units;
  uint32_t hq[M];
  uint64_t iq[M];
#pragma unroll
  for (int q = 0; q < M; ++q) {
    const uint32_t e = q * kRouteThreads + tid;
    iq[q] = e < n ? buf[e] : 0ull;
    hq[q] = static_cast<uint32_t>(splitmix64(iq[q] ^ pd.seed) >> 32);
  }
  for (int u = 0; u < units; ++u) {
#pragma unroll
    for (int q = 0; q < M; ++q) hq[q] = fmix32(hq[q] + static_cast<uint32_t>(u));
  }
#pragma unroll
  for (int q = 0; q < M; ++q) {
    const uint32_t e = q * kRouteThreads + tid;
    const uint64_t T = (one_thr || iq[q] < pd.drift_id) ? pd.thr0 : pd.thr1;
    const uint32_t bw = __ballot_sync(kFull, e < n && static_cast<uint64_t>(hq[q]) >= T);
    if (lane == 0 && q * kRouteThreads < n) s_vw[q * (kRouteThreads / 32) + warp] = bw;
  }
}

// Which hop-h evaluator ran (device order): returns the first predicate's kind, and the cheap run
// length in *run (0 when hop h is LINEAR or K1 has nothing to do).
__device__ __forceinline__ bool k1_runs(const DevState* st, int h, int* run) {
  const int P = st->n_pred;
  *run = 0;
  if (P == 0) return h == 0;
  if (h >= P || is_classifier(st->kind[st->order[h]])) return false;
  if (h > 0 && !is_classifier(st->kind[st->order[h - 1]])) return false;  // inside a run started earlier
  int r = 0;
  while (h + r < P && !is_classifier(st->kind[st->order[h + r]])) ++r;
  *run = r;
  return true;
}

}  // namespace

// ------------------------------------------------------------------------------------------
// K1: evaluate.  Persistent grid, tile t = positions [2048 t, 2048 t + 2048); thread = 8 positions.
// kCompact: the context has an expensive HASH predicate (units >= kCompactUnits), so the kernel
// carries the CTA-wide compaction path (more registers and 16 KB of shared memory)
constexpr int kLeanMaxRun = 4;  // K1 lean path: predicates per run

template <bool kCompact>
#ifndef HYDRO_K1_MINB
#define HYDRO_K1_MINB 3
#endif
__global__ void __launch_bounds__(kRouteThreads, kCompact ? 2 : HYDRO_K1_MINB) hydro_route_kernel(RouteParams p) {
  __shared__ PredDev s_pred[kMaxPred];
  __shared__ int32_t s_run_id[kMaxPred];
  // per-warp statistic slots (lane 0 of each warp owns its row: plain adds, no shared atomics)
  __shared__ uint32_t s_in[kRouteThreads / 32][kMaxPred], s_pass[kRouteThreads / 32][kMaxPred];
  __shared__ uint32_t s_comp[kRouteThreads / 32][kMaxPred];
  __shared__ unsigned long long s_cost[kRouteThreads / 32][kMaxPred];
  __shared__ uint32_t s_warp_cnt[2][kRouteThreads / 32];  // double-buffered: one barrier per tile
  __shared__ uint64_t s_cids[kCompact ? kRouteThreads / 32 : 1][kWarpSeg];  // compacted alive ids
  __shared__ uint32_t s_vw[kRouteTile / 32];                 // their fail bits, one word per 32 entries
  __shared__ uint32_t s_cw[kRouteThreads / 32];              // warp alive counts
  __shared__ int32_t s_work, s_nrun, s_n_and, s_need_id, s_need_bbox, s_need_label, s_lean;
  __shared__ const uint32_t* s_list_in;
  __shared__ const uint32_t* s_and[kMaxPred];
  __shared__ uint32_t* s_bits_out;
  __shared__ uint32_t s_count, s_range_base;
  __shared__ int32_t s_hop;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  DevState* st = p.st;

  if (tid == 0) {
    int32_t work = 1, nrun = 0, n_and = 0;
    const uint32_t* list_in = p.list_in;
    uint32_t count = 0;
    uint32_t* bits_out = p.bitmap_out;
    int32_t hop = -1;
    if (p.dispatch) {
      const int h = st->sched[p.hop];  // p.hop is the chain slot
      hop = h;
      int run = 0;
      work = h >= 0 && k1_runs(st, h, &run);
      if (work) {
        if (h == 0) {  // the batch: its position range, or the caller's selection
          list_in = p.sel0;
          count = p.sel0 ? *p.sel0_count : p.range_n;
        } else {
          list_in = p.lists + static_cast<uint64_t>(h) * p.list_stride;
          count = p.counts[h];
        }
        for (int r = 0; r < run; ++r) s_run_id[r] = st->order[h + r];
        nrun = run;
        bits_out = p.bits + static_cast<uint64_t>(h) * p.bits_stride;
      }
    } else {
      count = list_in ? *p.count_in : p.range_n;
      n_and = p.n_and;
      for (int a = 0; a < n_and; ++a) s_and[a] = p.and_bits[a];
      if (p.explicit_pred >= 0) {
        s_run_id[0] = p.explicit_pred;
        nrun = 1;
      }
    }
    int need_id = 0, need_bbox = 0, need_label = 0;
    for (int r = 0; r < nrun; ++r) {
      const PredDev& q = p.preds[s_run_id[r]];
      if (q.kind == kHash) {
        need_id = 1;
        if (q.units_per_area > 0) need_bbox = 1;
      } else {
        need_label = 1;
      }
      if (q.cache_known) need_id = 1;  // the verdict cache is keyed by tuple id
    }
    s_work = work;
    s_nrun = nrun;
    s_n_and = n_and;
    s_list_in = list_in;
    s_count = count;
    s_range_base = p.range_base;
    s_bits_out = bits_out;
    s_need_id = need_id;
    s_need_bbox = need_bbox;
    s_need_label = need_label;
    // lean path: a run of at most 4 LABEL_EQ / uniform-units HASH predicates over a position range
    // (the usual first hop), no verdict cache, no AND inputs, no per-area units, no compacted HASH
    int lean = (nrun >= 1 && nrun <= kLeanMaxRun && !need_bbox && n_and == 0 && list_in == nullptr) ? 1 : 0;
    for (int r = 0; r < nrun && lean; ++r) {
      const PredDev& q = p.preds[s_run_id[r]];
      if (q.cache_known || (q.kind == kHash && q.units >= kCompactUnits)) lean = 0;
    }
    s_lean = lean;
    s_hop = hop;
  }
  __syncthreads();
  if (!s_work) {
    // hop h is a classifier hop: clear the segment counts its K4 accumulates into
    const int h = s_hop;
    if (p.dispatch && h >= 0 && h < st->n_pred && is_classifier(st->kind[st->order[h]])) {
      const uint32_t n = h == 0 ? (p.sel0 ? *p.sel0_count : p.range_n) : p.counts[h];
      const uint32_t nseg = (n + kRouteTile - 1) / kRouteTile;
      for (uint32_t i = blockIdx.x * kRouteThreads + tid; i < nseg; i += gridDim.x * kRouteThreads) p.seg_counts[i] = 0;
      for (uint32_t i = blockIdx.x * kRouteThreads + tid; i < nseg * (kRouteTile / kWarpSeg); i += gridDim.x * kRouteThreads)
        p.warp_counts[i] = 0;
    }
    return;
  }
  const int nrun = s_nrun;
  if (tid < nrun) s_pred[tid] = p.preds[s_run_id[tid]];
  if (lane < kMaxPred) {
    s_in[warp][lane] = 0;
    s_pass[warp][lane] = 0;
    s_comp[warp][lane] = 0;
    s_cost[warp][lane] = 0;
  }
  __syncthreads();
  const uint32_t count = s_count;
  const uint32_t num_tiles = (count + kRouteTile - 1) / kRouteTile;
  const int n_and = s_n_and;
  const uint32_t* list_in = s_list_in;
  const uint32_t base = s_range_base;
  uint32_t* bits_out = s_bits_out;
  const bool need_id = s_need_id, need_bbox = s_need_bbox, need_label = s_need_label;

  uint32_t buf = 0;
  if (s_lean) {
    // ---- lean path: the columns of kTiles tiles are loaded before any is evaluated (labels 16 B,
    // ids 64 B per thread and tile), then each tile runs the predicates in order on 8 positions
    // per thread (HASH branch-free: 8 independent chains), writes the bitmap and the counts.
    // Statistics stay in registers (at most kLeanMaxRun predicates, unrolled) and are reduced
    // once; the cost charged is the generic path's quantity, sum over warp-tiles of cycles x
    // items evaluated (t0 / t1 are the warp's clock, so summing per thread gives it).
    const bool lab_aligned = ((reinterpret_cast<uintptr_t>(p.label + base)) & 15u) == 0;
    const bool id_aligned = ((reinterpret_cast<uintptr_t>(p.id + base)) & 15u) == 0;
    uint32_t n_in[kLeanMaxRun], n_pass[kLeanMaxRun];
    unsigned long long cost[kLeanMaxRun];
#pragma unroll
    for (int r = 0; r < kLeanMaxRun; ++r) n_in[r] = n_pass[r] = 0, cost[r] = 0;
    const uint32_t want0 = static_cast<uint32_t>(s_pred[0].label_value) & 0xFFFFu;
    auto lean_loop = [&](auto tiles_c, auto ids_c, auto one_label_c) {
      constexpr int kTiles = decltype(tiles_c)::value;
      constexpr bool kIds = decltype(ids_c)::value;
      constexpr bool kOneLabel = decltype(one_label_c)::value;  // the run is a single LABEL_EQ
      for (uint32_t t0i = blockIdx.x; t0i < num_tiles; t0i += kTiles * gridDim.x) {
        uint32_t labs[kTiles][kRouteItems / 2];
        uint64_t ids[kTiles][kIds ? kRouteItems : 1];
        uint32_t avail[kTiles];
#pragma unroll
        for (int u = 0; u < kTiles; ++u) {
          const uint32_t t = t0i + u * gridDim.x;
          const uint32_t p0 = t * kRouteTile + tid * kRouteItems;
          avail[u] = (t < num_tiles && p0 < count) ? min(count - p0, static_cast<uint32_t>(kRouteItems)) : 0u;
          const bool full = avail[u] == static_cast<uint32_t>(kRouteItems);
          labs[u][0] = labs[u][1] = labs[u][2] = labs[u][3] = 0u;
          if (need_label) {
            if (full && lab_aligned) {
              const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.label + base + p0));
              labs[u][0] = v.x; labs[u][1] = v.y; labs[u][2] = v.z; labs[u][3] = v.w;
            } else {
#pragma unroll
              for (int j = 0; j < kRouteItems; ++j)
                if (static_cast<uint32_t>(j) < avail[u])
                  labs[u][j >> 1] |= static_cast<uint32_t>(__ldg(p.label + base + p0 + j)) << (16 * (j & 1));
            }
          }
          if constexpr (kIds) {
            if (full && id_aligned) {
              const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p.id + base + p0);
#pragma unroll
              for (int j = 0; j < kRouteItems / 2; ++j) {
                const ulonglong2 v = __ldg(q + j);
                ids[u][2 * j] = v.x;
                ids[u][2 * j + 1] = v.y;
              }
            } else {
#pragma unroll
              for (int j = 0; j < kRouteItems; ++j)
                ids[u][j] = static_cast<uint32_t>(j) < avail[u] ? __ldg(p.id + base + p0 + j) : 0ull;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kTiles; ++u) {
          const uint32_t t = t0i + u * gridDim.x;
          if (t >= num_tiles) break;  // CTA-uniform
          const uint32_t p0 = t * kRouteTile + tid * kRouteItems;
          uint32_t mask = avail[u] >= static_cast<uint32_t>(kRouteItems) ? 0xFFu : ((1u << avail[u]) - 1u);
          if constexpr (kOneLabel) {
            const uint32_t in_mask = mask;
            const long long c0 = clock64();
#pragma unroll
            for (int j = 0; j < kRouteItems; ++j)
              if (((labs[u][j >> 1] >> (16 * (j & 1))) & 0xFFFFu) != want0) mask &= ~(1u << j);
            const long long c1 = clock64();
            n_in[0] += __popc(in_mask);
            n_pass[0] += __popc(mask);
            cost[0] += static_cast<unsigned long long>(c1 - c0) * __popc(in_mask);
          }
#pragma unroll
          for (int r = 0; r < kLeanMaxRun; ++r) {
            if (kOneLabel || r >= nrun) break;
            const PredDev& pd = s_pred[r];
            const uint32_t in_mask = mask;
            const long long c0 = clock64();
            if (pd.kind == kLabelEq) {
              const uint32_t want = static_cast<uint32_t>(pd.label_value) & 0xFFFFu;
#pragma unroll
              for (int j = 0; j < kRouteItems; ++j)
                if (((labs[u][j >> 1] >> (16 * (j & 1))) & 0xFFFFu) != want) mask &= ~(1u << j);
            } else if constexpr (kIds) {  // HASH, uniform units, all 8 positions branch-free
              uint32_t hv[kRouteItems];
#pragma unroll
              for (int j = 0; j < kRouteItems; ++j) hv[j] = static_cast<uint32_t>(splitmix64(ids[u][j] ^ pd.seed) >> 32);
              for (int rr = 0; rr < pd.units; ++rr) {
#pragma unroll
                for (int j = 0; j < kRouteItems; ++j) hv[j] = fmix32(hv[j] + static_cast<uint32_t>(rr));
              }
              uint32_t fail = 0;
              if (pd.thr0 == pd.thr1) {
                if (pd.thr0 <= 0xFFFFFFFFull) {
                  const uint32_t T32 = static_cast<uint32_t>(pd.thr0);
#pragma unroll
                  for (int j = 0; j < kRouteItems; ++j) fail |= (hv[j] >= T32 ? 1u : 0u) << j;
                }
              } else {
#pragma unroll
                for (int j = 0; j < kRouteItems; ++j) {
                  const uint64_t T = (ids[u][j] >= pd.drift_id) ? pd.thr1 : pd.thr0;
                  fail |= (static_cast<uint64_t>(hv[j]) < T ? 0u : 1u) << j;
                }
              }
              mask &= ~fail;
            }
            const long long c1 = clock64();
            n_in[r] += __popc(in_mask);
            n_pass[r] += __popc(mask);
            cost[r] += static_cast<unsigned long long>(c1 - c0) * __popc(in_mask);
          }
          uint32_t wbits = mask << (8 * (lane & 3));
          wbits |= __shfl_xor_sync(kFull, wbits, 1);
          wbits |= __shfl_xor_sync(kFull, wbits, 2);
          if ((lane & 3) == 0 && p0 < count) bits_out[p0 >> 5] = wbits;
          const uint32_t wc = __reduce_add_sync(kFull, __popc(mask));
          if (lane == 0) {
            s_warp_cnt[buf][warp] = wc;
            p.warp_counts[t * (kRouteTile / kWarpSeg) + warp] = wc;
          }
          __syncthreads();  // the other buffer is rewritten only after the next tile's barrier
          if (tid == 0) {
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < kRouteThreads / 32; ++w) tot += s_warp_cnt[buf][w];
            p.seg_counts[t] = tot;
          }
          buf ^= 1u;
        }
      }
    };
    if (need_id)
      lean_loop(std::integral_constant<int, 2>{}, std::true_type{}, std::false_type{});
    else if (nrun == 1)
      lean_loop(std::integral_constant<int, 4>{}, std::false_type{}, std::true_type{});
    else
      lean_loop(std::integral_constant<int, 4>{}, std::false_type{}, std::false_type{});
    if (p.collect_stats) {
#pragma unroll
      for (int r = 0; r < kLeanMaxRun; ++r) {
        const uint32_t a = __reduce_add_sync(kFull, n_in[r]);
        const uint32_t b = __reduce_add_sync(kFull, n_pass[r]);
        unsigned long long c = cost[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
        if (lane == 0 && r < nrun) {
          s_in[warp][r] = a;
          s_pass[warp][r] = b;
          s_comp[warp][r] = a;
          s_cost[warp][r] = c;
        }
      }
    }
  } else  // ---- generic path: any run of cheap predicates, range or list input, caches, AND inputs
  for (uint32_t t = blockIdx.x; t < num_tiles; t += gridDim.x, buf ^= 1u) {
    const uint32_t p0 = t * kRouteTile + tid * kRouteItems;
    uint32_t idx[kRouteItems];
    uint32_t mask = 0;
    if (list_in) {
      if (p0 + kRouteItems <= count) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(list_in + p0));
        const uint4 b = __ldg(reinterpret_cast<const uint4*>(list_in + p0 + 4));
        idx[0] = a.x; idx[1] = a.y; idx[2] = a.z; idx[3] = a.w;
        idx[4] = b.x; idx[5] = b.y; idx[6] = b.z; idx[7] = b.w;
        mask = 0xFFu;
      } else {
#pragma unroll
        for (int j = 0; j < kRouteItems; ++j) {
          idx[j] = 0;
          if (p0 + j < count) {
            idx[j] = __ldg(list_in + p0 + j);
            mask |= 1u << j;
          }
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < kRouteItems; ++j) {
        idx[j] = base + p0 + j;
        if (p0 + j < count) mask |= 1u << j;
      }
    }
    for (int a = 0; a < n_and; ++a) {
      if (mask) mask &= (__ldg(s_and[a] + (p0 >> 5)) >> (p0 & 31)) & 0xFFu;
    }
    const bool contiguous = (list_in == nullptr) && (mask == 0xFFu) && (((base + p0) & 7u) == 0);

    // columns the run needs, loaded once for the alive items (outside the per-predicate timing)
    uint64_t ids[kRouteItems];
    uint64_t bbs[kRouteItems];
    uint32_t labs[kRouteItems / 2];
    if (mask) {
      if (need_id) {
        if (contiguous && ((reinterpret_cast<uintptr_t>(p.id + base + p0) & 15u) == 0)) {
          const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p.id + base + p0);
#pragma unroll
          for (int j = 0; j < kRouteItems / 2; ++j) {
            const ulonglong2 v = __ldg(q + j);
            ids[2 * j] = v.x;
            ids[2 * j + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int j = 0; j < kRouteItems; ++j) ids[j] = ((mask >> j) & 1u) ? __ldg(p.id + idx[j]) : 0ull;
        }
      }
      if (need_bbox) {
#pragma unroll
        for (int j = 0; j < kRouteItems; ++j) bbs[j] = ((mask >> j) & 1u) ? __ldg(p.bbox + idx[j]) : 0ull;
      }
      if (need_label) {
        if (contiguous && ((reinterpret_cast<uintptr_t>(p.label + base + p0) & 15u) == 0)) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.label + base + p0));
          labs[0] = v.x; labs[1] = v.y; labs[2] = v.z; labs[3] = v.w;
        } else {
#pragma unroll
          for (int j = 0; j < kRouteItems / 2; ++j) {
            const uint32_t lo = ((mask >> (2 * j)) & 1u) ? __ldg(p.label + idx[2 * j]) : 0u;
            const uint32_t hi = ((mask >> (2 * j + 1)) & 1u) ? __ldg(p.label + idx[2 * j + 1]) : 0u;
            labs[j] = lo | (hi << 16);
          }
        }
      }
    }

    for (int r = 0; r < nrun; ++r) {
      const PredDev& pd = s_pred[r];
      const long long t0 = clock64();
      const uint32_t in_mask = mask;
      // verdict cache: alive items whose verdict is known are not evaluated
      uint32_t cm = 0, cpass = 0;
      if (pd.cache_known && mask) {
#pragma unroll
        for (int j = 0; j < kRouteItems; ++j) {
          if (((mask >> j) & 1u) && ids[j] < pd.cache_cap) {
            const uint64_t v = ids[j];
            const uint32_t kw = __ldg(pd.cache_known + (v >> 5)), pw = __ldg(pd.cache_pass + (v >> 5));
            cm |= ((kw >> (v & 31)) & 1u) << j;
            cpass |= ((pw >> (v & 31)) & 1u) << j;
          }
        }
        cpass &= cm;
        mask &= ~cm;  // evaluate the rest (mask = the items this predicate computes)
      }
      const uint32_t todo = mask;
      // compact only expensive HASH predicates: at 1 round the dense chains overlap better (measured),
      // but SIMT evaluates every position of a warp with any alive one, so without compaction an
      // expensive predicate costs the same whatever its input selectivity (the eddy's saving is lost)
      bool compacted = false;
      if (kCompact && pd.kind == kHash && pd.units >= kCompactUnits && pd.units_per_area <= 0) {  // CTA-uniform
        const uint32_t c = __popc(mask);
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) s_cw[warp] = x;
        __syncthreads();
        uint32_t wo = 0, n_cta = 0;
#pragma unroll
        for (int w2 = 0; w2 < kRouteThreads / 32; ++w2) {
          const uint32_t v = s_cw[w2];
          wo += w2 < warp ? v : 0u;
          n_cta += v;
        }
        if (n_cta > 0 && 4u * n_cta <= 3u * static_cast<uint32_t>(kRouteTile)) {
          // CTA-wide compaction: the tile's alive ids -> s_cids in position order, every thread then
          // hashes 4 entries at a time (independent chains), verdicts come back as ballot words
          compacted = true;
          const uint32_t off = wo + x - c;
          uint64_t* buf = &s_cids[0][0];
          uint32_t k = off;
#pragma unroll
          for (int j = 0; j < kRouteItems; ++j)
            if ((mask >> j) & 1u) buf[k++] = ids[j];
          __syncthreads();
          // ceil(n / 256) entries per thread (1..6 at <= 75% alive), as independent chains
          const uint32_t m = (n_cta + kRouteThreads - 1) / kRouteThreads;
          switch (m) {
            case 1: hash_compacted<1>(pd, buf, n_cta, tid, lane, warp, s_vw); break;
            case 2: hash_compacted<2>(pd, buf, n_cta, tid, lane, warp, s_vw); break;
            case 3: hash_compacted<3>(pd, buf, n_cta, tid, lane, warp, s_vw); break;
            case 4: hash_compacted<4>(pd, buf, n_cta, tid, lane, warp, s_vw); break;
            case 5: hash_compacted<5>(pd, buf, n_cta, tid, lane, warp, s_vw); break;
            default: hash_compacted<6>(pd, buf, n_cta, tid, lane, warp, s_vw); break;
          }
          __syncthreads();
          const uint32_t w0 = c ? s_vw[off >> 5] : 0u;
          const uint32_t w1 = (c && ((off & 31u) + c > 32u)) ? s_vw[(off >> 5) + 1] : 0u;
          const uint32_t fb = __funnelshift_r(w0, w1, off & 31u) & ((1u << c) - 1u);  // this thread's entries
          uint32_t fail = 0, t = 0;
#pragma unroll
          for (int j = 0; j < kRouteItems; ++j) {
            if ((mask >> j) & 1u) {
              fail |= ((fb >> t) & 1u) << j;
              ++t;
            }
          }
          mask &= ~fail;
        }
        __syncthreads();  // s_cw / s_cids / s_vw are reused by the next predicate or tile
      }
      if (!compacted && mask) {
        if (pd.kind == kLabelEq) {
          const uint32_t want = static_cast<uint32_t>(pd.label_value) & 0xFFFFu;
#pragma unroll
          for (int j = 0; j < kRouteItems; ++j)
            if (((labs[j >> 1] >> (16 * (j & 1))) & 0xFFFFu) != want) mask &= ~(1u << j);
        } else if (pd.units_per_area > 0) {  // HASH with per-tuple units (cfg4): per-item loop
#pragma unroll
          for (int j = 0; j < kRouteItems; ++j) {
            if ((mask >> j) & 1u) {
              if (!hash_pass(pd, ids[j], bbs[j])) mask &= ~(1u << j);
            }
          }
        } else {  // HASH, uniform units: the 8 items branch-free (independent chains, no divergence)
          uint32_t hv[kRouteItems];
#pragma unroll
          for (int j = 0; j < kRouteItems; ++j) hv[j] = static_cast<uint32_t>(splitmix64(ids[j] ^ pd.seed) >> 32);
          for (int r = 0; r < pd.units; ++r) {
#pragma unroll
            for (int j = 0; j < kRouteItems; ++j) hv[j] = fmix32(hv[j] + static_cast<uint32_t>(r));
          }
          uint32_t fail = 0;
          if (pd.thr0 == pd.thr1) {  // no drift: one threshold; T >= 2^32 passes everything
            if (pd.thr0 <= 0xFFFFFFFFull) {
              const uint32_t T32 = static_cast<uint32_t>(pd.thr0);
#pragma unroll
              for (int j = 0; j < kRouteItems; ++j) fail |= (hv[j] >= T32 ? 1u : 0u) << j;
            }
          } else {
#pragma unroll
            for (int j = 0; j < kRouteItems; ++j) {
              const uint64_t T = (ids[j] >= pd.drift_id) ? pd.thr1 : pd.thr0;
              fail |= (static_cast<uint64_t>(hv[j]) < T ? 0u : 1u) << j;
            }
          }
          mask &= ~fail;
        }
      }
      const long long t1 = clock64();
      if (pd.cache_known) {
        if ((pd.cache_fill || p.force_fill) && todo) {  // record the verdicts this predicate computed
#pragma unroll
          for (int j = 0; j < kRouteItems; ++j) {
            if (((todo >> j) & 1u) && ids[j] < pd.cache_cap) {
              const uint64_t v = ids[j];
              const uint32_t bit = 1u << (v & 31);
              if ((mask >> j) & 1u) atomicOr(pd.cache_pass + (v >> 5), bit);
              atomicOr(pd.cache_known + (v >> 5), bit);
            }
          }
        }
        mask |= cpass;  // cached passes rejoin the alive set
      }
      if (p.collect_stats) {
        const uint32_t ci = __reduce_add_sync(kFull, __popc(in_mask));
        const uint32_t cp = __reduce_add_sync(kFull, __popc(mask));
        const uint32_t cc = pd.cache_known ? __reduce_add_sync(kFull, __popc(todo)) : ci;
        if (lane == 0) {
          s_in[warp][r] += ci;
          s_pass[warp][r] += cp;
          s_comp[warp][r] += cc;
          // dense-equivalent cost: SIMT lanes without an item to evaluate idle, so the warp's cycles
          // are charged in proportion to the items it evaluated (cc of 256); SM-cycles = raw / (256 *
          // warps/SM).  Cache hits cost nothing (PAPER.md:604 assumes the lookup overhead negligible)
          s_cost[warp][r] += static_cast<unsigned long long>(t1 - t0) * cc;
        }
      }
    }

    // verdict bitmap (4 threads per 32-bit word) and the tile's survivor count
    uint32_t wbits = mask << (8 * (lane & 3));
    wbits |= __shfl_xor_sync(kFull, wbits, 1);
    wbits |= __shfl_xor_sync(kFull, wbits, 2);
    if ((lane & 3) == 0 && p0 < count) bits_out[p0 >> 5] = wbits;
    const uint32_t wc = __reduce_add_sync(kFull, __popc(mask));
    if (lane == 0) {
      s_warp_cnt[buf][warp] = wc;
      p.warp_counts[t * (kRouteTile / kWarpSeg) + warp] = wc;
    }
    __syncthreads();  // the other buffer is rewritten only after the next tile's barrier
    if (tid == 0) {
      uint32_t tot = 0;
#pragma unroll
      for (int w = 0; w < kRouteThreads / 32; ++w) tot += s_warp_cnt[buf][w];
      p.seg_counts[t] = tot;
    }
  }

  __syncthreads();
  if (p.collect_stats && tid < nrun) {
    const int k = s_run_id[tid];
    unsigned long long in = 0, pass = 0, cost = 0, comp = 0;
#pragma unroll
    for (int w = 0; w < kRouteThreads / 32; ++w) {
      in += s_in[w][tid];
      pass += s_pass[w][tid];
      cost += s_cost[w][tid];
      comp += s_comp[w][tid];
    }
    atomicAdd(&st->d_in[k], in);
    atomicAdd(&st->d_pass[k], pass);
    atomicAdd(&st->d_cost[k], cost);
    atomicAdd(&st->d_comp[k], comp);
  }
}

// ------------------------------------------------------------------------------------------
// K2: order-preserving compaction (eager materialization).  CTA c owns
// segments [4c, 4c + 4); its output offset is the sum of all earlier segments' counts (<= a few
// thousand L2-resident words), so no CTA ever waits for another.  Within a segment each warp owns
// a 256-position slice whose offset comes from the evaluator's per-warp counts: warp scan only,
// no block barrier; survivors are written in input order.
#ifndef HYDRO_K2_MINB
#define HYDRO_K2_MINB 4  // 64 registers: 4 CTAs per SM with the first segment preloaded (measured best of 1, 3, 4, 5, 6)
#endif
#ifndef HYDRO_K2_DENSE_DIV
#define HYDRO_K2_DENSE_DIV 10  // emit reads whole row columns once >= 1 in HYDRO_K2_DENSE_DIV positions survive
#endif
__global__ void __launch_bounds__(kRouteThreads, HYDRO_K2_MINB) hydro_compact_kernel(CompactParams p) {
  __shared__ uint32_t s_red[kRouteThreads / 32];
  __shared__ int32_t s_work, s_emit;
  __shared__ const uint32_t* s_list_in;
  __shared__ const uint32_t* s_bits;
  __shared__ uint32_t* s_list_out;
  __shared__ uint32_t* s_count_out;
  __shared__ uint32_t s_count, s_emit_off;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    int32_t work = 1, emit = p.emit;
    const uint32_t* list_in = p.list_in;
    const uint32_t* bits = p.bits_in;
    uint32_t* list_out = p.list_out;
    uint32_t* count_out = p.count_out;
    uint32_t count = 0;
    if (p.dispatch) {
      const DevState* st = p.st;
      const int h = st->sched[p.hop], P = st->n_pred;  // p.hop is the chain slot
      int run = 0;
      int next;
      if (h < 0) {
        work = 0;
        next = 0;
      } else if (k1_runs(st, h, &run)) {
        next = h + run;
      } else if (h < P && is_classifier(st->kind[st->order[h]])) {
        next = h + (is_pair_hop(st->order, P, h, st->pair_a, st->pair_b) ? 2 : 1);  // a fused pair covers two
      } else {
        work = 0;
        next = 0;
      }
      if (work) {
        if (h == 0) {  // the batch: its position range, or the caller's selection
          list_in = p.sel0;
          count = p.sel0 ? *p.sel0_count : p.range_n;
        } else {
          list_in = p.lists + static_cast<uint64_t>(h) * p.list_stride;
          count = p.counts[h];
        }
        bits = p.bits + static_cast<uint64_t>(h) * p.bits_stride;
        emit = next >= P;
        if (!emit) {
          list_out = p.lists + static_cast<uint64_t>(next) * p.list_stride;
          count_out = p.counts + next;
        }
      }
    } else {
      count = list_in ? *p.count_in : p.range_n;
    }
    s_work = work;
    s_emit = emit;
    s_list_in = list_in;
    s_bits = bits;
    s_list_out = list_out;
    s_count_out = count_out;
    s_count = count;
    s_emit_off = (emit && p.emit_offset) ? *p.emit_offset : 0u;
  }
  __syncthreads();
  if (!s_work) return;
  const uint32_t count = s_count;
  const uint32_t nseg = (count + kRouteTile - 1) / kRouteTile;
  const uint32_t seg0 = blockIdx.x * kCompactSegs;
  const bool emit = s_emit;
  const uint32_t* list_in = s_list_in;
  const uint32_t* bits = s_bits;
  const uint32_t base = p.range_base;
  if (seg0 >= nseg && !(nseg == 0 && blockIdx.x == 0)) return;

  // The first segment's rows are loaded before the prefix sum (they do not depend on it), so
  // their DRAM latency overlaps the prefix's L2 loads.  Dense = the emit reads the thread's 8 rows
  // contiguously (see below); the segment total comes from the evaluator's seg_counts.
  uint32_t sidx[kRouteItems];
  uint64_t sid[kRouteItems], sbb[kRouteItems];
  auto dense_seg = [&](uint32_t sg, uint32_t total) {
    const uint32_t q0 = sg * kRouteTile + tid * kRouteItems;
    return emit && !list_in && total * static_cast<uint32_t>(HYDRO_K2_DENSE_DIV) >= static_cast<uint32_t>(kRouteTile) &&
           q0 + kRouteItems <= count &&
           ((reinterpret_cast<uintptr_t>(p.id + base + q0) | reinterpret_cast<uintptr_t>(p.bbox + base + q0)) & 15u) == 0u;
  };
  auto load_dense = [&](uint32_t sg) {
    const uint32_t q0 = sg * kRouteTile + tid * kRouteItems;
    const ulonglong2* qi = reinterpret_cast<const ulonglong2*>(p.id + base + q0);
    const ulonglong2* qb = reinterpret_cast<const ulonglong2*>(p.bbox + base + q0);
#pragma unroll
    for (int j = 0; j < kRouteItems / 2; ++j) {
      const ulonglong2 a = __ldg(qi + j), b = __ldg(qb + j);
      sid[2 * j] = a.x;
      sid[2 * j + 1] = a.y;
      sbb[2 * j] = b.x;
      sbb[2 * j + 1] = b.y;
    }
  };
  const bool pre = seg0 < nseg && dense_seg(seg0, __ldg(p.seg_counts + seg0));
  if (pre) load_dense(seg0);

  // output offset of this CTA: survivors of every earlier segment
  uint32_t part = 0;
  {  // seg0 is a multiple of 4 (kCompactSegs): 16-byte loads, independent so they overlap
    const uint4* sc4 = reinterpret_cast<const uint4*>(p.seg_counts);
#pragma unroll 4
    for (uint32_t s = tid; s < seg0 / 4; s += kRouteThreads) {
      const uint4 v = __ldg(sc4 + s);
      part += v.x + v.y + v.z + v.w;
    }
  }
  part = __reduce_add_sync(kFull, part);
  if (lane == 0) s_red[warp] = part;
  __syncthreads();
  uint32_t prefix = 0;
#pragma unroll
  for (int w = 0; w < kRouteThreads / 32; ++w) prefix += s_red[w];
  prefix += s_emit_off;

  const uint32_t seg1 = min(seg0 + kCompactSegs, nseg);
  // Each warp walks its own 256-position slice of every segment, independently of the other
  // warps: its output offset is the segment's offset plus the survivors of the earlier warp
  // slices of the same segment (warp counts written by the evaluator), so there is no barrier.
  constexpr uint32_t kWarpsPerSeg = kRouteTile / kWarpSeg;
  for (uint32_t sgi = seg0; sgi < seg1; ++sgi) {
    const uint32_t wcv = lane < kWarpsPerSeg ? __ldg(p.warp_counts + sgi * kWarpsPerSeg + lane) : 0u;
    const uint32_t wexcl = __reduce_add_sync(kFull, lane < static_cast<uint32_t>(warp) ? wcv : 0u);
    const uint32_t seg_total = __reduce_add_sync(kFull, wcv);
    const uint32_t p0 = sgi * kRouteTile + tid * kRouteItems;
    uint32_t mask = 0;
    if (p0 < count) {
      mask = (__ldg(bits + (p0 >> 5)) >> (p0 & 31)) & 0xFFu;
      if (p0 + kRouteItems > count) mask &= (1u << (count - p0)) - 1u;
    }
    // emit from a dense range segment (>= 1 in 10 positions survive): the scattered gathers would
    // touch most DRAM bursts of the id / bbox columns anyway, so read the thread's 8 rows
    // contiguously (16-byte loads, fully coalesced) and keep the survivors
    const bool dense = dense_seg(sgi, seg_total);
    if (dense) {
      if (!(pre && sgi == seg0)) load_dense(sgi);
#pragma unroll
      for (int j = 0; j < kRouteItems; ++j) sidx[j] = base + p0 + j;
    } else {
#pragma unroll
      for (int j = 0; j < kRouteItems; ++j) {
        sidx[j] = 0;
        sid[j] = 0;
        sbb[j] = 0;
        if ((mask >> j) & 1u) {
          sidx[j] = list_in ? __ldg(list_in + p0 + j) : base + p0 + j;
          if (emit) {
            sid[j] = __ldg(p.id + sidx[j]);
            sbb[j] = __ldg(p.bbox + sidx[j]);
          }
        }
      }
    }
    const uint32_t c = __popc(mask);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    uint32_t pos = prefix + wexcl + (x - c);
    if (mask) {
      if (!emit) {
#pragma unroll
        for (int j = 0; j < kRouteItems; ++j)
          if ((mask >> j) & 1u) s_list_out[pos++] = sidx[j];
      } else {
#pragma unroll
        for (int j = 0; j < kRouteItems; ++j) {
          if ((mask >> j) & 1u) {
            p.out_ids[pos] = sid[j];
            p.out_bbox[pos] = sbb[j];
            if (p.out_pos) p.out_pos[pos] = sidx[j];
            ++pos;
          }
        }
      }
    }
    prefix += seg_total;
  }
  // the CTA holding the last segment publishes the count
  const bool last = (nseg == 0) ? (blockIdx.x == 0) : (seg1 == nseg);
  if (last && tid == 0) {
    if (emit) *p.emit_count = prefix;
    else *s_count_out = prefix;
  }
}

// ------------------------------------------------------------------------------------------
// K1F: the whole chain of a context without classifiers (LABEL_EQ / HASH predicates, range input,
// no verdict caches) in ONE pass: evaluate the run in the device order, then emit the survivors'
// (id, bbox) rows directly (eager materialization) at the offset given by a
// single-pass decoupled look-back over 2048-position tiles taken in increasing order from an
// atomic counter (a tile publishes its survivor count before it looks back, so it never waits on
// a tile that has not started).  Replaces K1 + K2 for such chains: the ids are read once (K2 used
// to re-read the id and bbox columns to emit), and only the survivors' bboxes are gathered.
// Statistics as K1's lean path (in / pass / computed per predicate, dense-equivalent cycles).
constexpr unsigned long long kLbAggregate = 1ull << 62, kLbPrefix = 2ull << 62, kLbFlags = 3ull << 62;

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

#ifndef HYDRO_K1F_MINB
#define HYDRO_K1F_MINB 4
#endif
#ifndef HYDRO_K1F_ITEMS
#define HYDRO_K1F_ITEMS 8
#endif
constexpr int kFItems = HYDRO_K1F_ITEMS;           // positions per thread
constexpr int kFTile = kRouteThreads * kFItems;     // positions per tile
__global__ void __launch_bounds__(kRouteThreads, HYDRO_K1F_MINB) hydro_route_emit_kernel(FusedParams f) {
  const RouteParams& p = f.r;
  __shared__ PredDev s_pred[kMaxPred];
  __shared__ int32_t s_pid[kMaxPred];
  __shared__ uint32_t s_wcnt[kRouteThreads / 32];
  __shared__ uint32_t s_tile, s_excl;
  __shared__ unsigned long long s_stat[kRouteThreads / 32][kFusedMaxRun][3];  // in, pass, cost per warp
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  DevState* st = p.st;
  const int P = st->n_pred;
  if (tid < P) {
    s_pid[tid] = st->order[tid];
    s_pred[tid] = p.preds[st->order[tid]];
  }
  __syncthreads();
  bool need_label = false, need_id = false;
  for (int r = 0; r < P; ++r) {
    if (s_pred[r].kind == kHash) need_id = true;
    else need_label = true;
  }
  const uint32_t count = p.range_n, base = p.range_base;
  const uint32_t ntiles = (count + kFTile - 1) / kFTile;
  const uint32_t emit_off = f.emit_offset ? *f.emit_offset : 0u;
  const bool lab_aligned = ((reinterpret_cast<uintptr_t>(p.label + base)) & 15u) == 0;
  const bool id_aligned = ((reinterpret_cast<uintptr_t>(p.id + base)) & 15u) == 0;
  // statistics: per warp in shared memory (lane 0 adds the warp's sums after each predicate)
  if (lane == 0)
    for (int r = 0; r < kFusedMaxRun; ++r) s_stat[warp][r][0] = s_stat[warp][r][1] = s_stat[warp][r][2] = 0;

  uint32_t it_k = 0;
  while (true) {
#ifdef HYDRO_K1F_DYNAMIC
    if (tid == 0) s_tile = atomicAdd(f.tile_counter, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
#else
    // static round-robin tiles: every CTA is co-resident (grid = occupancy x SMs) and walks its
    // tiles in increasing order, so a tile's predecessors always make progress
    const uint32_t t = blockIdx.x + it_k * gridDim.x;
    ++it_k;
#endif
    if (t >= ntiles) break;
    const uint32_t p0 = t * kFTile + tid * kFItems;
    const uint32_t avail = p0 < count ? min(count - p0, static_cast<uint32_t>(kFItems)) : 0u;
    const bool full = avail == static_cast<uint32_t>(kFItems);
    uint32_t labs[kFItems / 2];
#pragma unroll
    for (int j = 0; j < kFItems / 2; ++j) labs[j] = 0u;
    uint64_t ids[kFItems];
    if (need_label) {
      if (full && lab_aligned && kFItems == 8) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.label + base + p0));
        labs[0] = v.x; labs[1] = v.y; labs[kFItems / 2 - 2] = v.z; labs[kFItems / 2 - 1] = v.w;
      } else if (full && lab_aligned && kFItems == 4) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(p.label + base + p0));
        labs[0] = v.x; labs[1] = v.y;
      } else {
#pragma unroll
        for (int j = 0; j < kFItems; ++j)
          if (static_cast<uint32_t>(j) < avail)
            labs[j >> 1] |= static_cast<uint32_t>(__ldg(p.label + base + p0 + j)) << (16 * (j & 1));
      }
    }
    if (need_id && full && id_aligned) {
      const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p.id + base + p0);
#pragma unroll
      for (int j = 0; j < kFItems / 2; ++j) {
        const ulonglong2 v = __ldg(q + j);
        ids[2 * j] = v.x;
        ids[2 * j + 1] = v.y;
      }
    } else if (need_id) {
#pragma unroll
      for (int j = 0; j < kFItems; ++j)
        ids[j] = static_cast<uint32_t>(j) < avail ? __ldg(p.id + base + p0 + j) : 0ull;
    }
    uint32_t mask = full ? ((1u << kFItems) - 1u) : ((1u << avail) - 1u);
    for (int r = 0; r < P; ++r) {
      const PredDev& pd = s_pred[r];
      const uint32_t in_mask = mask;
      const long long c0 = clock64();
      if (pd.kind == kLabelEq) {
        const uint32_t want = static_cast<uint32_t>(pd.label_value) & 0xFFFFu;
#pragma unroll
        for (int j = 0; j < kFItems; ++j)
          if (((labs[j >> 1] >> (16 * (j & 1))) & 0xFFFFu) != want) mask &= ~(1u << j);
      } else {  // HASH, uniform units, all positions branch-free
        uint32_t hv[kFItems];
#pragma unroll
        for (int j = 0; j < kFItems; ++j) hv[j] = static_cast<uint32_t>(splitmix64(ids[j] ^ pd.seed) >> 32);
        for (int rr = 0; rr < pd.units; ++rr) {
#pragma unroll
          for (int j = 0; j < kFItems; ++j) hv[j] = fmix32(hv[j] + static_cast<uint32_t>(rr));
        }
        uint32_t fail = 0;
#pragma unroll
        for (int j = 0; j < kFItems; ++j) {
          const uint64_t T = (ids[j] >= pd.drift_id) ? pd.thr1 : pd.thr0;
          fail |= (static_cast<uint64_t>(hv[j]) < T ? 0u : 1u) << j;
        }
        mask &= ~fail;
      }
      const long long c1 = clock64();
      if (p.collect_stats) {
        const uint32_t a_in = __reduce_add_sync(kFull, __popc(in_mask));
        const uint32_t a_pass = __reduce_add_sync(kFull, __popc(mask));
        if (lane == 0) {  // dense-equivalent cost: the warp's cycles x the items it evaluated (as K1)
          s_stat[warp][r][0] += a_in;
          s_stat[warp][r][1] += a_pass;
          s_stat[warp][r][2] += static_cast<unsigned long long>(c1 - c0) * a_in;
        }
      }
    }
    // the survivors' rows: bbox (and id when no HASH loaded it) gathered now, before the look-back
    uint64_t bbs[kFItems];
#pragma unroll
    for (int j = 0; j < kFItems; ++j) {
      bbs[j] = 0;
      if ((mask >> j) & 1u) {
        bbs[j] = __ldg(p.bbox + base + p0 + j);
        if (!need_id) ids[j] = __ldg(p.id + base + p0 + j);
      }
    }
    // tile scan: thread -> warp -> tile
    const uint32_t c = __popc(mask);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wcnt[warp] = x;
    __syncthreads();
    uint32_t wexcl = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kRouteThreads / 32; ++w) {
      const uint32_t v = s_wcnt[w];
      wexcl += w < warp ? v : 0u;
      total += v;
    }
    if (warp == 0) {  // decoupled look-back
      if (lane == 0) st_relaxed_u64(f.tile_status + t, (t == 0 ? kLbPrefix : kLbAggregate) | total);
      uint32_t excl = 0;
      if (t > 0) {
        int j = static_cast<int>(t) - 1;
        while (true) {
          const int idx = j - lane;
          unsigned long long v = idx >= 0 ? ld_relaxed_u64(f.tile_status + idx) : kLbPrefix;
          while (__any_sync(kFull, (v & kLbFlags) == 0)) {
            if ((v & kLbFlags) == 0) v = ld_relaxed_u64(f.tile_status + idx);
          }
          const uint32_t pb = __ballot_sync(kFull, (v & kLbFlags) == kLbPrefix);
          if (pb) {
            const int k = __ffs(pb) - 1;  // the nearest predecessor with an inclusive prefix
            excl += __reduce_add_sync(kFull, lane <= k ? static_cast<uint32_t>(v) : 0u);
            break;
          }
          excl += __reduce_add_sync(kFull, static_cast<uint32_t>(v));
          j -= 32;
        }
        if (lane == 0) st_relaxed_u64(f.tile_status + t, kLbPrefix | (excl + total));
      }
      if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    uint32_t pos = emit_off + s_excl + wexcl + (x - c);
    if (mask) {
#pragma unroll
      for (int j = 0; j < kFItems; ++j) {
        if ((mask >> j) & 1u) {
          f.out_ids[pos] = ids[j];
          f.out_bbox[pos] = bbs[j];
          if (f.out_pos) f.out_pos[pos] = base + p0 + j;
          ++pos;
        }
      }
    }
    if (t == ntiles - 1 && tid == 0) *f.emit_count = emit_off + s_excl + total;
    __syncthreads();  // s_tile / s_wcnt / s_excl are rewritten by the next tile
  }
  if (ntiles == 0 && blockIdx.x == 0 && tid == 0) *f.emit_count = emit_off;
  if (p.collect_stats) {
    __syncthreads();
    if (tid < P) {
      unsigned long long in = 0, pass = 0, cs = 0;
#pragma unroll
      for (int w = 0; w < kRouteThreads / 32; ++w) {
        in += s_stat[w][tid][0];
        pass += s_stat[w][tid][1];
        cs += s_stat[w][tid][2];
      }
      const int k = s_pid[tid];
      if (in) {
        atomicAdd(&st->d_in[k], in);
        atomicAdd(&st->d_pass[k], pass);
        atomicAdd(&st->d_cost[k], cs);
        atomicAdd(&st->d_comp[k], in);
      }
    }
  }
}

void hydro_route_emit_launch(const FusedParams& f, int grid, cudaStream_t stream) {
  hydro_route_emit_kernel<<<grid, kRouteThreads, 0, stream>>>(f);
}

int hydro_route_emit_tile() { return kFTile; }

int hydro_route_emit_occupancy() {
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hydro_route_emit_kernel, kRouteThreads, 0);
  return occ < 1 ? 1 : occ;
}

// ------------------------------------------------------------------------------------------
// Verdict cache (reuse-aware routing).  K0 probe: for every predicate with a
// cache, the number of the batch's tuple ids whose verdict is cached ("the router algorithms first
// check the potential cache hit rate for a batch") -> d_hit; K5 mode 8 turns it
// into the batch's hit rates and the order by estimated cost.  put: records given verdicts.
__global__ void __launch_bounds__(kRouteThreads) hydro_probe_kernel(DevState* st, const PredDev* preds,
                                                                    const uint64_t* id, uint32_t base, uint32_t n) {
  __shared__ unsigned long long s_hit[kMaxPred];
  const int P = st->n_pred;
  if (threadIdx.x < kMaxPred) s_hit[threadIdx.x] = 0;
  __syncthreads();
  for (int k = 0; k < P; ++k) {
    const uint32_t* known = preds[k].cache_known;
    if (!known) continue;
    const uint64_t cap = preds[k].cache_cap;
    uint32_t c = 0;
    for (uint32_t i = blockIdx.x * kRouteThreads + threadIdx.x; i < n; i += gridDim.x * kRouteThreads) {
      const uint64_t v = __ldg(id + base + i);
      if (v < cap) c += (__ldg(known + (v >> 5)) >> (v & 31)) & 1u;
    }
    c = __reduce_add_sync(kFull, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_hit[k], static_cast<unsigned long long>(c));
  }
  __syncthreads();
  if (threadIdx.x < P && s_hit[threadIdx.x]) atomicAdd(&st->d_hit[threadIdx.x], s_hit[threadIdx.x]);
}

__global__ void hydro_cache_put_kernel(uint32_t* known, uint32_t* pass, uint64_t cap, const uint64_t* ids,
                                       const uint8_t* verdicts, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t v = ids[i];
    if (v >= cap) continue;
    const uint32_t bit = 1u << (v & 31);
    if (verdicts[i]) atomicOr(pass + (v >> 5), bit);
    else atomicAnd(pass + (v >> 5), ~bit);
    atomicOr(known + (v >> 5), bit);  // after the verdict bit: readers in later kernels see both
  }
}

// ------------------------------------------------------------------------------------------
// K5: fold.

__device__ __forceinline__ double policy_key(int policy, double c, double s, double hit) {
  if (policy == HYDRO_POLICY_COST) return c;
  if (policy == HYDRO_POLICY_SELECTIVITY) return s;
  if (policy == HYDRO_POLICY_REUSE) return (1.0 - hit) * c;  // estimated cost
  if (c == 0.0) return 0.0;                      // R1
  if (s >= 1.0) return __longlong_as_double(0x7FF0000000000000ll);  // +inf (R1)
  return c / (1.0 - s);
}

// keys from st->cost / sel / hit, stable order by (key, id) (R2), positions, hop slots
__device__ void order_by_keys(DevState* st) {
  const int P = st->n_pred;
  for (int k = 0; k < P; ++k) st->key[k] = policy_key(st->policy, st->cost[k], st->sel[k], st->hit[k]);
  if (st->policy != HYDRO_POLICY_FIXED_ORDER) {
    int ord[kMaxPred];
    for (int k = 0; k < P; ++k) ord[k] = k;
    for (int i = 1; i < P; ++i) {  // stable insertion sort by (key, id): R2
      const int v = ord[i];
      int j = i - 1;
      while (j >= 0 && st->key[ord[j]] > st->key[v]) {
        ord[j + 1] = ord[j];
        --j;
      }
      ord[j + 1] = v;
    }
    for (int i = 0; i < P; ++i) st->order[i] = ord[i];
  }
  for (int i = 0; i < P; ++i) st->position[st->order[i]] = i;
  build_sched(st->kind, st->order, P, st->sched, st->pair_a, st->pair_b);
}

// mode: bit 0 = PREP (batch deltas -> batch record + pending), bit 1 = APPLY (deltas -> decayed
// statistics -> keys -> order; from `pending`, or with bit 5 from the exchanged window
// xfer[apply_slot]), bit 2 = RECORD (order used by this batch's chain), bit 3 = REUSE (the batch's
// cache hit rates from the probe counts over n_batch tuples -> keys -> order), bit 4 = SNAPSHOT
// (pending -> xfer[snap_slot], pending cleared: the window the ranks' exchange sums).
// Order inside one launch: REUSE, RECORD, PREP, SNAPSHOT, APPLY.
__global__ void hydro_fold_kernel(DevState* st, BatchRec* rec, int32_t mode, uint32_t n_batch, int32_t snap_slot,
                                  int32_t apply_slot) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int P = st->n_pred;
  if (mode & 8) {
    for (int k = 0; k < P; ++k) {
      st->hit[k] = n_batch > 0 ? static_cast<double>(st->d_hit[k]) / static_cast<double>(n_batch) : 0.0;
      st->d_hit[k] = 0;
    }
    order_by_keys(st);
  }
  if (mode & 4) {
    for (int k = 0; k < kMaxPred; ++k) rec->order_used[k] = k < P ? st->order[k] : -1;
  }
  if (mode & 1) {
    for (int k = 0; k < P; ++k) {
      const unsigned long long di = st->d_in[k], dp = st->d_pass[k], dc = st->d_cost[k], dm = st->d_comp[k];
      rec->d_in[k] += di;
      rec->d_pass[k] += dp;
      rec->d_cost[k] += dc;
      rec->d_comp[k] += dm;
      st->pend[k] += di;
      st->pend[kMaxPred + k] += dp;
      st->pend[2 * kMaxPred + k] += dc;
      st->pend[3 * kMaxPred + k] += dm;
      st->tot_in[k] += di;
      st->tot_pass[k] += dp;
      st->tot_cost[k] += static_cast<double>(dc);
      st->tot_comp[k] += dm;
      st->d_in[k] = st->d_pass[k] = st->d_cost[k] = st->d_comp[k] = 0;
    }
  }
  if (mode & 16) {
    for (int i = 0; i < 4 * kMaxPred; ++i) {
      st->xfer[snap_slot][i] = st->pend[i];
      st->pend[i] = 0;
    }
  }
  if (mode & 2) {
    const double g = st->gamma;
    unsigned long long* src = (mode & 32) ? st->xfer[apply_slot] : st->pend;
    for (int k = 0; k < P; ++k) {
      const unsigned long long di = src[k];
      if (di > 0) {  // R4: fold only observed predicates
        st->s_in[k] = g * st->s_in[k] + static_cast<double>(di);
        st->s_pass[k] = g * st->s_pass[k] + static_cast<double>(src[kMaxPred + k]);
        st->s_cost[k] = g * st->s_cost[k] + static_cast<double>(src[2 * kMaxPred + k]) * st->cost_norm[k];
        st->s_comp[k] = g * st->s_comp[k] + static_cast<double>(src[3 * kMaxPred + k]);
      }
      src[k] = src[kMaxPred + k] = src[2 * kMaxPred + k] = src[3 * kMaxPred + k] = 0;
    }
    for (int k = 0; k < P; ++k) {
      double s, c;
      if (st->policy == HYDRO_POLICY_STATIC) {
        s = st->declared_sel[k];
        c = st->declared_cost[k];
      } else {
        s = st->s_in[k] > 0.0 ? st->s_pass[k] / st->s_in[k] : st->prior;  // PAPER.md:416, R3
        // cost of computing the predicate per evaluated tuple (cache hits excluded,
        // PAPER.md:600); without a cache every routed tuple is evaluated (s_comp == s_in)
        c = (st->cost_source == HYDRO_COST_DECLARED || st->s_comp[k] <= 0.0) ? st->declared_cost[k]
                                                                               : st->s_cost[k] / st->s_comp[k];
      }
      st->sel[k] = s;
      st->cost[k] = c;
    }
    order_by_keys(st);
  }
}

// Router of concurrent workers: worker i is a context
// holding one predicate on its own SM partition.  Its time per tuple is its folded cost (SM-cycles
// per tuple, R6) spread over its SMs, its selectivity the folded one; the workers are ordered by
// the policy key, lowest first, ties by index (R2).  One thread: at most 8 workers.
__global__ void hydro_route_workers_kernel(WorkerRoute w, int32_t* order, double* cost, double* sel) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double key[kMaxPred];
  int ord[kMaxPred];
  for (int k = 0; k < w.n; ++k) {
    const double c = w.st[k]->cost[0] / w.sms[k], s = w.st[k]->sel[0];
    key[k] = policy_key(w.policy, c, s, 0.0);
    cost[k] = c;
    sel[k] = s;
    ord[k] = k;
  }
  for (int i = 1; i < w.n; ++i) {  // stable insertion sort by (key, index)
    const int v = ord[i];
    int j = i - 1;
    while (j >= 0 && key[ord[j]] > key[v]) {
      ord[j + 1] = ord[j];
      --j;
    }
    ord[j + 1] = v;
  }
  for (int i = 0; i < w.n; ++i) order[i] = ord[i];
}

// ------------------------------------------------------------------------------------------
// Weight re-layout: W[rows][K] bf16 row-major (K = 12288: a linear head or MLP layer 1; K = hidden:
// MLP layer 2) -> [K/64 K-blocks][n_pad rows][128 B] with the
// 128-byte swizzle applied (16-byte chunk c of row n stored at chunk c ^ (n & 7)), i.e. the exact
// shared-memory image UMMA reads, so one 1-D bulk copy per stage lands it.  Rows >= C are 0.
// to_fp16 = 1 re-encodes every weight times `scale` (a power of two) as fp16 (identical value) and
// raises *inexact if any scaled weight is not exactly representable in fp16 (the runtime then
// re-tiles as bf16).
// crop_order = 1 (matrices over the 12288 crop features: linear heads, MLP W1) places feature
// crop_pos_feature(g, p) at position p of crop row g, the order K4's converters produce;
// crop_order = 2 uses crop_pos_feature_tm, the order of K4-T (A in tensor memory); crop_order = 3
// crop_pos_feature_area, the order of K4's AREA converter.
__global__ void hydro_tile_weights_kernel(const uint16_t* w, uint8_t* w_tiled, int32_t n_classes, int32_t n_pad,
                                          int32_t k_features, int32_t to_fp16, int32_t crop_order, int32_t* inexact,
                                          float scale) {
  const uint64_t total = static_cast<uint64_t>(k_features / kKBlock) * n_pad * 8;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = static_cast<uint32_t>(i & 7);
    const uint64_t rowi = i >> 3;
    const uint32_t n = static_cast<uint32_t>(rowi % n_pad);
    const uint32_t kb = static_cast<uint32_t>(rowi / n_pad);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (static_cast<int32_t>(n) < n_classes) {
      const uint16_t* wrow = w + static_cast<uint64_t>(n) * k_features;
      if (crop_order) {
        uint16_t e[8];
        const uint32_t g = kb / kKBlocksPerGroup, p0 = (kb % kKBlocksPerGroup) * kKBlock + c * 8;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          e[t] = wrow[crop_order == 3   ? crop_pos_feature_area(g, p0 + t)
                      : crop_order == 2 ? crop_pos_feature_tm(g, p0 + t)
                                        : crop_pos_feature(g, p0 + t)];
        v = make_uint4(e[0] | (static_cast<uint32_t>(e[1]) << 16), e[2] | (static_cast<uint32_t>(e[3]) << 16),
                       e[4] | (static_cast<uint32_t>(e[5]) << 16), e[6] | (static_cast<uint32_t>(e[7]) << 16));
      } else {
        v = *reinterpret_cast<const uint4*>(wrow + kb * kKBlock + c * 8);
      }
      if (to_fp16) {
        uint32_t* u = reinterpret_cast<uint32_t*>(&v);
        int bad = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // (scale: a power of two, so lo and hi stay the weights' exact values times 2^k)
          const float lo = __uint_as_float(u[j] << 16) * scale, hi = __uint_as_float(u[j] & 0xFFFF0000u) * scale;
          const __half hl = __float2half_rn(lo), hh = __float2half_rn(hi);
          bad |= (__half2float(hl) != lo) | (__half2float(hh) != hi);
          u[j] = static_cast<uint32_t>(__half_as_ushort(hl)) | (static_cast<uint32_t>(__half_as_ushort(hh)) << 16);
        }
        if (bad) atomicOr(inexact, 1);
      }
    }
    uint8_t* dst = w_tiled + (static_cast<uint64_t>(kb) * n_pad + n) * 128 + ((c ^ (n & 7)) << 4);
    *reinterpret_cast<uint4*>(dst) = v;
  }
}

// Host-side entry points (the kernel template stays inside this translation unit).
void hydro_route_launch(const RouteParams& r, int grid, cudaStream_t stream, bool compact) {
  if (compact) hydro_route_kernel<true><<<grid, kRouteThreads, 0, stream>>>(r);
  else hydro_route_kernel<false><<<grid, kRouteThreads, 0, stream>>>(r);
}

int hydro_route_occupancy(bool compact) {
  int occ = 1;
  if (compact) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hydro_route_kernel<true>, kRouteThreads, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hydro_route_kernel<false>, kRouteThreads, 0);
  return occ < 1 ? 1 : occ;
}
