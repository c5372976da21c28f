// K4-HSV: DogColorClassifier as the paper implements it (reading R27 in DESIGN.md
// §2): every pixel of the 64x64 nearest-exact crop (R10) -> 8-bit HSV in OpenCV's convention ->
// the colour class whose box contains it (red, black, gray, yellow, green, blue, purple, pink,
// white, else other) -> the class with most pixels (lowest index on ties) == target.
//
// A non-GEMM classifier hop: plain ALU work per pixel, so no tensor cores.  One warp evaluates the
// 32 tuples of one verdict-bitmap word, one tuple at a time: lane l takes output pixels l and
// l + 32 of every crop row (two aligned 32-bit loads from the L1-cached frame row, funnel shift),
// keeps 10 per-lane class counters packed 4 x 8 bits per register (a lane sees <= 128 pixels of a
// tuple), then one warp reduction per class.  HSV is OpenCV's fixed-point conversion (two table
// lookups in shared memory per pixel, no divisions).
#include <algorithm>

#include "hydro_internal.cuh"

using namespace hydro;

namespace {

constexpr int kHsvThreads = 256;
constexpr uint32_t kFullMask = 0xFFFFFFFFu;

// 8-bit HSV class of one RGB pixel (R27): OpenCV's cvtColor(RGB2HSV) fixed-point arithmetic with
// its reciprocal tables (hsv_shift 12; sdiv = round(255 * 2^12 / V), hdiv = round(30 * 2^12 / d),
// in shared memory), then the disjoint class boxes (pinned in tests/test_oracle.py):
//   S = (d sdiv[V] + 2^11) >> 12,  H = (h hdiv[d] + 2^11) >> 12 (+180 if < 0),
//   h = G - B (V = R), B - R + 2d (V = G), R - G + 4d (V = B).
// Branch-free; checked against the oracle (= cv2) on all 2^24 colours
// (tests/test_gpu_parity.py::test_hsv_every_rgb_colour).
__device__ __forceinline__ uint32_t hsv_class_of(uint32_t R, uint32_t G, uint32_t B, const int* sdiv,
                                                 const int* hdiv) {
  const int r = static_cast<int>(R), g = static_cast<int>(G), b = static_cast<int>(B);
  const int V = max(max(r, g), b), d = V - min(min(r, g), b);
  const int sd = d * sdiv[V];  // S <= 18 <=> sd < 19 * 4096 - 2048;  S >= 50 <=> sd >= 50 * 4096 - 2048
  const int hn = (V == r) ? g - b : ((V == g) ? b - r + 2 * d : r - g + 4 * d);
  int H = (hn * hdiv[d] + 2048) >> 12;
  H += H < 0 ? 180 : 0;
  // hue classes of chromatic pixels (S >= 50, V >= 70), picked from a nibble table by the number of
  // hue bounds at or below H: red <= 9 < other <= 19 < yellow <= 34 < green <= 89 < blue <= 128
  // < purple <= 158 < pink <= 169 < red (PAPER.md:395 with the hue wrap)
  const uint32_t ipos = static_cast<uint32_t>(H >= 10) + static_cast<uint32_t>(H >= 20) +
                        static_cast<uint32_t>(H >= 35) + static_cast<uint32_t>(H >= 90) +
                        static_cast<uint32_t>(H >= 129) + static_cast<uint32_t>(H >= 159) +
                        static_cast<uint32_t>(H >= 170);
  const uint32_t hc = (0x07654390u >> (4u * ipos)) & 15u;
  uint32_t cls = (sd >= 50 * 4096 - 2048 && V >= 70) ? hc : 9u;
  cls = sd < 19 * 4096 - 2048 ? (V <= 230 ? 2u : 8u) : cls;  // S <= 18: gray (V 31..230) / white (V 231..255)
  return V <= 30 ? 1u : cls;                                // black: (0,0,0)-(179,255,30)
}

__device__ __forceinline__ uint32_t ldg32(const uint8_t* p) { return __ldg(reinterpret_cast<const uint32_t*>(p)); }

}  // namespace

__global__ void __launch_bounds__(kHsvThreads, 3) hydro_hsv_kernel(ClsParams p) {
  DevState* st = p.st;
  int pred;
  const uint32_t* list_in;
  uint32_t count, base = p.range_base;
  uint32_t* bits_out;
  if (p.dispatch) {
    const int h = st->sched[p.hop];
    if (h < 0 || h >= st->n_pred) return;
    pred = st->order[h];
    if (st->kind[pred] != kHsv) return;
    if (h == 0) {  // the batch: its position range, or the caller's selection
      list_in = p.sel0;
      count = p.sel0 ? *p.sel0_count : p.range_n;
    } else {
      list_in = p.lists + static_cast<uint64_t>(h) * p.list_stride;
      count = p.counts[h];
    }
    bits_out = p.bits + static_cast<uint64_t>(h) * p.bits_stride;
  } else {
    pred = p.explicit_pred;
    list_in = p.list_in;
    count = list_in ? *p.count_in : p.range_n;
    bits_out = p.bits_out;
  }
  const uint32_t* ind = cls_redirect(p, p.preds[pred], list_in, count);  // cached hop: uncached tuples
  const bool fill = p.preds[pred].cache_known && (p.preds[pred].cache_fill || p.force_fill);
  // OpenCV's reciprocal tables (exact integer rounding; no .5 ties occur for i < 2^13)
  __shared__ int s_sdiv[256], s_hdiv[256];
  for (int i = threadIdx.x; i < 256; i += kHsvThreads) {
    s_sdiv[i] = i ? (2 * (255 << 12) + i) / (2 * i) : 0;
    s_hdiv[i] = i ? (2 * (30 << 12) + i) / (2 * i) : 0;
  }
  if (threadIdx.x == 0) ktimer_begin(st, 5);
  __syncthreads();
  const int target = p.preds[pred].target;
  const int lane = threadIdx.x & 31;
  const uint32_t words = (count + 31) / 32;
  const uint32_t pitch = static_cast<uint32_t>(p.frame_w * 3);
  uint32_t n_in = 0, n_pass = 0;
  unsigned long long cyc = 0;
  for (uint32_t wi = (blockIdx.x * kHsvThreads + threadIdx.x) / 32; wi < words;
       wi += (gridDim.x * kHsvThreads) / 32) {
    const long long t0 = clock64();
    // metadata of the word's 32 tuples: lane i loads tuple 32 wi + i
    const uint32_t pos_l = wi * 32 + lane;
    const bool valid_l = pos_l < count;
    uint32_t fid = 0, x0 = 0, y0 = 0, w = 1, hh = 1;
    if (valid_l) {
      const uint32_t idx = list_in ? __ldg(list_in + pos_l) : base + pos_l;
      fid = min(__ldg(p.frame_id + idx), static_cast<uint32_t>(p.n_frames - 1));
      const uint64_t bb = __ldg(p.bbox + idx);
      int bx0 = static_cast<int>(bb & 0xFFFF), by0 = static_cast<int>((bb >> 16) & 0xFFFF);
      int bx1 = static_cast<int>((bb >> 32) & 0xFFFF), by1 = static_cast<int>((bb >> 48) & 0xFFFF);
      bx0 = min(bx0, p.frame_w - 1);  // clamp: no-op for valid tuples, memory safety otherwise
      by0 = min(by0, p.frame_h - 1);
      bx1 = max(min(bx1, p.frame_w), bx0 + 1);
      by1 = max(min(by1, p.frame_h), by0 + 1);
      x0 = static_cast<uint32_t>(bx0);
      y0 = static_cast<uint32_t>(by0);
      w = static_cast<uint32_t>(bx1 - bx0);
      hh = static_cast<uint32_t>(by1 - by0);
    }
    const uint32_t bvalid = __ballot_sync(kFullMask, valid_l);
    uint32_t vbits = 0;
    for (int i = 0; i < 32; ++i) {
      if (!((bvalid >> i) & 1u)) break;  // valid positions are a prefix of the word
      const uint32_t tf = __shfl_sync(kFullMask, fid, i), tx = __shfl_sync(kFullMask, x0, i);
      const uint32_t ty = __shfl_sync(kFullMask, y0, i), tw = __shfl_sync(kFullMask, w, i);
      const uint32_t th = __shfl_sync(kFullMask, hh, i);
      const uint8_t* frame = p.frames + static_cast<uint64_t>(tf) * p.frame_h * pitch;
      // byte offsets of this lane's two output columns dx = lane, lane + 32 (nearest-exact, R10)
      const uint32_t o0 = 3u * (tx + (((2u * lane + 1u) * tw) >> 7));
      const uint32_t o1 = 3u * (tx + (((2u * (lane + 32u) + 1u) * tw) >> 7));
      uint32_t c0 = 0, c1 = 0, c2 = 0;  // class counters, 4 x 8 bits per register
      constexpr int kRows = 8;           // crop rows in flight per step (16 pixel loads issued first)
      for (int dy0 = 0; dy0 < 64; dy0 += kRows) {
        uint32_t px[kRows][2];
#pragma unroll
        for (int rr = 0; rr < kRows; ++rr) {
          const uint8_t* row = frame + (ty + (((2u * (dy0 + rr) + 1u) * th) >> 7)) * pitch;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const uint32_t o = k ? o1 : o0;
            const uint32_t a = o & ~3u;
            const uint32_t hi = (o & 3u) > 1u ? ldg32(row + a + 4) : 0u;  // only if the pixel straddles
            px[rr][k] = __funnelshift_r(ldg32(row + a), hi, o << 3);
          }
        }
#pragma unroll
        for (int rr = 0; rr < kRows; ++rr) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const uint32_t q = px[rr][k];
            const uint32_t cls = hsv_class_of(q & 0xFF, (q >> 8) & 0xFF, (q >> 16) & 0xFF, s_sdiv, s_hdiv);
            const uint32_t inc = 1u << ((cls & 3u) * 8u);
            c0 += cls < 4 ? inc : 0u;
            c1 += (cls >= 4 && cls < 8) ? inc : 0u;
            c2 += cls >= 8 ? inc : 0u;
          }
        }
      }
      int best = -1, bc = 0;
#pragma unroll
      for (int c = 0; c < 10; ++c) {
        const uint32_t reg = c < 4 ? c0 : (c < 8 ? c1 : c2);
        const int v = static_cast<int>(__reduce_add_sync(kFullMask, (reg >> ((c & 3) * 8)) & 0xFFu));
        if (v > best) {  // strict: lowest class index wins ties
          best = v;
          bc = c;
        }
        if (p.dbg_logits && lane == 0) p.dbg_logits[static_cast<uint64_t>(wi * 32 + i) * 10 + c] = static_cast<float>(v);
      }
      if (bc == target) vbits |= 1u << i;
    }
    cls_emit(p, bits_out, ind, list_in, base, wi * 32, pos_l, valid_l, (vbits >> lane) & 1u, p.preds[pred], fill);
    if (p.dbg_verdict && valid_l) p.dbg_verdict[pos_l] = (vbits >> lane) & 1u;
    n_in += __popc(bvalid);
    n_pass += __popc(vbits);
    // dense-equivalent warp cycles (R6): charged in proportion to the word's occupancy
    cyc += static_cast<unsigned long long>(clock64() - t0) * __popc(bvalid) / 32u;
  }
  if (p.collect_stats && lane == 0 && n_in) {
    atomicAdd(&st->d_in[pred], static_cast<unsigned long long>(n_in));
    atomicAdd(&st->d_pass[pred], static_cast<unsigned long long>(n_pass));
    atomicAdd(&st->d_comp[pred], static_cast<unsigned long long>(n_in));
    atomicAdd(&st->d_cost[pred], cyc);
  }
  if (lane == 0 && n_in) atomicAdd(&st->kt_items[5], static_cast<unsigned long long>(n_in));
  __syncthreads();
  if (threadIdx.x == 0) ktimer_end(st, 5);
}

void hydro_hsv_launch(const ClsParams& c, uint64_t max_positions, int num_sms, cudaStream_t stream) {
  const uint64_t warps = (max_positions + 31) / 32;
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, static_cast<uint64_t>(num_sms) * 8));
  hydro_hsv_kernel<<<static_cast<int>(blocks), kHsvThreads, 0, stream>>>(c);
}

int hydro_hsv_warps_per_sm() {
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hydro_hsv_kernel, kHsvThreads, 0);
  return std::max(occ, 1) * (kHsvThreads / 32);
}
