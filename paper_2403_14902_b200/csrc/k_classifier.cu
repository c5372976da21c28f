// K4: fused Crop(frame, bbox) -> 64x64 resize gather -> linear-head GEMM on tcgen05 tensor cores
// -> argmax verdict (readings R10-R14, R19 in DESIGN.md §2).
//
// One persistent CTA per SM walks M-tiles of 128 alive tuples.  The K = 12288 features of a tile
// are streamed as 64 crop rows ("groups") of 3 UMMA K-blocks (64 elements = 128 B per row).
// Warp roles:
//   warps 0-3  epilogue: tcgen05.ld the fp32 accumulator (TMEM lane = tuple), + bias, argmax,
//              verdict ballot -> bitmap, pass counters
//   warp  4    loader: 1-D bulk copies (TMA engine) of the pre-swizzled weight K-blocks into the B
//              ring; L2 prefetch of the crop-row segments a few groups ahead
//   warp  5    MMA: TMEM alloc; one thread issues tcgen05.mma (M=128, N=n_pad, K=16) x 4 per
//              K-block, tcgen05.commit releases A / B stages and publishes finished tiles
//   warps 6-13 converters: stage each tuple's source row segment [3*x0 & ~15, roundup16(3*x1))
//              of frame row sy = y0 + ((2dy+1)h)>>7 into shared memory with coalesced 16-byte
//              cp.async (two 4-row quads ahead); then 8 lanes x 8 output pixels per crop row
//              (lane j: pixels j + 8k, the interleaved K order of crop_pos_feature), 4 rows per
//              warp instruction; nearest-exact pixel selection sx = x0 + ((2dx+1)w)>>7,
//              exact u8 -> fp16 (PRMT 0x64vv = 1024+v, HSUB2 1024) or bf16, st.shared into the
//              128B-swizzled K-major A ring (conflict-free), fence.proxy.async, arrive.
// The A operand never touches HBM: only the crop-row segments of the frames are read.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "hydro_internal.cuh"

using namespace hydro;

namespace {

#ifdef HYDRO_2CTA
constexpr int kPair = 2;  // CTA pairs (cta_group::2, M=256): each CTA holds half of every weight K-block
#else
constexpr int kPair = 1;
#endif
#ifdef HYDRO_PAIR_SMALL_B
static_assert(kPair == 2, "HYDRO_PAIR_SMALL_B needs HYDRO_2CTA");
constexpr int kBStages = kBRing;  // pair mode: half-size stages, half the B-ring bytes (freed for staging)
#else
constexpr int kBStages = kBRing * kPair;  // same B-ring bytes; half-size stages in pair mode
#endif

#ifndef HYDRO_AREA_WARPS
#define HYDRO_AREA_WARPS 20
#endif
constexpr int kMaxCW = HYDRO_AREA_WARPS > kConvWarps ? HYDRO_AREA_WARPS : kConvWarps;
struct ClsCtrl {
  uint64_t full_a[kARing], empty_a[kARing];
  uint64_t full_b[kBStages], empty_b[kBStages];
  uint64_t tfull[2], tempty[2];
  uint64_t hready, tfull2;  // MLP: hidden layer written back to TMEM / second GEMM done
  uint64_t astg[kMaxCW][8];      // AREA converter: staged items landed (bulk copies, complete_tx)
  float area_rcp[32];            // AREA converter: RN(1 / n) for bin pixel counts n <= 25
  uint32_t area_cost[kTileM];    // data-aware AREA tiles: estimated converter work of each tile row
  uint8_t area_perm[kMaxCW * 16];  // tile rows of converter warp c = area_perm[16c .. 16c+15] (0xFF: none)
  uint32_t tmem_base;
  uint32_t pad;
  float bias[HYDRO_MAX_CLASSES];
  float bias1[HYDRO_MLP_HIDDEN_MAX];  // MLP: b1
};

// worst-case carve-up of both classifier kernels: [A ring][B ring (3 x 16 KB)][ctrl][staging]
static_assert(1023 + kARing * kAKBlockBytes + 3 * 16384 + sizeof(ClsCtrl) + 15 +
                      kConvWarps * kQuadSlots * kQuadSlotBytes <= kClsSmemBytes,
              "classifier shared memory exceeds 227 KB");

__device__ __forceinline__ uint32_t bf16_bits_of_byte(uint32_t b) {
  // exact: the float 2^23 + b minus 2^23 is b; its top 16 bits are the bf16 of b (b < 256)
  const float f = __uint_as_float(0x4B000000u | b) - 8388608.0f;
  return __float_as_uint(f) >> 16;
}

__device__ __forceinline__ uint32_t f16x2_sub(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ uint32_t bf16x2_of_bytes(uint32_t lo, uint32_t hi) {
  const float flo = __uint_as_float(0x4B000000u | lo) - 8388608.0f;
  const float fhi = __uint_as_float(0x4B000000u | hi) - 8388608.0f;
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(fhi), "f"(flo));
  return d;
}

__device__ __forceinline__ uint32_t ldg32(const uint8_t* p) { return __ldg(reinterpret_cast<const uint32_t*>(p)); }

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
#ifdef HYDRO_PRED_LDS
// predicated load: lanes with !pred issue no shared-memory access (and cause no bank conflict)
__device__ __forceinline__ uint32_t lds32_if(uint32_t addr, bool pred) {
  uint32_t v = 0;
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.shared.b32 %0, [%1];\n}"
               : "+r"(v) : "r"(addr), "r"(static_cast<uint32_t>(pred)));
  return v;
}
#endif
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

struct RowMeta {  // per alive tuple of the tile
  uint32_t row16;    // offset of (frame, y0, 0) in the frame pool, in 16-byte units (pools < 64 GiB)
  uint32_t seg_lo;   // 16-byte aligned start of the crop's byte span inside a frame row
  uint32_t seg_len;  // bytes to stage per crop row (multiple of 16), 0 when invalid
  int32_t x0, w, h;
  int32_t valid;
};

// frame-pool address of a 16-byte-unit offset (64-bit: the pool may exceed 4 GiB)
__device__ __forceinline__ const uint8_t* at16(const uint8_t* frames, uint32_t off16) {
  return frames + (static_cast<uint64_t>(off16) << 4);
}

__device__ __forceinline__ RowMeta load_meta(const ClsParams& p, const uint32_t* list_in, uint32_t base,
                                             uint32_t pos, uint32_t count) {
  RowMeta m{};
  m.valid = pos < count;
  if (!m.valid) return m;
  const uint32_t idx = list_in ? __ldg(list_in + pos) : base + pos;
  uint32_t fid = __ldg(p.frame_id + idx);
  const uint64_t bb = __ldg(p.bbox + idx);
  fid = min(fid, static_cast<uint32_t>(p.n_frames - 1));
  int x0 = static_cast<int>(bb & 0xFFFF), y0 = static_cast<int>((bb >> 16) & 0xFFFF);
  int x1 = static_cast<int>((bb >> 32) & 0xFFFF), y1 = static_cast<int>((bb >> 48) & 0xFFFF);
  // clamp to the frame (no-op for valid tuples; keeps device-side inputs memory-safe)
  x0 = min(x0, p.frame_w - 1);
  y0 = min(y0, p.frame_h - 1);
  x1 = max(min(x1, p.frame_w), x0 + 1);
  y1 = max(min(y1, p.frame_h), y0 + 1);
  const uint32_t pitch = static_cast<uint32_t>(p.frame_w * 3);
  // (the frame row pitch 3 * frame_w is a multiple of 48, so every row starts on 16 bytes)
  m.row16 = static_cast<uint32_t>((static_cast<uint64_t>(fid) * static_cast<uint32_t>(p.frame_h) * pitch +
                                   static_cast<uint64_t>(y0) * pitch) >> 4);
  m.seg_lo = (3u * x0) & ~15u;
  m.seg_len = ((3u * x1 + 15u) & ~15u) - m.seg_lo;  // frame_w % 16 == 0 keeps this inside the row
  m.x0 = x0;
  m.w = x1 - x0;
  m.h = y1 - y0;
  return m;
}

// Which M-tiles of the hop a CTA walks.  Round-robin (the default): unit u of the
// CTA is tile u * kP + crank, units first, first + step, ...  Data-aware (
// HYDRO_BALANCE_DATA_AWARE, AREA heads): the CTA owns the contiguous position range [lo, lim)
// whose estimated cost (sum of input sizes w*h) K6 made equal across CTAs; its units are the
// 128-position tiles lo + 128u (the last one ragged).  Every position range start is a multiple
// of 32, so each verdict word has exactly one writer.
struct TileWalk {
  uint32_t first, step, end;  // units
  uint32_t lo, lim;           // positions >= lim are invalid
  uint32_t kp, crank;
  bool bal;   // K6 position ranges (data-aware, few tiles per CTA)
  bool wbal;  // data-aware: rows dealt to the converter warps by estimated work
  __device__ __forceinline__ uint32_t pos0(uint32_t unit) const {
    return bal ? lo + unit * static_cast<uint32_t>(kTileM) : (unit * kp + crank) * static_cast<uint32_t>(kTileM);
  }
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
// 16-byte cp.async at [dst + kOff] <- [src + kOff] when p (no branch; the offset is an immediate)
template <int kOff>
__device__ __forceinline__ void cp_async16_if(uint32_t dst, const void* src, bool p) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.cg.shared.global [%0+%3], [%1+%3], 16;\n}" ::"r"(dst),
      "l"(src), "r"(static_cast<int>(p)), "n"(kOff)
      : "memory");
}
// one crop-row segment of nch 16-byte chunks: lane j copies chunks j + 8c (c < 7)
__device__ __forceinline__ void stage_segment(uint32_t dst, const uint8_t* row, uint32_t j, uint32_t nch) {
  const uint32_t d = dst + 16u * j;
  const uint8_t* s = row + 16u * j;
  const int rem = static_cast<int>(nch) - static_cast<int>(j);
  cp_async16_if<0>(d, s, rem > 0);
  cp_async16_if<128>(d, s, rem > 8);
  cp_async16_if<256>(d, s, rem > 16);
  cp_async16_if<384>(d, s, rem > 24);
  cp_async16_if<512>(d, s, rem > 32);
  cp_async16_if<640>(d, s, rem > 40);
  cp_async16_if<768>(d, s, rem > 48);
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// per-thread L2 prefetch of one line (a regular LSU op: unlike the uniform-datapath
// cp.async.bulk.prefetch it does not serialise across the lanes of a warp)
__device__ __forceinline__ void prefetch_line_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// ---- CTA-pair (cta_group::2) helpers: the two CTAs of a cluster share one M=256 MMA stream

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
#ifdef HYDRO_SPINWAIT
#define HYDRO_PIPE_WAIT mbar_wait
#else
#define HYDRO_PIPE_WAIT mbar_wait_backoff<64>  // producer / MMA waits poll with a short sleep
#endif
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same shared-memory offset in the leader CTA (rank 0)
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit to the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]^T, CTA pair (the MLP's second layer reads the bf16 hidden
// activations straight from tensor memory: lane = tuple, 32-bit column j = elements 2j, 2j+1)
__device__ __forceinline__ void tc_mma_pair_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_st_32x32b_x8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s_u32(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

}  // namespace

// RN(a / b) for an AREA bin sum a and its pixel count b, given y = RN(1 / b): one Markstein
// correction step after a * y (checked equal to the IEEE quotient for every a <= 2^18, b <= 1100 by
// tools/check_area_div.c, run in tests/test_oracle.py); the reciprocal is shared by a bin's channels
__device__ __forceinline__ float area_div(float a, float b, float y) {
  const float q = __fmul_rn(a, y);
  return __fmaf_rn(__fmaf_rn(-q, b, a), y, q);
}

// One quad (4 crop rows x 8 lanes) of output pixels: lane (r, j) produces pixels j + 8k (k = 0..7,
// the interleaved K order of crop_pos_feature) of row m from its staged segment `seg` (smem
// address).  po[q] packs the byte offsets (relative to the segment) of pixels j+16q and j+16q+8.  Branch-free: both words around a pixel are always
// read (the slots carry slack), the funnel shift uses the wrap mode (shift = 8*o mod 32).
template <bool kFp16, bool kDbg>
__device__ __forceinline__ void convert_quad(uint32_t seg, const uint32_t (&po)[4], uint32_t row_base, uint32_t j,
                                             uint32_t m, uint16_t* dbg) {
  uint32_t px[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const uint32_t o = h2 ? (po[q] >> 16) : (po[q] & 0xFFFFu);
      const uint32_t a = (seg + o) & ~3u;
      const uint32_t w0 = lds32(a);
#ifdef HYDRO_PRED_LDS
      const uint32_t w1 = lds32_if(a + 4, (o & 3u) > 1u);  // only when the 3 bytes straddle words
#else
      const uint32_t w1 = lds32(a + 4);
#endif
      px[2 * q + h2] = __funnelshift_r(w0, w1, o << 3);
    }
  }
  uint32_t e[12];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t p0 = px[2 * q], p1 = px[2 * q + 1];
    if (kFp16) {
      const uint32_t K = 0x64646464u;  // fp16 0x64vv == 1024 + v exactly
      e[3 * q + 0] = f16x2_sub(__byte_perm(p0, K, 0x4140), 0x64006400u);
      e[3 * q + 1] = f16x2_sub(__byte_perm(__byte_perm(p0, p1, 0x0042), K, 0x4140), 0x64006400u);
      e[3 * q + 2] = f16x2_sub(__byte_perm(p1, K, 0x4241), 0x64006400u);
    } else {
      e[3 * q + 0] = bf16x2_of_bytes(p0 & 0xFF, (p0 >> 8) & 0xFF);
      e[3 * q + 1] = bf16x2_of_bytes((p0 >> 16) & 0xFF, p1 & 0xFF);
      e[3 * q + 2] = bf16x2_of_bytes((p1 >> 8) & 0xFF, (p1 >> 16) & 0xFF);
    }
  }
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const uint32_t c = 3u * j + t;  // 16-byte chunk of the 192-element crop row
    const uint32_t addr = row_base + (c >> 3) * kAKBlockBytes + (((c & 7u) ^ (m & 7u)) << 4);
    sts128(addr, e[4 * t], e[4 * t + 1], e[4 * t + 2], e[4 * t + 3]);
  }
  if (kDbg && dbg) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      dbg[24 * kk + 0] = static_cast<uint16_t>(bf16_bits_of_byte(px[kk] & 0xFF));  // pixel j + 8kk
      dbg[24 * kk + 1] = static_cast<uint16_t>(bf16_bits_of_byte((px[kk] >> 8) & 0xFF));
      dbg[24 * kk + 2] = static_cast<uint16_t>(bf16_bits_of_byte((px[kk] >> 16) & 0xFF));
    }
  }
}


// AREA crop (R10, cfg4): output pixel (dy, dx) is the mean over the bin
// [y0 + dy*h//64, y0 + ceil((dy+1)h/64)) x [x0 + dx*w//64, x0 + ceil((dx+1)w/64)), one IEEE f32
// division then bf16 round-to-nearest-even; the bf16 value is staged exactly (fp16 or bf16).
// Bins are read straight from global memory (L1-cached); used for tiles holding a crop wider than
// a staging slot.  Lane (r, j) makes the 8 pixels of positions 24j .. 24j+23 of the AREA K order
// (crop_pos_feature_area): pixel k is dx = 4j + k/2 + 32 (k % 2).  dbg: the crop row's features.
template <bool kFp16, bool kDbg>
__device__ __forceinline__ void convert_quad_area(const uint8_t* frames, uint32_t row0, uint32_t h, uint32_t x0,
                                                  uint32_t w, uint32_t pitch, uint32_t g, uint32_t row_base,
                                                  uint32_t j, uint32_t m, uint16_t* dbg) {
  const uint32_t ys = (g * h) >> 6, ye = ((g + 1u) * h + 63u) >> 6;
  uint32_t xs[8], bw[8], bwmax = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t dx = 4u * j + (k >> 1) + 32u * (k & 1);
    xs[k] = x0 + ((dx * w) >> 6);
    bw[k] = x0 + (((dx + 1u) * w + 63u) >> 6) - xs[k];
    bwmax = max(bwmax, bw[k]);
  }
  uint32_t s[8][3];
#pragma unroll
  for (int k = 0; k < 8; ++k) s[k][0] = s[k][1] = s[k][2] = 0u;
  // Bin row y, bin column t: the loads of all 8 bins are issued before any is summed (16
  // independent L1/L2 requests in flight per lane instead of one dependent chain per pixel).
  for (uint32_t y = ys; y < ye; ++y) {
    const uint8_t* rp = frames + row0 + y * pitch;
    for (uint32_t t = 0; t < bwmax; ++t) {
      uint32_t w0[8], w1[8], sh[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const bool on = t < bw[k];
        const uint32_t o = 3u * (xs[k] + t);
        sh[k] = on ? o << 3 : 0u;
        w0[k] = on ? ldg32(rp + (o & ~3u)) : 0u;
        w1[k] = (on && (o & 3u) > 1u) ? ldg32(rp + (o & ~3u) + 4) : 0u;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t pxl = __funnelshift_r(w0[k], w1[k], sh[k]);
        s[k][0] += pxl & 0xFFu;
        s[k][1] += (pxl >> 8) & 0xFFu;
        s[k][2] += (pxl >> 16) & 0xFFu;
      }
    }
  }
  uint32_t half[24];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float cnt = static_cast<float>(max((ye - ys) * bw[k], 1u));
    const float rcp = __frcp_rn(cnt);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const __nv_bfloat16 b = __float2bfloat16_rn(area_div(static_cast<float>(s[k][ch]), cnt, rcp));
      const uint32_t bbits = __bfloat16_as_ushort(b);
      half[3 * k + ch] = kFp16 ? static_cast<uint32_t>(__half_as_ushort(__float2half_rn(__bfloat162float(b)))) : bbits;
      if (kDbg && dbg) dbg[3u * (4u * j + (k >> 1) + 32u * (k & 1)) + ch] = static_cast<uint16_t>(bbits);
    }
  }
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const uint32_t c = 3u * j + t;
    const uint32_t addr = row_base + (c >> 3) * kAKBlockBytes + (((c & 7u) ^ (m & 7u)) << 4);
    sts128(addr, half[8 * t] | (half[8 * t + 1] << 16), half[8 * t + 2] | (half[8 * t + 3] << 16),
           half[8 * t + 4] | (half[8 * t + 5] << 16), half[8 * t + 6] | (half[8 * t + 7] << 16));
  }
}

// Wide-crop staging: lane j of a row copies the words around its 8 sampled pixels k = 8j .. 8j+7
// to slot bytes [8k, 8k + 8) (the second word only when the pixel straddles it, so nothing past the
// crop row is read).  Out of line: it must not cost the common path registers.
__device__ __noinline__ void stage_wide_row(uint32_t dst, const uint8_t* row, uint32_t xw, uint32_t j) {
  const uint32_t x0 = xw & 0xFFFFu, w = xw >> 16;
  const uint8_t* base_row = row - ((3u * x0) & ~15u);  // frame row start (row = start + seg_lo)
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const uint32_t dx = 8u * j + t;
    const uint32_t b = 3u * (x0 + (((2u * dx + 1u) * w) >> 7));
    cp_async4(dst + 8u * dx, base_row + (b & ~3u));
    if ((b & 3u) > 1u) cp_async4(dst + 8u * dx + 4u, base_row + (b & ~3u) + 4u);
  }
}

// One M-tile of a converter warp: 64 K-groups (crop rows) of its 16 tuples (see converter_role).
// A crop wider than a staging slot (w > 255 px) is staged as a gather instead of its contiguous
// segment: for each of the 64 sampled pixels the two words around it (2 x 4-byte cp.async) go to
// slot bytes [8k, 8k + 8), and its pixel offsets become 8k + (byte-in-word), so the conversion
// itself is unchanged.
template <bool kDbg, bool kArea, int kP, int kQD, bool kWide>
__device__ __forceinline__ void convert_tile(const ClsParams& p, ClsCtrl* ctrl, const uint32_t* list_in, uint32_t lim,
                                             uint32_t pos0, uint32_t crank, int cu, int lane, uint32_t slots, uint32_t a_ring,
                                             uint32_t row_pitch, bool area, bool fp16, const RowMeta& mm,
                                             uint32_t my_row, uint32_t& gg) {
  constexpr int kQS = kQD + 1;
  const int r = lane >> 3, j = lane & 7;
  const uint8_t* frames = p.frames;
  const uint32_t my_src = mm.row16 + (mm.seg_lo >> 4);         // 16-byte units; + sy * pitch per crop row
  const bool my_wide = kWide && lane < 16 && mm.valid && mm.seg_len > static_cast<uint32_t>(kMaxSegBytes);
  // staged bytes per crop row: the segment, or (wide rows) a negative marker for the gather
  const uint32_t my_len = (lane < 16 && mm.valid) ? (my_wide ? 0xFFFFFFFFu : mm.seg_len) : 0u;
  const uint32_t my_h = static_cast<uint32_t>(mm.h);
  const uint32_t my_xw = kWide ? static_cast<uint32_t>(mm.x0) | (static_cast<uint32_t>(mm.w) << 16) : 0u;
  uint32_t po[4][4];
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int src = 4 * it + r;
    const uint32_t x0 = __shfl_sync(0xFFFFFFFFu, static_cast<uint32_t>(mm.x0), src);
    const uint32_t w = __shfl_sync(0xFFFFFFFFu, static_cast<uint32_t>(mm.w), src);
    const uint32_t slo = __shfl_sync(0xFFFFFFFFu, mm.seg_lo, src);
    const bool wide = kWide && __shfl_sync(0xFFFFFFFFu, my_wide, src);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t dx0 = j + 16u * q, dx1 = dx0 + 8u;  // pixels k = 2q, 2q+1 of lane j
      const uint32_t b0 = 3u * (x0 + (((2u * dx0 + 1u) * w) >> 7)), b1 = 3u * (x0 + (((2u * dx1 + 1u) * w) >> 7));
      const uint32_t o0 = wide ? 8u * dx0 + (b0 & 3u) : b0 - slo;
      const uint32_t o1 = wide ? 8u * dx1 + (b1 & 3u) : b1 - slo;
      po[it][q] = o0 | (o1 << 16);
    }
  }
  // Stage quad k = 4*g + it (rows 4*it .. 4*it+3 of this warp, crop row g) into slot k % kQS:
  // lanes 8r .. 8r+7 copy row r's segment in 16-byte chunks j + 8c (c < 7: segments <= 784 B).
  auto stage_quad = [&](int k, uint32_t slot) {
    if (!area && k < kGroups * 4) {
      const int g = k >> 2, it = k & 3;
      const int src_lane = 4 * it + r;
      const uint32_t len = __shfl_sync(0xFFFFFFFFu, my_len, src_lane);
      const uint32_t off = __shfl_sync(0xFFFFFFFFu, my_src, src_lane);
      const uint32_t h = __shfl_sync(0xFFFFFFFFu, my_h, src_lane);
      const uint32_t xw = kWide ? __shfl_sync(0xFFFFFFFFu, my_xw, src_lane) : 0u;  // (all lanes: before the branch)
      const uint8_t* row = at16(frames, off) + (((2u * g + 1u) * h) >> 7) * row_pitch;
      const uint32_t dst = slots + slot * kQuadSlotBytes + r * kSegPitch;
      if (!kWide || len != 0xFFFFFFFFu) {
        stage_segment(dst, row, j, len >> 4);
      } else {  // wide crop (rare): gather this lane's 8 sampled pixels
        stage_wide_row(dst, row, xw, j);
      }
    }
    cp_async_commit();  // one group per quad (possibly empty) keeps wait_group counting uniform
  };
  uint32_t slot_stage = 0, slot_use = 0;
#pragma unroll
  for (int k = 0; k < kQD; ++k) {
    stage_quad(k, slot_stage);
    slot_stage = slot_stage + 1 == kQS ? 0 : slot_stage + 1;
  }
  for (int g = 0; g < kGroups; ++g, ++gg) {
    const uint32_t set = (gg & 1u) * kKBlocksPerGroup, aph = (gg >> 1) & 1u;
#pragma unroll
    for (int kbr = 0; kbr < kKBlocksPerGroup; ++kbr) mbar_wait(&ctrl->empty_a[set + kbr], aph ^ 1u);
    const uint32_t a_set = a_ring + set * kAKBlockBytes;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      stage_quad(4 * g + it + kQD, slot_stage);
      slot_stage = slot_stage + 1 == kQS ? 0 : slot_stage + 1;
      cp_async_wait<kQD>();  // this thread's copies of quad k have landed
      __syncwarp();                 // ... and every lane's
      // rows past the tile's count convert stale bytes into A rows whose results are masked
      const uint32_t m = __shfl_sync(0xFFFFFFFFu, my_row, 4 * it + r);  // tile row of this lane's tuple
      const bool row_ok = m < static_cast<uint32_t>(kTileM);          // (a slot without a row: nothing to store)
      const uint32_t seg = slots + slot_use * kQuadSlotBytes + r * kSegPitch;
      const uint32_t row_base = a_set + (m >> 3) * 1024u + (m & 7u) * 128u;
      uint16_t* dbg = (kDbg && p.dbg_crops && pos0 + m < lim)
                          ? p.dbg_crops + static_cast<uint64_t>(pos0 + m) * kFeatures + g * 192 + 3 * j
                          : nullptr;
      uint32_t ar0 = 0, ah = 0, ax0 = 0, aw = 0;
      if (kArea && area) {  // (all lanes shuffle before the per-row branch below)
        const int src_lane = 4 * it + r;
        ar0 = __shfl_sync(0xFFFFFFFFu, mm.row16, src_lane);
        ah = __shfl_sync(0xFFFFFFFFu, static_cast<uint32_t>(mm.h), src_lane);
        ax0 = __shfl_sync(0xFFFFFFFFu, static_cast<uint32_t>(mm.x0), src_lane);
        aw = __shfl_sync(0xFFFFFFFFu, static_cast<uint32_t>(mm.w), src_lane);
      }
      if (!row_ok) {
      } else if (kArea && area) {
        uint16_t* dbg_row = dbg ? dbg - 3 * j : nullptr;  // (AREA K order: the crop row's features)
        if (fp16) convert_quad_area<true, kDbg>(at16(frames, ar0), 0u, ah, ax0, aw, row_pitch, g, row_base, j, m, dbg_row);
        else convert_quad_area<false, kDbg>(at16(frames, ar0), 0u, ah, ax0, aw, row_pitch, g, row_base, j, m, dbg_row);
      } else {
        if (fp16) convert_quad<true, kDbg>(seg, po[it], row_base, j, m, dbg);
        else convert_quad<false, kDbg>(seg, po[it], row_base, j, m, dbg);
      }
      slot_use = slot_use + 1 == kQS ? 0 : slot_use + 1;
      __syncwarp();  // the slot is refilled kQD quads later
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int kbr = 0; kbr < kKBlocksPerGroup; ++kbr) {
        if (kP == 2 && crank != 0) mbar_arrive_leader(&ctrl->full_a[set + kbr]);
        else mbar_arrive(&ctrl->full_a[set + kbr]);
      }
    }
  }
  cp_async_wait<0>();
}

// AREA crops, row-cooperative (R10, cfg4): the converter warp makes ONE tuple's crop
// row at a time.  An "item" (crop row g, tuple t of the warp's 16) is the tuple's row segment in its
// bin rows ys .. ye-1 (ys = g*h/64, ye = ceil((g+1)h/64), at most 5 rows): one 1-D bulk copy (TMA
// engine) per source row into a per-warp byte ring, packed back to back, completion on the item's
// mbarrier (8 in flight).  Then
//   vertical:   lane l sums the 16-byte chunks l, l + 32 of the item's rows bytewise (u16 halves:
//               <= 5 x 255) and stores them as V[b] (u16 per segment byte) in the warp's scratch;
//   horizontal: lane q makes output pixels q and q + 32: each channel's bin sum is the sum of V over
//               the bin's columns (<= 5 terms; the 3 channels of a column from two aligned words),
//               then one f32 RN division (area_div with y = RN(1/count) from a table), bf16 RNE, and
//               the 6 features go to the tuple's A row as 3 words at positions 6q .. 6q+5
//               (crop_pos_feature_area).
// Per source pixel the warp issues one shared load per 16 bytes (instead of 2 per pixel per bin),
// and every lane works on the same tuple (no divergence between bin widths of different tuples).
// Crops wider or taller than 256 px take the global-load converter (converter_role).
constexpr int kAreaQ = 8;                                   // items in flight per converter warp
constexpr uint32_t kAreaFixedCost = 12288;  // data-aware warp balance: per-tuple fixed work, in (h+64)(w+16) units
static_assert(kAreaQ == sizeof(ClsCtrl::astg[0]) / sizeof(uint64_t), "one mbarrier per AREA item in flight");
constexpr uint32_t kAreaVBytes = 2u * 784u + 16u;           // V scratch: u16 per byte of a segment (+ overread)
// per converter warp: V buffers (2 with two tuples per pass) + the item ring; the K4 AREA instance
// with 12 converter warps (kAreaWarps) has room for one V buffer and a 5 KB ring per warp
// Per converter warp: one item ring; an item's vertical sums V (2 bytes per segment byte) are written
// over its own staged rows (an item is allocated max(hb, 2) rows), so no separate V buffer; 16 bytes
// of slack after the ring keep the last column's second word inside the warp's region.
template <int kCW>
struct AreaCfg {
  static constexpr bool kPairItems = kCW == kConvWarps;  // (two tuples per pass: the ring holds two items)
  static constexpr int kBS = kCW > 12 ? 2 : 3;  // the kernel's weight stages (16 KB each at N = 128)
  static constexpr uint32_t kAvail =
      static_cast<uint32_t>(kClsSmemBytes - 1023 - kARing * kAKBlockBytes - kBS * 16384 - sizeof(ClsCtrl) - 15);
  static constexpr uint32_t kFit = ((kAvail / kCW - 16u) & ~15u) < 9600u ? ((kAvail / kCW - 16u) & ~15u) : 9600u;
#ifndef HYDRO_AREA_RING_FIT  // a power-of-two ring (offsets by mask) when it still holds the pass's items
  static constexpr uint32_t kPow2 = kFit >= 8192u ? 8192u : (kFit >= 4096u ? 4096u : kFit);
  static constexpr uint32_t kRing = kPow2 >= (kCW == kConvWarps ? 2u : 1u) * 3920u ? kPow2 : kFit;
#else
  static constexpr uint32_t kRing = kFit;
#endif
  static constexpr uint32_t kRegion = kRing + 16u;
  static_assert(kRing >= (kPairItems ? 2u : 1u) * 5u * 784u && kRing % 16u == 0,
                "the worst-case AREA items of a pass (5 source rows of 784 B each) must fit the ring");
  static_assert(1023 + kARing * kAKBlockBytes + kBS * 16384 + sizeof(ClsCtrl) + 15 + kCW * kRegion <= kClsSmemBytes,
                "AREA staging exceeds shared memory");
};
constexpr int kAreaWarps = HYDRO_AREA_WARPS;  // converter warps of K4's AREA-only instance (launched beside K4-T)

__device__ __forceinline__ uint32_t f16x2_of_bf16x2(uint32_t b) {  // exact (bf16 means of u8 pixels)
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(__uint_as_float(b & 0xFFFF0000u)), "f"(__uint_as_float(b << 16)));
  return d;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float ldsf(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t a) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(a) : "memory");
}

template <bool kDbg, int kP, int kCW>
__device__ __forceinline__ void convert_tile_area(const ClsParams& p, ClsCtrl* ctrl, uint32_t lim, uint32_t pos0,
                                                  uint32_t crank, int cu, int lane, uint32_t region, uint32_t a_ring,
                                                  uint32_t row_pitch, bool fp16, const RowMeta& mm, uint32_t my_row,
                                                  uint32_t& gg, uint32_t& qseq) {
  const uint8_t* frames = p.frames;
  constexpr uint32_t kAreaRing = AreaCfg<kCW>::kRing;
  constexpr bool kPairItems = AreaCfg<kCW>::kPairItems;
  const uint32_t ring = region;
  const uint32_t rcp_tab = smem_u32(ctrl->area_rcp);
  // tuple t of the band = lane t (valid tuples are a prefix: rows past the hop's count are masked)
  const uint32_t nv = __popc(__ballot_sync(0xFFFFFFFFu, lane < 16 && mm.valid));
  const uint32_t my_src = mm.row16 + (mm.seg_lo >> 4), my_len = mm.seg_len, my_h = static_cast<uint32_t>(mm.h);
  const uint32_t my_xw = static_cast<uint32_t>(mm.x0) | (static_cast<uint32_t>(mm.w) << 16);
  const uint32_t total = kGroups * nv;
  // this lane's 3 A words: byte o = 12q + 4i of the 384-byte crop row -> K-block o / 128, 16-byte
  // chunk (o / 16) % 8 (swizzled with the row), byte o % 16
  uint32_t st_off[3], st_chk[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t o = 12u * static_cast<uint32_t>(lane) + 4u * i;
    st_off[i] = (o >> 7) * kAKBlockBytes + (o & 15u);
    st_chk[i] = (o >> 4) & 7u;
  }
  // ring allocation (producer and consumer replay the same rule): an item starts at the cursor, or
  // at the next ring start when it would cross the ring's end
  auto place = [](uint32_t cur, uint32_t bytes) {
    const uint32_t ph = cur % kAreaRing;
    return ph + bytes > kAreaRing ? cur + (kAreaRing - ph) : cur;
  };
  uint32_t pk = 0, pg = 0, pt = 0, pcur = 0;  // producer: next item, its (g, t), ring cursor
  uint32_t cnext = 0, clive = 0, ck = 0;      // consumer: end of the last consumed item, oldest live byte, next item
  // stage items ahead while the queue and the ring have room (oldest = start of item ck)
  auto produce = [&](uint32_t oldest) {
    while (pk < total && pk - ck < static_cast<uint32_t>(kAreaQ)) {
      const uint32_t Lp = __shfl_sync(0xFFFFFFFFu, my_len, pt);
      const uint32_t hp = __shfl_sync(0xFFFFFFFFu, my_h, pt);
      const uint32_t srcp = __shfl_sync(0xFFFFFFFFu, my_src, pt);
      const uint32_t ysp = (pg * hp) >> 6, hbp = (((pg + 1u) * hp + 63u) >> 6) - ysp;
      const uint32_t bytes = max(hbp, 2u) * Lp;  // (V is written over the item: 2 bytes per segment byte)
      const uint32_t ps = place(pcur, bytes);
      if (ps + bytes - min(oldest, ps) > kAreaRing) break;  // the ring is full
      uint64_t* bar = &ctrl->astg[cu][(qseq + pk) % kAreaQ];
      if (lane == 0) mbar_arrive_expect_tx(bar, hbp * Lp);
      __syncwarp();
      if (static_cast<uint32_t>(lane) < hbp)
        bulk_g2s_u32(ring + ps % kAreaRing + lane * Lp, at16(frames, srcp) + (ysp + lane) * row_pitch, Lp, bar);
      pcur = ps + bytes;
      ++pk;
      if (++pt == nv) {
        pt = 0;
        ++pg;
      }
    }
  };
  // consume item ck (crop row g of tuple t): wait for its rows, vertical sums -> V over the item
  // (every lane's loads of both of its chunks before any V store; the item stays live until the
  // pass's horizontal sums are done: clive)
  auto consume = [&](uint32_t g, uint32_t t, uint32_t& vb_out, uint32_t& hb_out, uint32_t& xw_out) {
    const uint32_t L = __shfl_sync(0xFFFFFFFFu, my_len, t);
    const uint32_t h = __shfl_sync(0xFFFFFFFFu, my_h, t);
    xw_out = __shfl_sync(0xFFFFFFFFu, my_xw, t);
    const uint32_t ys = (g * h) >> 6, hb = (((g + 1u) * h + 63u) >> 6) - ys;
    hb_out = hb;
    const uint32_t cstart = place(cnext, max(hb, 2u) * L);
    produce(clive == cnext ? cstart : clive);
    mbar_wait(&ctrl->astg[cu][(qseq + ck) % kAreaQ], ((qseq + ck) / kAreaQ) & 1u);
    const uint32_t item = ring + cstart % kAreaRing;
    uint32_t s[2][8];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
#pragma unroll
      for (int q = 0; q < 8; ++q) s[k][q] = 0u;
      const uint32_t c16 = static_cast<uint32_t>(lane) + 32u * k;
      if (16u * c16 < L) {
        uint32_t a = item + 16u * c16;
        for (uint32_t i = 0; i < hb; ++i, a += L) {
          const uint4 r = lds128(a);
          s[k][0] += __byte_perm(r.x, 0u, 0x4140);  // bytes 0, 1 as u16 halves
          s[k][1] += __byte_perm(r.x, 0u, 0x4342);  // bytes 2, 3
          s[k][2] += __byte_perm(r.y, 0u, 0x4140);
          s[k][3] += __byte_perm(r.y, 0u, 0x4342);
          s[k][4] += __byte_perm(r.z, 0u, 0x4140);
          s[k][5] += __byte_perm(r.z, 0u, 0x4342);
          s[k][6] += __byte_perm(r.w, 0u, 0x4140);
          s[k][7] += __byte_perm(r.w, 0u, 0x4342);
        }
      }
    }
    __syncwarp();  // every lane's loads of the item are done: V may overwrite it
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t c16 = static_cast<uint32_t>(lane) + 32u * k;
      if (16u * c16 < L) {
        sts128(item + 32u * c16, s[k][0], s[k][1], s[k][2], s[k][3]);
        sts128(item + 32u * c16 + 16u, s[k][4], s[k][5], s[k][6], s[k][7]);
      }
    }
    vb_out = item;
    cnext = cstart + max(hb, 2u) * L;
    ++ck;
  };
  for (uint32_t g = 0; g < static_cast<uint32_t>(kGroups); ++g, ++gg) {
    const uint32_t set = (gg & 1u) * kKBlocksPerGroup, aph = (gg >> 1) & 1u;
#pragma unroll
    for (int kbr = 0; kbr < kKBlocksPerGroup; ++kbr) mbar_wait(&ctrl->empty_a[set + kbr], aph ^ 1u);
    const uint32_t a_set = a_ring + set * kAKBlockBytes;
    // two tuples per pass: their vertical sums in turn (the ring holds one worst-case item), then
    // the horizontal sums, divisions and stores of both interleaved
    for (uint32_t t = 0; t < nv; t += kPairItems ? 2u : 1u) {
      const bool two = kPairItems && t + 1 < nv;
      uint32_t hb[2], xw[2], vbs[2];
      consume(g, t, vbs[0], hb[0], xw[0]);
      if (two) consume(g, t + 1, vbs[1], hb[1], xw[1]);
      else hb[1] = xw[1] = 0u, vbs[1] = vbs[0];
      __syncwarp();  // V complete
      // ---- horizontal bin sums of pixels q and q + 32 of both tuples
      uint32_t b2[2][2], bw[2][2], par[2][2], bwmax = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t x0 = xw[u] & 0xFFFFu, w = xw[u] >> 16, slo = (3u * x0) & ~15u;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t dx = static_cast<uint32_t>(lane) + 32u * e;
          const uint32_t xs = (dx * w) >> 6;
          bw[u][e] = (((dx + 1u) * w + 63u) >> 6) - xs;  // 0 for an absent second tuple (w = 0)
          const uint32_t b = 3u * (x0 + xs) - slo;  // V index of the bin's first column, channel 0
          b2[u][e] = vbs[u] + 2u * b;  // byte address of V[b]
          par[u][e] = b & 1u;                          // V[b] is the high half of its word
          bwmax = max(bwmax, bw[u][e]);
        }
      }
      uint32_t s01[2][2] = {{0u, 0u}, {0u, 0u}}, s2[2][2] = {{0u, 0u}, {0u, 0u}};
      for (uint32_t c = 0; c < bwmax; ++c) {
        uint32_t w0[2][2], w1[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool on = c < bw[u][e];
            const uint32_t a = (b2[u][e] + 6u * c) & ~3u;  // column xs + c (V buffers are 16-byte aligned)
            w0[u][e] = on ? lds32(a) : 0u;
            w1[u][e] = on ? lds32(a + 4u) : 0u;
          }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool odd = (par[u][e] ^ c) & 1u;
            s01[u][e] += __byte_perm(w0[u][e], w1[u][e], odd ? 0x5432 : 0x3210);
            s2[u][e] += __byte_perm(w1[u][e], 0u, odd ? 0x4432 : 0x4410);
          }
      }
      // ---- means: one RN division each (area_div), bf16 RNE; 6 features = 3 words per tuple
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && !two) break;
        float v[6];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t n = hb[u] * bw[u][e];
          const float cnt = static_cast<float>(n);
          const float rcp = ldsf(rcp_tab + 4u * n);  // RN(1 / n), n <= 25
          v[3 * e + 0] = area_div(static_cast<float>(s01[u][e] & 0xFFFFu), cnt, rcp);
          v[3 * e + 1] = area_div(static_cast<float>(s01[u][e] >> 16), cnt, rcp);
          v[3 * e + 2] = area_div(static_cast<float>(s2[u][e]), cnt, rcp);
        }
        const uint32_t m = __shfl_sync(0xFFFFFFFFu, my_row, t + u);  // tile row of the tuple
        const uint32_t row_base = a_set + (m >> 3) * 1024u + (m & 7u) * 128u;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const uint32_t bb = bf16x2_rn(v[2 * i], v[2 * i + 1]);
          sts32(row_base + st_off[i] + ((st_chk[i] ^ (m & 7u)) << 4), fp16 ? f16x2_of_bf16x2(bb) : bb);
          if (kDbg && p.dbg_crops && pos0 + m < lim) {
            uint16_t* dbg = p.dbg_crops + static_cast<uint64_t>(pos0 + m) * kFeatures + g * 192u;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const uint32_t pp = 2u * i + hf;  // position 6q + pp
              dbg[3u * (static_cast<uint32_t>(lane) + 32u * (pp / 3u)) + pp % 3u] =
                  static_cast<uint16_t>(hf ? bb >> 16 : bb & 0xFFFFu);
            }
          }
        }
      }
      __syncwarp();  // the pass's items (V) are released
      clive = cnext;
    }
    // group g complete: publish its A stages
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int kbr = 0; kbr < kKBlocksPerGroup; ++kbr) {
        if (kP == 2 && crank != 0) mbar_arrive_leader(&ctrl->full_a[set + kbr]);
        else mbar_arrive(&ctrl->full_a[set + kbr]);
      }
    }
  }
  qseq += total;
}

// Converter warps (shared by the linear and the MLP classifier kernels): cp.async-staged crop-row
// segments -> pixels -> the swizzled K-major A ring, one K-group (crop row g of all 128 tuples of
// the CTA's M-tile) at a time, full_a / empty_a handshake with the MMA issuer.
template <bool kDbg, bool kArea, int kP, int kQD, int kCW = kConvWarps>
__device__ __forceinline__ void converter_role(const ClsParams& p, ClsCtrl* ctrl, const uint32_t* list_in,
                                               uint32_t base, const TileWalk& tw, uint32_t crank, int warp, int lane,
                                               uint32_t staging_addr, uint32_t a_ring, uint32_t row_pitch, bool area,
                                               bool fp16) {
  constexpr int kQS = kQD + 1;
  // ===================== converters: cp.async-staged segments -> pixels -> swizzled A ring
  // Warp cu owns up to 16 rows of the tile (kCW = 8: rows 16*cu .. 16*cu+15; the AREA instance's
  // 16 warps: 8 rows each; data-aware AREA tiles: the rows dealt to it by estimated work).  Nearest
  // and wide tiles walk them as "quads" of 4 rows (one warp instruction = 4 rows x 8 lanes x 8
  // output pixels), their source segments copied (16-byte cp.async) kQD quads ahead into fixed
  // slots; AREA tiles run the row-cooperative converter (convert_tile_area).
  const int cu = warp - kConvWarp0;
  const uint32_t slots = staging_addr + static_cast<uint32_t>(cu) * (kQS * kQuadSlotBytes);
  uint32_t gg = 0, qseq = 0;
  for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step) {
    const uint32_t pos0 = tw.pos0(unit);
    // rows' metadata: lane l < 16 holds this warp's l-th row (8 warps: rows 16*cu + l; 16 warps:
    // rows 8*cu + l; other counts: floor or ceil of 128/kCW consecutive rows; lanes past them hold none)
    constexpr uint32_t kRowsLo = kTileM / kCW, kRowsRem = kTileM % kCW;
    const uint32_t my_n = kRowsLo + (static_cast<uint32_t>(cu) < kRowsRem ? 1u : 0u);
    const uint32_t my_base = static_cast<uint32_t>(cu) * kRowsLo + min(static_cast<uint32_t>(cu), kRowsRem);
    uint32_t my_row = static_cast<uint32_t>(lane & 15) < my_n ? my_base + (lane & 15) : 0xFFu;
    RowMeta mm = load_meta(p, list_in, base, pos0 + my_row, (lane < 16 && my_row < kTileM) ? tw.lim : 0u);
#ifdef HYDRO_AREA_BAL_ALWAYS
    if (kArea && area) {
#else
    if (kArea && area && tw.wbal) {
#endif
      // data-aware AREA tiles (R28) at warp granularity: the converter warps are the tile's
      // workers; each tile row's work is estimated from its input size, kAreaFixedCost + (h + 64)(w + 16)
      // (~ source bytes staged and summed per crop, plus the per-tuple fixed part), the rows are
      // ranked by it (ties: lower row first) and dealt to the warps in snake order (rank k -> warp
      // k % 8, or 7 - k % 8 on odd rounds, slot k / 8), so every warp's load is within one row of
      // the others' and the hop's invalid rows (ranked last) stay a suffix of every warp's slots
      if (lane < 16 && my_row < kTileM)
        ctrl->area_cost[my_row] =
            mm.valid ? kAreaFixedCost + static_cast<uint32_t>((mm.h + 64) * (mm.w + 16)) : 0u;
      if (kCW * 16 > kTileM && lane < 16) ctrl->area_perm[cu * 16 + lane] = 0xFFu;  // slots left empty
      named_bar_sync(1, kCW * 32);
      if (cu < kTileM / 32) {
        const uint32_t m = static_cast<uint32_t>(cu * 32 + lane), cm = ctrl->area_cost[m];
        uint32_t k = 0;
        for (uint32_t j = 0; j < static_cast<uint32_t>(kTileM); ++j) {
          const uint32_t cj = ctrl->area_cost[j];
          k += (cj > cm || (cj == cm && j < m)) ? 1u : 0u;
        }
        const uint32_t s = k / kCW, c = (s & 1u) ? kCW - 1u - k % kCW : k % kCW;
        ctrl->area_perm[c * 16 + s] = static_cast<uint8_t>(m);
      }
      named_bar_sync(1, kCW * 32);
      my_row = ctrl->area_perm[cu * 16 + (lane & 15)];
      mm = load_meta(p, list_in, base, pos0 + my_row, (lane < 16 && my_row < kTileM) ? tw.lim : 0u);
    }
    // a tile with a crop wider than a staging slot (rare) runs the gather-staging variant
    const bool any_wide =
        __any_sync(0xFFFFFFFFu, lane < 16 && mm.valid && mm.seg_len > static_cast<uint32_t>(kMaxSegBytes));
    // AREA: the row-cooperative converter takes bins of <= 5 x 5 pixels (w, h <= 256: a bin spans
    // <= ceil(w/64) + 1 columns); a tile with a larger crop takes the direct global-load converter
    const bool area_big = kArea && area &&
                          __any_sync(0xFFFFFFFFu, lane < 16 && mm.valid && (mm.w > 256 || mm.h > 256));
    if (kArea && area && !any_wide && !area_big)
      convert_tile_area<kDbg, kP, kCW>(p, ctrl, tw.lim, pos0, crank, cu, lane,
                                       staging_addr + cu * AreaCfg<kCW>::kRegion, a_ring, row_pitch, fp16, mm,
                                       my_row, gg, qseq);
    else if (any_wide || area_big)
      convert_tile<kDbg, kArea, kP, kQD, true>(p, ctrl, list_in, tw.lim, pos0, crank, cu, lane, slots, a_ring, row_pitch,
                                               area, fp16, mm, my_row, gg);
    else
      convert_tile<kDbg, kArea, kP, kQD, false>(p, ctrl, list_in, tw.lim, pos0, crank, cu, lane, slots, a_ring,
                                                row_pitch, area, fp16, mm, my_row, gg);
  }
  if (kP == 2) {  // drain: both A sets released (the leader's commits land here)
    for (int e = 0; e < 2; ++e, ++gg) {
      const uint32_t set = (gg & 1u) * kKBlocksPerGroup, aph = (gg >> 1) & 1u;
      for (int kbr = 0; kbr < kKBlocksPerGroup; ++kbr) mbar_wait(&ctrl->empty_a[set + kbr], aph ^ 1u);
    }
  }
}

extern __shared__ __align__(1024) uint8_t hydro_cls_smem[];

template <bool kDbg, bool kArea, int kCW = kConvWarps>
__global__ void __launch_bounds__((kConvWarp0 + kCW) * 32, 1) hydro_classifier_kernel(ClsParams p) {
  // weight (B) stages: 3, or 2 for the instance with more than 12 converter warps (whose staging
  // takes the third stage's 16 KB; the MMA is far from binding on AREA hops)
  constexpr int kBS = kCW > 12 ? 2 : kBStages;
  DevState* st = p.st;
  // ---- dispatch (uniform across the CTA: every thread reads the same device words)
  int pred;
  const uint32_t* list_in;
  uint32_t count, base = p.range_base;
  uint32_t* bits_out;
  if (p.dispatch) {
    const int h = st->sched[p.hop];  // p.hop is the chain slot
    if (h < 0 || h >= st->n_pred) return;
    pred = st->order[h];
    if (st->kind[pred] != kLinear) return;  // (an MLP hop runs in hydro_mlp_kernel)
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
  // cached classifier hop: only the uncached tuples (K0c's list), verdict bits by hop position
  const uint32_t* ind = cls_redirect(p, p.preds[pred], list_in, count);
  const bool fill = p.preds[pred].cache_known && (p.preds[pred].cache_fill || p.force_fill);
  const uint32_t num_tiles = (count + kTileM - 1) / kTileM;
  const PredDev& pdg = p.preds[pred];
  const bool area = kArea && pdg.crop_mode == HYDRO_CROP_AREA;  // kArea: the context has an AREA head
  if (p.area_only && !area) return;  // a nearest hop: K4-T (launched beside this kernel) evaluates it
  // work unit = kPair consecutive M-tiles (one per CTA of the cluster); both CTAs of a pair walk
  // the same units, so a pair's last unit may hold a tile past num_tiles (all rows invalid)
  const uint32_t crank = kPair == 2 ? cluster_ctarank() : 0u;
  TileWalk tw{blockIdx.x / kPair, gridDim.x / kPair, (num_tiles + kPair - 1) / kPair, 0u, count, kPair, crank, false};
  const bool data_aware = kPair == 1 && area && p.bounds && !ind;
  tw.wbal = data_aware;
  if (data_aware && count < kBalRangeTilesPerCta * kTileM * gridDim.x) {  // this CTA's balanced position range
    tw.bal = true;
    tw.lo = min(p.bounds[blockIdx.x], count);
    tw.lim = min(p.bounds[blockIdx.x + 1], count);
    tw.first = 0;
    tw.step = 1;
    tw.end = tw.lim > tw.lo ? (tw.lim - tw.lo + kTileM - 1) / kTileM : 0u;
  }
  if (threadIdx.x == 0) ktimer_begin(st, 1);
  if (tw.first >= tw.end) {
    if (threadIdx.x == 0) ktimer_end(st, 1);
    return;
  }

  const long long t_start = clock64();
  const int n_classes = pdg.n_classes, n_pad = pdg.n_pad, target = pdg.target;
  const bool fp16 = pdg.a_fp16 != 0;
  const float unscale = pdg.w_unscale;
  const uint8_t* w_tiled = pdg.w_tiled;
  const int n_alloc = n_pad <= 32 ? 32 : (n_pad <= 64 ? 64 : 128);
  const uint32_t tmem_cols = 2u * n_alloc;
  const uint32_t b_stage_bytes = static_cast<uint32_t>(n_pad) * 128u;
  const uint32_t b_load_bytes = b_stage_bytes / kPair;  // pair: CTA r holds weight rows [r*N/2, (r+1)*N/2)
  const uint32_t row_pitch = static_cast<uint32_t>(p.frame_w * 3);

  // ---- shared memory carve-up: [A ring][B ring][ctrl][staging ring]
  const uint32_t raw = smem_u32(hydro_cls_smem);
  uint8_t* smem = hydro_cls_smem + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t a_ring = smem_u32(smem);
  const uint32_t b_ring = a_ring + kARing * kAKBlockBytes;
  const uint32_t ctrl_off = kARing * kAKBlockBytes + kBS * b_load_bytes;
  ClsCtrl* ctrl = reinterpret_cast<ClsCtrl*>(smem + ctrl_off);
  const uint32_t stg_off = (ctrl_off + static_cast<uint32_t>(sizeof(ClsCtrl)) + 15u) & ~15u;
  uint8_t* staging = smem + stg_off;
  const uint32_t staging_addr = smem_u32(staging);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kARing; ++s) {
      mbar_init(&ctrl->full_a[s], kCW * kPair);
      mbar_init(&ctrl->empty_a[s], 1);
    }
    for (int s = 0; s < kBS; ++s) {
      mbar_init(&ctrl->full_b[s], crank == 0 ? kPair : 1);  // pair: + the peer's relay
      mbar_init(&ctrl->empty_b[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&ctrl->tfull[a], 1);
      mbar_init(&ctrl->tempty[a], kEpiWarps * kPair);
    }
    if (kArea)
      for (int w = 0; w < kCW; ++w)
        for (int s = 0; s < kAreaQ; ++s) mbar_init(&ctrl->astg[w][s], 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    if constexpr (kPair == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&ctrl->tmem_base)),
                   "r"(tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&ctrl->tmem_base)),
                   "r"(tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  if (tid < HYDRO_MAX_CLASSES) ctrl->bias[tid] = tid < n_classes ? pdg.bias[tid] : 0.0f;
  if (kArea && tid < 32) ctrl->area_rcp[tid] = __frcp_rn(static_cast<float>(max(tid, 1)));
  tc_fence_before();
  if constexpr (kPair == 2) cluster_sync_all();  // the peer's barriers are initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = ctrl->tmem_base;

  if (warp == kLoaderWarp) {
    // ===================== loader: weight K-blocks (bulk copy) + L2 prefetch of crop rows
#ifndef HYDRO_PF_GROUPS
#define HYDRO_PF_GROUPS 4
#endif
    constexpr int kPrefetchGroups = HYDRO_PF_GROUPS;
    const uint64_t pol_w = policy_evict_last();  // weights are re-read by every tile: keep them in L2
    uint32_t itb = 0;
    for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step) {
      const uint32_t pos0 = tw.pos0(unit);
      RowMeta mr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) mr[r] = load_meta(p, list_in, base, pos0 + lane * 4 + r, tw.lim);
      auto prefetch_group = [&](int g) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (!mr[r].valid) continue;
          if (area) {
            // AREA: no L2 prefetch by default (the converters' bulk copies run up to 8 items ahead;
            // prefetching 4 groups ahead measured 84 vs 52 GB of DRAM reads per 1M crops at the
            // same speed).  HYDRO_AREA_PF: every source row of the crop row's bins, whole lines
#ifndef HYDRO_AREA_PF
            continue;
#endif
            const uint32_t h = static_cast<uint32_t>(mr[r].h);
            const uint32_t ys = (static_cast<uint32_t>(g) * h) >> 6, ye = ((static_cast<uint32_t>(g) + 1u) * h + 63u) >> 6;
            for (uint32_t y = ys; y < ye; ++y) {
              const uint8_t* a = at16(p.frames, mr[r].row16) + y * row_pitch + mr[r].seg_lo;
              for (uint32_t c = 0; c < mr[r].seg_len; c += 128u) prefetch_line_l2(a + c);
            }
            continue;
          }
          const uint32_t sy = static_cast<uint32_t>(((2 * g + 1) * mr[r].h) >> 7);
          const uint8_t* a = at16(p.frames, mr[r].row16) + sy * row_pitch + mr[r].seg_lo;
#if defined(HYDRO_L2_PREFETCH)  // measured slightly slower on B200 (line-granular overfetch, L2 pressure)
          for (uint32_t c = 0; c < mr[r].seg_len; c += 128u) prefetch_line_l2(a + c);
#else
          (void)a;
#endif
        }
      };
      for (int g = 0; g < kPrefetchGroups; ++g) prefetch_group(g);
      for (int kb = 0; kb < kNumKBlocks; ++kb, ++itb) {
        if (kb % kKBlocksPerGroup == 0) {
          const int g = kb / kKBlocksPerGroup + kPrefetchGroups;
          if (g < kGroups) prefetch_group(g);
        }
        if (lane == 0) {
          const uint32_t s = itb % kBS, ph = (itb / kBS) & 1u;
          HYDRO_PIPE_WAIT(&ctrl->empty_b[s], ph ^ 1u);
          mbar_arrive_expect_tx(&ctrl->full_b[s], b_load_bytes);
          bulk_g2s_hint(smem + (b_ring - a_ring) + s * b_load_bytes,
                        w_tiled + static_cast<uint64_t>(kb) * b_stage_bytes + crank * b_load_bytes, b_load_bytes,
                        &ctrl->full_b[s], pol_w);
        }
        __syncwarp();
      }
    }
    if (kPair == 2 && lane == 0) {  // drain: every B stage released (the leader's commits land here)
      for (int e = 0; e < kBS; ++e, ++itb) mbar_wait(&ctrl->empty_b[itb % kBS], ((itb / kBS) & 1u) ^ 1u);
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (single thread)
    if (kPair == 2 && crank != 0 && lane == 0) {
      // peer: relay "my half of B landed" to the leader's full_b (the bulk copy completes locally)
      uint32_t itb = 0;
      for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step) {
        for (int kb = 0; kb < kNumKBlocks; ++kb, ++itb) {
          const uint32_t s = itb % kBS;
          mbar_wait(&ctrl->full_b[s], (itb / kBS) & 1u);
          mbar_arrive_leader(&ctrl->full_b[s]);
        }
      }
    } else if (lane == 0) {
      const uint32_t idesc = idesc_f16_f32(kTileM * kPair, static_cast<uint32_t>(n_pad), !fp16);
      uint32_t itb = 0, gg = 0, tl = 0;
      for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step, ++tl) {
        const uint32_t acc = tl & 1u, aph = (tl >> 1) & 1u;
        mbar_wait_backoff<256>(&ctrl->tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * static_cast<uint32_t>(n_alloc);
        for (int g = 0; g < kGroups; ++g, ++gg) {
          const uint32_t set = (gg & 1u) * kKBlocksPerGroup, aph2 = (gg >> 1) & 1u;
#pragma unroll
          for (int kbr = 0; kbr < kKBlocksPerGroup; ++kbr, ++itb) {
            const uint32_t sa = set + kbr;
            const uint32_t sb = itb % kBS, bph = (itb / kBS) & 1u;
            // (pair: the leader's barriers also count the peer's remote arrivals)
            HYDRO_PIPE_WAIT(&ctrl->full_a[sa], aph2);
            HYDRO_PIPE_WAIT(&ctrl->full_b[sb], bph);
            tc_fence_after();
            const uint32_t a_addr = a_ring + sa * kAKBlockBytes;
            const uint32_t b_addr = b_ring + sb * b_load_bytes;
#pragma unroll
            for (int kk = 0; kk < kKBlock / 16; ++kk) {
              if constexpr (kPair == 2)
                tc_mma_pair(d_tmem, desc_sw128(a_addr + kk * 32), desc_sw128(b_addr + kk * 32), idesc,
                            (g | kbr | kk) != 0 ? 1u : 0u);
              else
                tc_mma_bf16(d_tmem, desc_sw128(a_addr + kk * 32), desc_sw128(b_addr + kk * 32), idesc,
                            (g | kbr | kk) != 0 ? 1u : 0u);
            }
            if constexpr (kPair == 2) {
              tc_commit_pair(&ctrl->empty_a[sa]);
              tc_commit_pair(&ctrl->empty_b[sb]);
            } else {
              tc_commit(&ctrl->empty_a[sa]);
              tc_commit(&ctrl->empty_b[sb]);
            }
          }
        }
        if constexpr (kPair == 2) tc_commit_pair(&ctrl->tfull[acc]);
        else tc_commit(&ctrl->tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= kConvWarp0) {
    converter_role<kDbg, kArea, kPair, kQuadDepth, kCW>(p, ctrl, list_in, base, tw, crank, warp, lane, staging_addr,
                                                        a_ring, row_pitch, area, fp16);
  } else {
    // ===================== epilogue warps 0..3 (TMEM lane quadrant = warp)
    const int q = warp;
    uint32_t n_in = 0, n_pass = 0, tl = 0;
    for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step, ++tl) {
      const uint32_t pos0 = tw.pos0(unit);
      const uint32_t acc = tl & 1u, aph = (tl >> 1) & 1u;
      mbar_wait_backoff<1024>(&ctrl->tfull[acc], aph);
      tc_fence_after();
      const int m = q * 32 + lane;
      const uint32_t pos = pos0 + m;
      const bool valid = pos < tw.lim;
      float best = -3.402823466e38f;
      int bi = 0;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * static_cast<uint32_t>(n_alloc);
      for (int c0 = 0; c0 < n_pad; c0 += 16) {
        uint32_t v[16];
        tc_ld_32x32b_x16(taddr + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int c = c0 + jj;
          if (c < n_classes) {
            const float z = __uint_as_float(v[jj]) * unscale + ctrl->bias[c];  // 2^-k: exact
            if (z > best) {  // strict: lowest index wins ties (R12)
              best = z;
              bi = c;
            }
            if (kDbg && p.dbg_logits && valid) p.dbg_logits[static_cast<uint64_t>(pos) * n_classes + c] = z;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (kPair == 2 && crank != 0) mbar_arrive_leader(&ctrl->tempty[acc]);
        else mbar_arrive(&ctrl->tempty[acc]);
      }
      const bool verdict = valid && (bi == target);
      const uint32_t bv = __ballot_sync(0xFFFFFFFFu, verdict);
      const uint32_t bvalid = __ballot_sync(0xFFFFFFFFu, valid);
      cls_emit(p, bits_out, ind, list_in, base, pos0 + q * 32, pos, valid, verdict, pdg, fill);
      if (kDbg && p.dbg_verdict && valid) p.dbg_verdict[pos] = verdict ? 1 : 0;
      n_in += __popc(bvalid);
      n_pass += __popc(bv);
    }
    if (p.collect_stats && lane == 0) {
      atomicAdd(&st->d_in[pred], static_cast<unsigned long long>(n_in));
      atomicAdd(&st->d_pass[pred], static_cast<unsigned long long>(n_pass));
      atomicAdd(&st->d_comp[pred], static_cast<unsigned long long>(n_in));  // no verdict cache here
    }
    if (lane == 0) atomicAdd(&st->kt_items[1], static_cast<unsigned long long>(n_in));
  }

  tc_fence_before();
  if constexpr (kPair == 2) cluster_sync_all();  // no CTA leaves while its peer may still touch it
  else __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    if constexpr (kPair == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols)
                   : "memory");
  }
  if (tid == 0 && p.collect_stats) {
    atomicAdd(&st->d_cost[pred], static_cast<unsigned long long>(clock64() - t_start));
  }
  if (tid == 0) ktimer_end(st, 1);
}

// ------------------------------------------------------------------------------------------
// K4-MLP (R25): z = W2 . bf16(relu(W1 . Crop(frame, bbox) + b1)) + b2, verdict
// argmax z == target.  CTA pairs (cta_group::2, M = 256 tuples per unit): the first layer is
// 12288 x hidden (hidden = 256 / 512), N = 256 per MMA, its fp32 accumulator fills the CTA's whole
// TMEM (512 columns).  The epilogue adds b1, applies ReLU, rounds to bf16 and writes the packed
// activations back into TMEM columns [0, hidden/2); the second layer then runs with A read from
// TMEM (no shared-memory round trip) into columns [256, 256 + n_pad).  W1 K-blocks (each CTA
// loads its half of every N=256 slice) and W2 K-blocks stream through a 2 x 32 KB ring; the
// converters are the linear kernel's, with a one-quad staging lookahead (shared memory).
template <bool kDbg>
__global__ void __launch_bounds__(kClsThreads, 1) hydro_mlp_kernel(ClsParams p) {
  // B stage = this CTA's half of one N=256 slice of a W1 K-block (16 KB) or of a W2 K-block;
  // 3 stages leave room for the linear kernel's two-quad staging lookahead
  constexpr int kP = 2, kQD = kQuadDepth, kMB = 3;
  constexpr uint32_t kMlpBStage = 16384;
  DevState* st = p.st;
  int pred;
  const uint32_t* list_in;
  uint32_t count, base = p.range_base;
  uint32_t* bits_out;
  if (p.dispatch) {
    const int h = st->sched[p.hop];
    if (h < 0 || h >= st->n_pred) return;
    pred = st->order[h];
    if (st->kind[pred] != kMlp) return;
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
  // cached classifier hop: only the uncached tuples (K0c's list), verdict bits by hop position
  const uint32_t* ind = cls_redirect(p, p.preds[pred], list_in, count);
  const bool fill = p.preds[pred].cache_known && (p.preds[pred].cache_fill || p.force_fill);
  const uint32_t num_tiles = (count + kTileM - 1) / kTileM;
  const uint32_t crank = cluster_ctarank();
  const TileWalk tw{blockIdx.x / kP, gridDim.x / kP, (num_tiles + kP - 1) / kP, 0u, count, kP, crank, false};
  if (threadIdx.x == 0) ktimer_begin(st, 4);
  if (tw.first >= tw.end) {
    if (threadIdx.x == 0) ktimer_end(st, 4);
    return;
  }

  const long long t_start = clock64();
  const PredDev& pdg = p.preds[pred];
  const int n_classes = pdg.n_classes, n_pad = pdg.n_pad, target = pdg.target, hidden = pdg.hidden;
  const bool fp16 = pdg.a_fp16 != 0;
  const int n_mma1 = hidden / 256;                                     // N=256 slices of layer 1
  const uint32_t w1_kb = static_cast<uint32_t>(hidden) * 128u;          // one tiled W1 K-block
  const uint32_t w2_load = static_cast<uint32_t>(n_pad / 2) * 128u;     // this CTA's half of a W2 K-block
  const uint32_t w2_kb = static_cast<uint32_t>(n_pad) * 128u;
  const int n_kb2 = hidden / kKBlock;
  const uint32_t tmem_cols = 512;
  const uint32_t row_pitch = static_cast<uint32_t>(p.frame_w * 3);

  const uint32_t raw = smem_u32(hydro_cls_smem);
  uint8_t* smem = hydro_cls_smem + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t a_ring = smem_u32(smem);
  const uint32_t b_ring = a_ring + kARing * kAKBlockBytes;
  const uint32_t ctrl_off = kARing * kAKBlockBytes + kMB * kMlpBStage;
  ClsCtrl* ctrl = reinterpret_cast<ClsCtrl*>(smem + ctrl_off);
  const uint32_t stg_off = (ctrl_off + static_cast<uint32_t>(sizeof(ClsCtrl)) + 15u) & ~15u;
  const uint32_t staging_addr = smem_u32(smem + stg_off);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kARing; ++s) {
      mbar_init(&ctrl->full_a[s], kConvWarps * kP);
      mbar_init(&ctrl->empty_a[s], 1);
    }
    for (int s = 0; s < kMB; ++s) {
      mbar_init(&ctrl->full_b[s], crank == 0 ? 2 : 1);
      mbar_init(&ctrl->empty_b[s], 1);
    }
    mbar_init(&ctrl->tfull[0], 1);
    mbar_init(&ctrl->tempty[0], kEpiWarps * kP);
    mbar_init(&ctrl->hready, kEpiWarps * kP);
    mbar_init(&ctrl->tfull2, 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&ctrl->tmem_base)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid < HYDRO_MAX_CLASSES) ctrl->bias[tid] = tid < n_classes ? pdg.bias[tid] : 0.0f;
  for (int i = tid; i < hidden; i += kClsThreads) ctrl->bias1[i] = pdg.bias1[i];
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = ctrl->tmem_base;
  const int kb_per_tile = kNumKBlocks * n_mma1 + n_kb2;  // B stages per unit

  if (warp == kLoaderWarp) {
    // ===================== loader: W1 K-blocks (this CTA's half of each N=256 slice), then W2
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_last();
      uint32_t itb = 0;
      for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step) {
        for (int kb = 0; kb < kb_per_tile; ++kb, ++itb) {
          const uint32_t s = itb % kMB, ph = (itb / kMB) & 1u;
          HYDRO_PIPE_WAIT(&ctrl->empty_b[s], ph ^ 1u);
          uint8_t* dst = smem + (b_ring - a_ring) + s * kMlpBStage;
          if (kb < kNumKBlocks * n_mma1) {  // W1 K-block kb / n_mma1, N slice kb % n_mma1
            const int k1 = kb / n_mma1, m = kb % n_mma1;
            mbar_arrive_expect_tx(&ctrl->full_b[s], 16384u);
            bulk_g2s_hint(dst, pdg.w_tiled + static_cast<uint64_t>(k1) * w1_kb + (m * 256 + crank * 128) * 128u, 16384u,
                          &ctrl->full_b[s], pol_w);
          } else {
            mbar_arrive_expect_tx(&ctrl->full_b[s], w2_load);
            bulk_g2s_hint(dst, pdg.w2_tiled + static_cast<uint64_t>(kb - kNumKBlocks * n_mma1) * w2_kb + crank * w2_load,
                          w2_load, &ctrl->full_b[s], pol_w);
          }
        }
      }
      for (int e = 0; e < kMB; ++e, ++itb) mbar_wait(&ctrl->empty_b[itb % kMB], ((itb / kMB) & 1u) ^ 1u);
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    if (crank != 0 && lane == 0) {
      // peer: relay "my half of the B stage landed" to the leader
      uint32_t itb = 0;
      for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step) {
        for (int kb = 0; kb < kb_per_tile; ++kb, ++itb) {
          const uint32_t s = itb % kMB;
          mbar_wait(&ctrl->full_b[s], (itb / kMB) & 1u);
          mbar_arrive_leader(&ctrl->full_b[s]);
        }
      }
    } else if (lane == 0) {
      // ===================== leader MMA issuer
      const uint32_t idesc1 = idesc_f16_f32(kTileM * kP, 256u, !fp16);
      const uint32_t idesc2 = idesc_f16_f32(kTileM * kP, static_cast<uint32_t>(n_pad), true);
      uint32_t itb = 0, gg = 0, tl = 0;
      for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step, ++tl) {
        mbar_wait_sleep(&ctrl->tempty[0], (tl & 1u) ^ 1u);  // previous unit's logits read out
        tc_fence_after();
        for (int g = 0; g < kGroups; ++g, ++gg) {
          const uint32_t set = (gg & 1u) * kKBlocksPerGroup, aph2 = (gg >> 1) & 1u;
#pragma unroll
          for (int kbr = 0; kbr < kKBlocksPerGroup; ++kbr) {
            const uint32_t sa = set + kbr;
            HYDRO_PIPE_WAIT(&ctrl->full_a[sa], aph2);
            const uint32_t a_addr = a_ring + sa * kAKBlockBytes;
            for (int m = 0; m < n_mma1; ++m, ++itb) {
              const uint32_t sb = itb % kMB, bph = (itb / kMB) & 1u;
              HYDRO_PIPE_WAIT(&ctrl->full_b[sb], bph);
              tc_fence_after();
              const uint32_t b_addr = b_ring + sb * kMlpBStage;
#pragma unroll
              for (int kk = 0; kk < kKBlock / 16; ++kk)
                tc_mma_pair(tmem_base + m * 256, desc_sw128(a_addr + kk * 32), desc_sw128(b_addr + kk * 32), idesc1,
                            (g | kbr | kk) != 0 ? 1u : 0u);
              tc_commit_pair(&ctrl->empty_b[sb]);
            }
            tc_commit_pair(&ctrl->empty_a[sa]);
          }
        }
        tc_commit_pair(&ctrl->tfull[0]);
        mbar_wait_sleep(&ctrl->hready, tl & 1u);  // bf16 hidden activations back in TMEM (both CTAs)
        tc_fence_after();
        for (int kb2 = 0; kb2 < n_kb2; ++kb2, ++itb) {
          const uint32_t sb = itb % kMB, bph = (itb / kMB) & 1u;
          HYDRO_PIPE_WAIT(&ctrl->full_b[sb], bph);
          tc_fence_after();
          const uint32_t b_addr = b_ring + sb * kMlpBStage;
#pragma unroll
          for (int kk = 0; kk < kKBlock / 16; ++kk)
            tc_mma_pair_ts(tmem_base + 256, tmem_base + kb2 * (kKBlock / 2) + kk * 8, desc_sw128(b_addr + kk * 32), idesc2,
                           (kb2 | kk) != 0 ? 1u : 0u);
          tc_commit_pair(&ctrl->empty_b[sb]);
        }
        tc_commit_pair(&ctrl->tfull2);
      }
    }
    __syncwarp();
  } else if (warp >= kConvWarp0) {
    converter_role<kDbg, false, kP, kQD>(p, ctrl, list_in, base, tw, crank, warp, lane,
                                         staging_addr, a_ring, row_pitch, false, fp16);
  } else {
    // ===================== epilogue warps 0..3 (TMEM lane quadrant = warp)
    const int q = warp;
    uint32_t n_in = 0, n_pass = 0, tl = 0;
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step, ++tl) {
      const uint32_t pos0 = tw.pos0(unit);
      mbar_wait_sleep(&ctrl->tfull[0], tl & 1u);
      tc_fence_after();
      // hidden: + b1, ReLU, bf16 RNE, packed pairs written back over the consumed fp32 columns
      for (int c0 = 0; c0 < hidden; c0 += 16) {
        uint32_t v[16], w[8];
        tc_ld_32x32b_x16(taddr + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float lo = fmaxf(__uint_as_float(v[2 * t]) + ctrl->bias1[c0 + 2 * t], 0.0f);
          const float hi = fmaxf(__uint_as_float(v[2 * t + 1]) + ctrl->bias1[c0 + 2 * t + 1], 0.0f);
          w[t] = bf16x2_rn(lo, hi);
        }
        tc_st_32x32b_x8(taddr + c0 / 2, w);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (crank != 0) mbar_arrive_leader(&ctrl->hready);
        else mbar_arrive(&ctrl->hready);
      }
      mbar_wait_sleep(&ctrl->tfull2, tl & 1u);
      tc_fence_after();
      const int m = q * 32 + lane;
      const uint32_t pos = pos0 + m;
      const bool valid = pos < tw.lim;
      float best = -3.402823466e38f;
      int bi = 0;
      for (int c0 = 0; c0 < n_pad; c0 += 16) {
        uint32_t v[16];
        tc_ld_32x32b_x16(taddr + 256 + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int c = c0 + jj;
          if (c < n_classes) {
            const float z = __uint_as_float(v[jj]) + ctrl->bias[c];
            if (z > best) {  // strict: lowest index wins ties (R12)
              best = z;
              bi = c;
            }
            if (kDbg && p.dbg_logits && valid) p.dbg_logits[static_cast<uint64_t>(pos) * n_classes + c] = z;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (crank != 0) mbar_arrive_leader(&ctrl->tempty[0]);
        else mbar_arrive(&ctrl->tempty[0]);
      }
      const bool verdict = valid && (bi == target);
      const uint32_t bv = __ballot_sync(0xFFFFFFFFu, verdict);
      const uint32_t bvalid = __ballot_sync(0xFFFFFFFFu, valid);
      cls_emit(p, bits_out, ind, list_in, base, pos0 + q * 32, pos, valid, verdict, pdg, fill);
      if (kDbg && p.dbg_verdict && valid) p.dbg_verdict[pos] = verdict ? 1 : 0;
      n_in += __popc(bvalid);
      n_pass += __popc(bv);
    }
    if (p.collect_stats && lane == 0) {
      atomicAdd(&st->d_in[pred], static_cast<unsigned long long>(n_in));
      atomicAdd(&st->d_pass[pred], static_cast<unsigned long long>(n_pass));
      atomicAdd(&st->d_comp[pred], static_cast<unsigned long long>(n_in));  // no verdict cache here
    }
    if (lane == 0) atomicAdd(&st->kt_items[4], static_cast<unsigned long long>(n_in));
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols) : "memory");
  }
  if (tid == 0 && p.collect_stats) {
    atomicAdd(&st->d_cost[pred], static_cast<unsigned long long>(clock64() - t_start));
  }
  if (tid == 0) ktimer_end(st, 4);
}

// ------------------------------------------------------------------------------------------
// K4-T `hydro_classifier_tm_kernel` (nearest crops): the same warp roles and weight
// stream as hydro_classifier_kernel, but the A operand lives in TENSOR MEMORY.  Converter warps
// write their crop pixels with tcgen05.st (16x256b: thread t owns TMEM lanes t/4 and t/4 + 8 of
// its 16-row band, 2 columns per 8-column repetition) into a 2-group TMEM ring (columns
// [a_col0, 512), 3-4 crop rows of 96 columns); the MMA reads A from TMEM (tcgen05.mma ... [d], [a], b_desc),
// so neither the A stores nor the tensor core's A reads touch shared memory, and the 96 KB the
// shared-memory A ring took become crop-row staging: each converter warp owns a 22 KB ring of
// "units" (one crop row of its 16 tuples, segments packed back to back) and stages up to 3 units
// ahead instead of 2 quads.
// Converter warp cu owns tile rows [32*((6+cu)%4) + 16*(cu/4), +16) (the TMEM lane quarter of
// warp 6+cu).  Thread t handles local tuples a = t/4 and a + 8, output pixels dx = 4k + (t%4)
// (k = 0..15) of every crop row; K order inside a crop row = crop_pos_feature_tm.
constexpr int kTmASlots = 4;  // crop rows of A in TMEM at most: 4 when the accumulators fit in 128
                               // columns (N <= 128, or two buffers of N <= 64), else 3 (a fused pair)
constexpr int kTmGroupCols = 96;   // one crop row of A: 192 fp16 = 96 32-bit columns per lane
#ifndef HYDRO_TM_SLOTS
#define HYDRO_TM_SLOTS 3
#endif
constexpr int kTmMaxSlots = HYDRO_TM_SLOTS;
#ifdef HYDRO_TM_CPASYNC
constexpr bool kTmBulk = false;  // stage crop rows with per-lane 16-byte cp.async (A/B variant)
#else
constexpr bool kTmBulk = true;   // stage crop rows with one 1-D bulk copy per row segment
#endif  // staging units per converter warp (depth <= slots - 1)
constexpr int kTmBStages = 3;
struct TmCtrl {
  uint64_t stg[kConvWarps][kTmMaxSlots];  // staging units landed (bulk copies, complete_tx)
  uint64_t full_a[kTmASlots], empty_a[kTmASlots];
  uint64_t full_b[kTmBStages], empty_b[kTmBStages];
  uint64_t tfull[2], tempty[2];
  uint32_t tmem_base;
  uint32_t pad;
  float bias[144];
};
constexpr int kTmBStageBytes = 144 * 128;  // one weight K-block of N <= 144 rows (a fused pair: 128 + 16)
constexpr int kTmBRingBytes = kTmBStages * kTmBStageBytes;
constexpr int kTmCtrlBytes = (static_cast<int>(sizeof(TmCtrl)) + 127) & ~127;
// per-warp staging ring (16-byte multiple) + 64 B of slack at the end of the region (reads of the
// word after a pixel, and of stale offsets in invalid rows, stay inside the allocation)
constexpr int kTmWarpStage = ((kClsSmemBytes - 1023 - kTmBRingBytes - kTmCtrlBytes - 64) / kConvWarps) & ~15;
static_assert(kTmWarpStage >= 16 * 784, "one unit of 16 worst-case segments must fit a converter ring");

__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_st_16x256b_x4(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tc_st_16x256b_x2(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}


// 8 staged pixels (byte offsets packed 2 per word, relative to `unit`) -> 12 words of fp16x2 (or
// bf16x2) in feature order f = 3 * pixel + ch
template <bool kFp16>
__device__ __forceinline__ void tm_convert8(uint32_t unit, const uint32_t (&po)[4], uint32_t (&e)[12], uint32_t (&px)[8]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const uint32_t o = h2 ? (po[q] >> 16) : (po[q] & 0xFFFFu);
      const uint32_t a = unit + (o & ~3u);
      px[2 * q + h2] = __funnelshift_r(lds32(a), lds32(a + 4), o << 3);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t p0 = px[2 * q], p1 = px[2 * q + 1];
    if (kFp16) {
      const uint32_t K = 0x64646464u;  // fp16 0x64vv == 1024 + v exactly
      e[3 * q + 0] = f16x2_sub(__byte_perm(p0, K, 0x4140), 0x64006400u);
      e[3 * q + 1] = f16x2_sub(__byte_perm(__byte_perm(p0, p1, 0x0042), K, 0x4140), 0x64006400u);
      e[3 * q + 2] = f16x2_sub(__byte_perm(p1, K, 0x4241), 0x64006400u);
    } else {
      e[3 * q + 0] = bf16x2_of_bytes(p0 & 0xFF, (p0 >> 8) & 0xFF);
      e[3 * q + 1] = bf16x2_of_bytes((p0 >> 16) & 0xFF, p1 & 0xFF);
      e[3 * q + 2] = bf16x2_of_bytes((p1 >> 8) & 0xFF, (p1 >> 16) & 0xFF);
    }
  }
}

__device__ __forceinline__ void tm_wait_depth(uint32_t d) {
  // cp.async.wait_group needs an immediate: the runtime depth of this tile picks the case
  if (d >= 5) cp_async_wait<5>();
  else if (d == 4) cp_async_wait<4>();
  else if (d == 3) cp_async_wait<3>();
  else if (d == 2) cp_async_wait<2>();
  else if (d == 1) cp_async_wait<1>();
  else cp_async_wait<0>();
}

template <bool kDbg, bool kWide>
__device__ __forceinline__ void tm_convert_tile(const ClsParams& p, TmCtrl* ctrl, uint32_t lim, uint32_t pos0, int cu,
                                                int lane, uint32_t ring, uint32_t tmem_base, uint32_t row_pitch,
                                                bool fp16, const RowMeta& mm, uint32_t band, uint32_t& gg,
                                                uint32_t& stg_par, uint32_t a_slots, uint32_t a_col0) {
  const uint8_t* frames = p.frames;
  const int a = lane >> 2, t0 = lane & 3;
  // unit layout: the segments of local tuples 0..15 back to back (lane l < 16 holds tuple l)
  const bool my_wide = kWide && lane < 16 && mm.valid && mm.seg_len > static_cast<uint32_t>(kMaxSegBytes);
  const uint32_t slen = (lane < 16 && mm.valid) ? (my_wide ? 512u : mm.seg_len) : 0u;
  uint32_t incl = slen;
#pragma unroll
  for (int d = 1; d < 16; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += v;
  }
  const uint32_t soff = incl - slen;
  const uint32_t ubytes = max(__shfl_sync(0xFFFFFFFFu, incl, 15), 16u);
  const uint32_t nslot = min(static_cast<uint32_t>(kTmMaxSlots), static_cast<uint32_t>(kTmWarpStage) / ubytes);
  const uint32_t depth = nslot - 1u;
  // this thread's pixel offsets inside a unit: tuples a (tt = 0) and a + 8 (tt = 1), pixels 4k + t0
  uint32_t po[2][8];
#pragma unroll
  for (int tt = 0; tt < 2; ++tt) {
    const int src = a + 8 * tt;
    const uint32_t x0 = __shfl_sync(0xFFFFFFFFu, static_cast<uint32_t>(mm.x0), src);
    const uint32_t w = __shfl_sync(0xFFFFFFFFu, static_cast<uint32_t>(mm.w), src);
    const uint32_t slo = __shfl_sync(0xFFFFFFFFu, mm.seg_lo, src);
    const uint32_t so = __shfl_sync(0xFFFFFFFFu, soff, src);
    const bool wide = kWide && __shfl_sync(0xFFFFFFFFu, my_wide, src);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      const uint32_t dx0 = 8u * k2 + t0, dx1 = dx0 + 4u;  // pixels k = 2*k2, 2*k2 + 1
      const uint32_t b0 = 3u * (x0 + (((2u * dx0 + 1u) * w) >> 7)), b1 = 3u * (x0 + (((2u * dx1 + 1u) * w) >> 7));
      const uint32_t o0 = so + (wide ? 8u * dx0 + (b0 & 3u) : b0 - slo);
      const uint32_t o1 = so + (wide ? 8u * dx1 + (b1 & 3u) : b1 - slo);
      po[tt][k2] = o0 | (o1 << 16);
    }
  }
  // staging: lanes (r = lane/8, j = lane%8) copy segment 4*pass + r in 16-byte chunks j + 8c
  const int r = lane >> 3, j = lane & 7;
  const uint32_t my_src = mm.row16 + (mm.seg_lo >> 4);  // 16-byte units
  const uint32_t my_h = static_cast<uint32_t>(mm.h);
  const uint32_t my_lo = slen | (soff << 16);
  const uint32_t my_xw =
      kWide ? static_cast<uint32_t>(mm.x0) | (static_cast<uint32_t>(mm.w) << 16) | (my_wide ? 0x80000000u : 0u) : 0u;
  const uint32_t utot = __shfl_sync(0xFFFFFFFFu, incl, 15);  // bytes of one unit (0: no valid tuple)
  auto stage_unit = [&](int g, uint32_t slot) {
    if (kTmBulk && !kWide) {
      // one 1-D bulk copy (TMA engine) per row segment, completion counted on the slot's mbarrier:
      // the shared-memory writes bypass the LSU pipe the pixel loads use
      if (g < kGroups) {
        uint64_t* bar = &ctrl->stg[cu][slot];
        if (lane == 0) mbar_arrive_expect_tx(bar, utot);
        __syncwarp();
        if (slen != 0) {
          const uint8_t* row = at16(frames, my_src) + (((2u * g + 1u) * my_h) >> 7) * row_pitch;
          bulk_g2s_u32(ring + slot * ubytes + soff, row, slen, bar);
        }
      }
      return;
    }
    if (g < kGroups) {
      const uint32_t dst0 = ring + slot * ubytes;
#pragma unroll
      for (int pass = 0; pass < 4; ++pass) {
        const int L = 4 * pass + r;
        const uint32_t lo = __shfl_sync(0xFFFFFFFFu, my_lo, L);
        const uint32_t off = __shfl_sync(0xFFFFFFFFu, my_src, L);
        const uint32_t h = __shfl_sync(0xFFFFFFFFu, my_h, L);
        const uint32_t xw = kWide ? __shfl_sync(0xFFFFFFFFu, my_xw, L) : 0u;
        const uint32_t len = lo & 0xFFFFu;
        const uint8_t* row = at16(frames, off) + (((2u * g + 1u) * h) >> 7) * row_pitch;
        const uint32_t dst = dst0 + (lo >> 16);
        if (!kWide || !(xw >> 31)) stage_segment(dst, row, j, len >> 4);
        else stage_wide_row(dst, row, xw & 0x7FFFFFFFu, j);  // wide crop (rare): 64-pixel gather
      }
    }
    cp_async_commit();  // one group per unit (possibly empty) keeps wait_group counting uniform
  };
  uint32_t slot_stage = 0, slot_use = 0;
  for (uint32_t k = 0; k < depth; ++k) {
    stage_unit(static_cast<int>(k), slot_stage);
    slot_stage = slot_stage + 1 == nslot ? 0 : slot_stage + 1;
  }
  const uint32_t lane_addr = tmem_base + (band << 16) + a_col0;
  for (int g = 0; g < kGroups; ++g, ++gg) {
    stage_unit(g + static_cast<int>(depth), slot_stage);
    slot_stage = slot_stage + 1 == nslot ? 0 : slot_stage + 1;
    if (!kTmBulk || kWide) {
      tm_wait_depth(depth);  // this thread's copies of unit g have landed
      __syncwarp();          // ... and every lane's
    } else {
      mbar_wait(&ctrl->stg[cu][slot_use], (stg_par >> slot_use) & 1u);  // unit g's bulk copies landed
      stg_par ^= 1u << slot_use;
    }
    const uint32_t sa = gg % a_slots, aph = (gg / a_slots) & 1u;
    mbar_wait(&ctrl->empty_a[sa], aph ^ 1u);  // the MMA has consumed group gg - a_slots from this slot
    tc_fence_after();
    const uint32_t unit = ring + slot_use * ubytes;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      uint32_t ea[12], eb[12], pa[8], pb[8];
      const uint32_t qa[4] = {po[0][4 * hh], po[0][4 * hh + 1], po[0][4 * hh + 2], po[0][4 * hh + 3]};
      const uint32_t qb[4] = {po[1][4 * hh], po[1][4 * hh + 1], po[1][4 * hh + 2], po[1][4 * hh + 3]};
      if (fp16) {
        tm_convert8<true>(unit, qa, ea, pa);
        tm_convert8<true>(unit, qb, eb, pb);
      } else {
        tm_convert8<false>(unit, qa, ea, pa);
        tm_convert8<false>(unit, qb, eb, pb);
      }
      const uint32_t taddr = lane_addr + sa * kTmGroupCols + 48u * hh;
      const uint32_t v4[16] = {ea[0], ea[1], eb[0], eb[1], ea[2], ea[3], eb[2], eb[3],
                               ea[4], ea[5], eb[4], eb[5], ea[6], ea[7], eb[6], eb[7]};
      const uint32_t v2[8] = {ea[8], ea[9], eb[8], eb[9], ea[10], ea[11], eb[10], eb[11]};
      tc_st_16x256b_x4(taddr, v4);
      tc_st_16x256b_x2(taddr + 32u, v2);
      if (kDbg && p.dbg_crops) {
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          const uint32_t m = band + static_cast<uint32_t>(a + 8 * tt);  // tile row
          if (pos0 + m < lim) {
            uint16_t* dbg = p.dbg_crops + static_cast<uint64_t>(pos0 + m) * kFeatures + g * 192;
            const uint32_t (&px)[8] = tt ? pb : pa;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t dx = 4u * (8u * hh + kk) + t0;
#pragma unroll
              for (int ch = 0; ch < 3; ++ch)
                dbg[3 * dx + ch] = static_cast<uint16_t>(bf16_bits_of_byte((px[kk] >> (8 * ch)) & 0xFF));
            }
          }
        }
      }
    }
    slot_use = slot_use + 1 == nslot ? 0 : slot_use + 1;
    tc_wait_st();  // this thread's TMEM stores have completed
    tc_fence_before();
    __syncwarp();  // every lane's stores (and smem reads of the unit) are done
    if (lane == 0) mbar_arrive(&ctrl->full_a[sa]);
  }
  if (!kTmBulk || kWide) cp_async_wait<0>();
}

extern __shared__ __align__(1024) uint8_t hydro_tm_smem[];

template <bool kDbg>
__global__ void __launch_bounds__(kClsThreads, 1) hydro_classifier_tm_kernel(ClsParams p) {
  DevState* st = p.st;
  int pred;
  const uint32_t* list_in;
  uint32_t count, base = p.range_base;
  uint32_t* bits_out;
  int pred2 = -1;  // fused pair hop: the second head (order position h + 1)
  if (p.dispatch) {
    const int h = st->sched[p.hop];
    if (h < 0 || h >= st->n_pred) return;
    pred = st->order[h];
    if (st->kind[pred] != kLinear) return;
    if (p.pair_w_tiled && is_pair_hop(st->order, st->n_pred, h, st->pair_a, st->pair_b)) pred2 = st->order[h + 1];
    if (h == 0) {
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
  // cached classifier hop: only the uncached tuples (K0c's list), verdict bits by hop position
  if (p.preds[pred].crop_mode != HYDRO_CROP_NEAREST) return;  // AREA hops run in K4 (launched beside)
  const uint32_t* ind = cls_redirect(p, p.preds[pred], list_in, count);
  const bool fill = p.preds[pred].cache_known && (p.preds[pred].cache_fill || p.force_fill);
  const uint32_t num_tiles = (count + kTileM - 1) / kTileM;
  const PredDev& pdg = p.preds[pred];
  TileWalk tw{blockIdx.x, gridDim.x, num_tiles, 0u, count, 1u, 0u, false};
  if (threadIdx.x == 0) ktimer_begin(st, 1);
  if (tw.first >= tw.end) {
    if (threadIdx.x == 0) ktimer_end(st, 1);
    return;
  }
  const long long t_start = clock64();
  // a fused pair hop contracts with both heads' weights at once: head pair_a in columns
  // [0, pair_npa), head pair_b after them (one crop gather, N = pair_n_pad)
  const bool pair = pred2 >= 0;
  const int n_classes = pdg.n_classes, target = pdg.target;
  const int n_pad = pair ? p.pair_n_pad : pdg.n_pad;
  const bool fp16 = pdg.a_fp16 != 0;
  const float unscale = pdg.w_unscale;
  const uint8_t* w_tiled = pair ? p.pair_w_tiled : pdg.w_tiled_tm;
  const uint32_t n_alloc = n_pad <= 32 ? 32u : (n_pad <= 64 ? 64u : (n_pad <= 128 ? 128u : static_cast<uint32_t>(n_pad)));
  const uint32_t n_acc = 2u * n_alloc <= 128u ? 2u : 1u;  // accumulator buffers below the A ring
  // A ring: 4 crop rows when the accumulators fit in 128 columns, else 3
  const uint32_t a_slots = n_acc * n_alloc <= 128u ? 4u : 3u;
  const uint32_t a_col0 = 512u - a_slots * kTmGroupCols;
  const uint32_t b_stage_bytes = static_cast<uint32_t>(n_pad) * 128u;
  const uint32_t row_pitch = static_cast<uint32_t>(p.frame_w * 3);

  // shared memory: [B ring 3 x 16 KB][ctrl][8 converter staging rings]
  const uint32_t raw = smem_u32(hydro_tm_smem);
  uint8_t* smem = hydro_tm_smem + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t b_ring = smem_u32(smem);
  TmCtrl* ctrl = reinterpret_cast<TmCtrl*>(smem + kTmBRingBytes);
  const uint32_t stage0 = b_ring + kTmBRingBytes + kTmCtrlBytes;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kTmASlots; ++s) {
      mbar_init(&ctrl->full_a[s], kConvWarps);
      mbar_init(&ctrl->empty_a[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctrl->tfull[s], 1);
      mbar_init(&ctrl->tempty[s], kEpiWarps);
    }
    for (int s = 0; s < kTmBStages; ++s) {
      mbar_init(&ctrl->full_b[s], 1);
      mbar_init(&ctrl->empty_b[s], 1);
    }
    for (int w = 0; w < kConvWarps; ++w)
      for (int s = 0; s < kTmMaxSlots; ++s) mbar_init(&ctrl->stg[w][s], 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&ctrl->tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (pair) {
    if (tid < n_pad) ctrl->bias[tid] = p.pair_bias[tid];
  } else if (tid < HYDRO_MAX_CLASSES) {
    ctrl->bias[tid] = tid < n_classes ? pdg.bias[tid] : 0.0f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = ctrl->tmem_base;

  if (warp == kLoaderWarp) {
    // ===================== loader: weight K-blocks (1-D bulk copies, L2 evict_last)
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_last();
      uint32_t itb = 0;
      for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step) {
        for (int kb = 0; kb < kNumKBlocks; ++kb, ++itb) {
          const uint32_t s = itb % kTmBStages, ph = (itb / kTmBStages) & 1u;
          HYDRO_PIPE_WAIT(&ctrl->empty_b[s], ph ^ 1u);
          mbar_arrive_expect_tx(&ctrl->full_b[s], b_stage_bytes);
          bulk_g2s_hint(smem + s * kTmBStageBytes, w_tiled + static_cast<uint64_t>(kb) * b_stage_bytes, b_stage_bytes,
                        &ctrl->full_b[s], pol_w);
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer: A from TMEM, B from the shared-memory ring
    if (lane == 0) {
      const uint32_t idesc = idesc_f16_f32(kTileM, static_cast<uint32_t>(n_pad), !fp16);
      uint32_t itb = 0, gg = 0, tl = 0;
      for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step, ++tl) {
        const uint32_t acc = tl % n_acc, aph = (tl / n_acc) & 1u;
        mbar_wait_backoff<256>(&ctrl->tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * n_alloc;
        for (int g = 0; g < kGroups; ++g, ++gg) {
          const uint32_t sa = gg % a_slots;
          HYDRO_PIPE_WAIT(&ctrl->full_a[sa], (gg / a_slots) & 1u);
          tc_fence_after();
          const uint32_t a_col = tmem_base + a_col0 + sa * kTmGroupCols;
#pragma unroll
          for (int kbr = 0; kbr < kKBlocksPerGroup; ++kbr, ++itb) {
            const uint32_t sb = itb % kTmBStages, bph = (itb / kTmBStages) & 1u;
            HYDRO_PIPE_WAIT(&ctrl->full_b[sb], bph);
            tc_fence_after();
            const uint32_t b_addr = b_ring + sb * static_cast<uint32_t>(kTmBStageBytes);
#pragma unroll
            for (int kk = 0; kk < kKBlock / 16; ++kk)
              tc_mma_ts(d_tmem, a_col + (kbr * 4 + kk) * 8, desc_sw128(b_addr + kk * 32), idesc,
                        (g | kbr | kk) != 0 ? 1u : 0u);
            tc_commit(&ctrl->empty_b[sb]);
          }
          tc_commit(&ctrl->empty_a[sa]);
        }
        tc_commit(&ctrl->tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= kConvWarp0) {
    // ===================== converters
    const int cu = warp - kConvWarp0;
    const uint32_t band = 32u * static_cast<uint32_t>(warp & 3) + 16u * static_cast<uint32_t>(cu >> 2);
    const uint32_t ring = stage0 + static_cast<uint32_t>(cu) * kTmWarpStage;
    uint32_t gg = 0, stg_par = 0;
    for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step) {
      const uint32_t pos0 = tw.pos0(unit);
      const RowMeta mm = load_meta(p, list_in, base, pos0 + band + (lane & 15), lane < 16 ? tw.lim : 0u);
      const bool any_wide =
          __any_sync(0xFFFFFFFFu, lane < 16 && mm.valid && mm.seg_len > static_cast<uint32_t>(kMaxSegBytes));
      if (any_wide)
        tm_convert_tile<kDbg, true>(p, ctrl, tw.lim, pos0, cu, lane, ring, tmem_base, row_pitch, fp16, mm, band, gg,
                                    stg_par, a_slots, a_col0);
      else
        tm_convert_tile<kDbg, false>(p, ctrl, tw.lim, pos0, cu, lane, ring, tmem_base, row_pitch, fp16, mm, band, gg,
                                     stg_par, a_slots, a_col0);
    }
  } else {
    // ===================== epilogue warps 0..3 (TMEM lane quadrant = warp)
    const int q = warp;
    uint32_t n_in = 0, n_pass = 0, tl = 0;
    // fused pair: head pair_a in columns [0, pair_npa), pair_b after; n_p1 = survivors of the first
    const int pnpa = p.pair_npa;
    const int pca = pair ? p.preds[st->pair_a].n_classes : 0, pcb = pair ? p.preds[st->pair_b].n_classes : 0;
    const int pta = pair ? p.preds[st->pair_a].target : 0, ptb = pair ? p.preds[st->pair_b].target : 0;
    const float pua = p.pair_unscale_a, pub = p.pair_unscale_b;
    const bool first_is_a = pair && pred == st->pair_a;
    uint32_t n_p1 = 0;
    for (uint32_t unit = tw.first; unit < tw.end; unit += tw.step, ++tl) {
      const uint32_t pos0 = tw.pos0(unit);
      const uint32_t acc = tl % n_acc, aph = (tl / n_acc) & 1u;
      mbar_wait_backoff<1024>(&ctrl->tfull[acc], aph);
      tc_fence_after();
      const int m = q * 32 + lane;
      const uint32_t pos = pos0 + m;
      const bool valid = pos < tw.lim;
      float best = -3.402823466e38f, best2 = -3.402823466e38f;
      int bi = 0, bi2 = 0;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * n_alloc;
      for (int c0 = 0; c0 < n_pad; c0 += 16) {
        uint32_t v[16];
        tc_ld_32x32b_x16(taddr + c0, v);
        tc_wait_ld();
        if (!pair || c0 < pnpa) {  // (the single head, or pair head pair_a: columns [0, pair_npa))
          const int nc = pair ? pca : n_classes;
          const float us = pair ? pua : unscale;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const int c = c0 + jj;
            if (c < nc) {
              const float z = __uint_as_float(v[jj]) * us + ctrl->bias[c];  // 2^-k: exact
              if (z > best) {  // strict: lowest index wins ties (R12)
                best = z;
                bi = c;
              }
              if (kDbg && p.dbg_logits && valid) p.dbg_logits[static_cast<uint64_t>(pos) * n_classes + c] = z;
            }
          }
        } else {  // pair head pair_b: columns [pair_npa, pair_npa + C_b)
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const int c = c0 + jj - pnpa;
            if (c < pcb) {
              const float z = __uint_as_float(v[jj]) * pub + ctrl->bias[c0 + jj];
              if (z > best2) {
                best2 = z;
                bi2 = c;
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->tempty[acc]);
      bool verdict = valid && (bi == target);
      if (pair) {  // verdicts of pair_a and pair_b -> the order's first and second head
        const bool va = valid && bi == pta, vb = valid && bi2 == ptb;
        const bool v1 = first_is_a ? va : vb, v2 = first_is_a ? vb : va;
        n_p1 += __popc(__ballot_sync(0xFFFFFFFFu, v1));
        verdict = v1 && v2;  // the hop's survivors pass both heads
      }
      const uint32_t bv = __ballot_sync(0xFFFFFFFFu, verdict);
      const uint32_t bvalid = __ballot_sync(0xFFFFFFFFu, valid);
      cls_emit(p, bits_out, ind, list_in, base, pos0 + q * 32, pos, valid, verdict, pdg, fill);
      if (kDbg && p.dbg_verdict && valid) p.dbg_verdict[pos] = verdict ? 1 : 0;
      n_in += __popc(bvalid);
      n_pass += __popc(bv);
    }
    if (p.collect_stats && lane == 0) {
      if (pair) {  // as if evaluated in turn: the second head sees the first head's survivors
        atomicAdd(&st->d_in[pred], static_cast<unsigned long long>(n_in));
        atomicAdd(&st->d_pass[pred], static_cast<unsigned long long>(n_p1));
        atomicAdd(&st->d_comp[pred], static_cast<unsigned long long>(n_in));
        atomicAdd(&st->d_in[pred2], static_cast<unsigned long long>(n_p1));
        atomicAdd(&st->d_pass[pred2], static_cast<unsigned long long>(n_pass));
        atomicAdd(&st->d_comp[pred2], static_cast<unsigned long long>(n_p1));
      } else {
        atomicAdd(&st->d_in[pred], static_cast<unsigned long long>(n_in));
        atomicAdd(&st->d_pass[pred], static_cast<unsigned long long>(n_pass));
        atomicAdd(&st->d_comp[pred], static_cast<unsigned long long>(n_in));
      }
    }
    if (lane == 0) atomicAdd(&st->kt_items[1], static_cast<unsigned long long>(n_in));
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
  if (tid == 0 && p.collect_stats) {
    const unsigned long long cyc = static_cast<unsigned long long>(clock64() - t_start);
    if (pair) {  // the CTA's cycles split between the two heads by their share of the N columns
      const uint32_t n_first = pred == st->pair_a ? static_cast<uint32_t>(p.pair_npa)
                                                  : static_cast<uint32_t>(n_pad - p.pair_npa);
      const unsigned long long c1 = cyc * n_first / static_cast<uint32_t>(n_pad);
      atomicAdd(&st->d_cost[pred], c1);
      atomicAdd(&st->d_cost[pred2], cyc - c1);
    } else {
      atomicAdd(&st->d_cost[pred], cyc);
    }
  }
  if (tid == 0) ktimer_end(st, 1);
}

// ------------------------------------------------------------------------------------------
// K0c: verdict-cache split of a classifier hop (reuse-aware routing on expensive UDFs, PAPER.md:
// 589-605; R26).  Exits unless the chain slot's hop is a classifier whose predicate has a cache.
// One warp per 32 hop-input positions: cached verdicts go straight into the hop's bitmap word
// (and the survivor counts); the uncached tuples are appended (warp-aggregated atomic) to the
// list the classifier kernel evaluates next.  Cache hits count as routed and passed, never as
// computed or charged (R26).
__global__ void __launch_bounds__(256) hydro_cache_split_kernel(ClsParams p) {
  DevState* st = p.st;
  const int h = st->sched[p.hop];
  if (h < 0 || h >= st->n_pred) return;
  const int pred = st->order[h];
  if (!is_classifier(st->kind[pred])) return;
  const PredDev& pd = p.preds[pred];
  if (!pd.cache_known) return;
  const uint32_t* list_in;
  uint32_t count;
  const uint32_t base = p.range_base;
  if (h == 0) {
    list_in = p.sel0;
    count = p.sel0 ? *p.sel0_count : p.range_n;
  } else {
    list_in = p.lists + static_cast<uint64_t>(h) * p.list_stride;
    count = p.counts[h];
  }
  uint32_t* bits_out = p.bits + static_cast<uint64_t>(h) * p.bits_stride;
  const int lane = threadIdx.x & 31;
  const uint32_t words = (count + 31) / 32;
  uint32_t n_hit = 0, n_hit_pass = 0;
  for (uint32_t wi = (blockIdx.x * blockDim.x + threadIdx.x) / 32; wi < words; wi += (gridDim.x * blockDim.x) / 32) {
    const uint32_t pos = wi * 32 + lane;
    const bool valid = pos < count;
    uint32_t idx = 0;
    bool known = false, pass = false;
    if (valid) {
      idx = list_in ? __ldg(list_in + pos) : base + pos;
      const uint64_t id = __ldg(p.id + idx);
      if (id < pd.cache_cap) {
        known = (__ldg(pd.cache_known + (id >> 5)) >> (id & 31)) & 1u;
        pass = known && ((__ldg(pd.cache_pass + (id >> 5)) >> (id & 31)) & 1u);
      }
    }
    const uint32_t vb = __ballot_sync(0xFFFFFFFFu, pass);
    const uint32_t kb = __ballot_sync(0xFFFFFFFFu, known);
    const uint32_t ub = __ballot_sync(0xFFFFFFFFu, valid && !known);
    if (lane == 0) {
      bits_out[wi] = vb;  // the classifier ORs the computed verdicts in
      if (vb) {
        atomicAdd(p.seg_counts + (wi * 32) / kRouteTile, static_cast<uint32_t>(__popc(vb)));
        atomicAdd(p.warp_counts + (wi * 32) / kWarpSeg, static_cast<uint32_t>(__popc(vb)));
      }
    }
    uint32_t at = 0;
    if (lane == 0 && ub) at = atomicAdd(p.cache_count, static_cast<uint32_t>(__popc(ub)));
    at = __shfl_sync(0xFFFFFFFFu, at, 0);
    if (valid && !known) {
      const uint32_t r = at + static_cast<uint32_t>(__popc(ub & ((1u << lane) - 1u)));
      p.cache_idx[r] = idx;
      p.cache_pos[r] = pos;
    }
    n_hit += __popc(kb);
    n_hit_pass += __popc(vb);
  }
  if (p.collect_stats && lane == 0 && n_hit) {
    atomicAdd(&st->d_in[pred], static_cast<unsigned long long>(n_hit));
    atomicAdd(&st->d_pass[pred], static_cast<unsigned long long>(n_hit_pass));
  }
}

// Host-side entry points (the kernel templates stay inside this translation unit).
cudaError_t hydro_classifier_configure() {
  void (*ks[])(ClsParams) = {hydro_classifier_kernel<false, false>, hydro_classifier_kernel<true, false>,
                             hydro_classifier_kernel<false, true>, hydro_classifier_kernel<true, true>,
                             hydro_classifier_kernel<false, true, kAreaWarps>, hydro_classifier_kernel<true, true, kAreaWarps>,
                             hydro_mlp_kernel<false>, hydro_mlp_kernel<true>,
                             hydro_classifier_tm_kernel<false>, hydro_classifier_tm_kernel<true>};
  for (auto k : ks) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kClsSmemBytes);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

namespace {
// CTA-pair launch: grid = 2 x min(pairs of tiles, co-resident clusters of this kernel)
void launch_pairs(void (*k)(ClsParams), int* max_clusters, const ClsParams& c, int grid, cudaStream_t stream) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kClsThreads);
  cfg.dynamicSmemBytes = kClsSmemBytes;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (*max_clusters == 0) {
    cfg.gridDim = dim3(2 * 74);
    if (cudaOccupancyMaxActiveClusters(max_clusters, k, &cfg) != cudaSuccess || *max_clusters < 1) *max_clusters = 1;
    if (getenv("HYDRO_DEBUG_LAUNCH")) fprintf(stderr, "hydro: K4 CTA pairs, %d co-resident clusters\n", *max_clusters);
  }
  const int pairs = std::min((grid + 1) / 2, *max_clusters);
  cfg.gridDim = dim3(2 * pairs);
  cudaLaunchKernelEx(&cfg, k, c);
}
}  // namespace

void hydro_classifier_launch(const ClsParams& c, int grid, cudaStream_t stream, bool debug, bool area) {
  if (kPair == 1 && area && c.area_only) {  // AREA hops only: the instance with 12 converter warps
    void (*ka)(ClsParams) = debug ? hydro_classifier_kernel<true, true, kAreaWarps>
                                  : hydro_classifier_kernel<false, true, kAreaWarps>;
    ka<<<grid, (kConvWarp0 + kAreaWarps) * 32, kClsSmemBytes, stream>>>(c);
    return;
  }
  void (*k)(ClsParams) = area ? (debug ? hydro_classifier_kernel<true, true> : hydro_classifier_kernel<false, true>)
                              : (debug ? hydro_classifier_kernel<true, false> : hydro_classifier_kernel<false, false>);
  if constexpr (kPair == 2) {
    static int max_clusters = 0;
    launch_pairs(k, &max_clusters, c, grid, stream);
  } else {
    k<<<grid, kClsThreads, kClsSmemBytes, stream>>>(c);
  }
}

void hydro_classifier_tm_launch(const ClsParams& c, int grid, cudaStream_t stream, bool debug) {
  if (debug) hydro_classifier_tm_kernel<true><<<grid, kClsThreads, kClsSmemBytes, stream>>>(c);
  else hydro_classifier_tm_kernel<false><<<grid, kClsThreads, kClsSmemBytes, stream>>>(c);
}

void hydro_cache_split_launch(const ClsParams& c, uint64_t max_positions, int num_sms, cudaStream_t stream) {
  const uint64_t warps = (max_positions + 31) / 32;
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, static_cast<uint64_t>(num_sms) * 8));
  hydro_cache_split_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(c);
}

void hydro_mlp_launch(const ClsParams& c, int grid, cudaStream_t stream, bool debug) {
  static int max_clusters = 0;
  launch_pairs(debug ? hydro_mlp_kernel<true> : hydro_mlp_kernel<false>, &max_clusters, c, grid, stream);
}
