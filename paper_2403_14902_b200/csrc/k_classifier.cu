// K4: fused Crop(frame, bbox) -> 64x64 resize gather -> bf16 linear-head GEMM on tcgen05 tensor
// cores -> argmax verdict (readings R10-R14, R19 in DESIGN.md §2).
//
// One persistent CTA per SM walks M-tiles of 128 alive tuples.  Per tile the K = 12288 features
// are streamed as 64 crop rows ("groups"); a group is one 64-pixel crop row x 3 channels =
// 3 UMMA K-blocks of 64 bf16.  Warp roles:
//   warps 0-3  epilogue: tcgen05.ld the fp32 accumulator (TMEM lane = tuple), + bias, argmax,
//              verdict ballot -> bitmap, pass counters
//   warp  4    loader: 1-D bulk copy (TMA engine) of the pre-swizzled weight K-blocks into the
//              stage's B buffer; L2 prefetch of upcoming crop-row segments
//   warp  5    MMA: allocates TMEM, one elected thread issues tcgen05.mma (M=128, N=n_pad,
//              K=16) x 12 per group, tcgen05.commit releases the stage / publishes the tile
//   warps 6-13 converters: nearest-exact source pixel fetch (sy = y0 + ((2dy+1)h)>>7,
//              sx = x0 + ((2dx+1)w)>>7), exact u8 -> bf16, st.shared into the 128B-swizzled
//              K-major A stage, fence.proxy.async, mbarrier arrive.
// The A tile never touches HBM: only the sampled frame bytes are read.
#include "hydro_internal.cuh"

using namespace hydro;

namespace {

struct ClsCtrl {
  uint64_t full_a[4];
  uint64_t full_b[4];
  uint64_t empty[4];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  uint32_t pad;
  float bias[HYDRO_MAX_CLASSES];
};

__device__ __forceinline__ uint32_t bf16_bits_of_byte(uint32_t b) {
  // exact: the float 2^23 + b minus 2^23 is b; its top 16 bits are the bf16 of b (b < 256)
  const float f = __uint_as_float(0x4B000000u | b) - 8388608.0f;
  return __float_as_uint(f) >> 16;
}

__device__ __forceinline__ uint32_t ldg32(const uint8_t* p) { return __ldg(reinterpret_cast<const uint32_t*>(p)); }

struct RowMeta {  // per alive tuple of the tile
  uint32_t frame_off;  // byte offset of frame row 0
  int32_t x0, y0, w, h;
  int32_t valid;
};

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
  m.frame_off = fid * static_cast<uint32_t>(p.frame_h * p.frame_w * 3);
  m.x0 = x0;
  m.y0 = y0;
  m.w = x1 - x0;
  m.h = y1 - y0;
  return m;
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

}  // namespace

extern __shared__ __align__(1024) uint8_t hydro_cls_smem[];

__global__ void __launch_bounds__(kClsThreads, 1) hydro_classifier_kernel(ClsParams p) {
  DevState* st = p.st;
  // ---- dispatch (uniform across the CTA: every thread reads the same device words)
  int pred;
  const uint32_t* list_in;
  uint32_t count, base = p.range_base;
  uint32_t* bits_out;
  if (p.dispatch) {
    if (p.hop >= st->n_pred) return;
    pred = st->order[p.hop];
    if (st->kind[pred] != kLinear) return;
    if (p.hop == 0) {
      list_in = nullptr;
      count = p.range_n;
    } else {
      list_in = p.lists + static_cast<uint64_t>(p.hop) * p.list_stride;
      count = p.counts[p.hop];
    }
    bits_out = p.bits + static_cast<uint64_t>(p.hop) * p.bits_stride;
  } else {
    pred = p.explicit_pred;
    list_in = p.list_in;
    count = list_in ? *p.count_in : p.range_n;
    bits_out = p.bits_out;
  }
  const uint32_t num_tiles = (count + kTileM - 1) / kTileM;
  if (blockIdx.x >= num_tiles) return;

  const long long t_start = clock64();
  const PredDev& pdg = p.preds[pred];
  const int n_classes = pdg.n_classes, n_pad = pdg.n_pad, target = pdg.target;
  const uint8_t* w_tiled = pdg.w_tiled;
  const int n_alloc = n_pad <= 32 ? 32 : (n_pad <= 64 ? 64 : 128);
  const uint32_t tmem_cols = 2u * n_alloc;
  const uint32_t b_stage_bytes = kKBlocksPerGroup * n_pad * 128;
  const uint32_t stage_bytes = (kAStageBytes + b_stage_bytes + 1023u) & ~1023u;

  // ---- shared memory carve-up (1024-aligned for the 128B swizzle)
  const uint32_t raw = smem_u32(hydro_cls_smem);
  uint8_t* smem = hydro_cls_smem + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t avail = kClsSmemBytes - 1024u - static_cast<uint32_t>(sizeof(ClsCtrl)) - 64u;
  const uint32_t S = min(4u, avail / stage_bytes);
  ClsCtrl* ctrl = reinterpret_cast<ClsCtrl*>(smem + S * stage_bytes);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&ctrl->full_a[s], kConvWarps);
      mbar_init(&ctrl->full_b[s], 1);
      mbar_init(&ctrl->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&ctrl->tfull[a], 1);
      mbar_init(&ctrl->tempty[a], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&ctrl->tmem_base)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid < HYDRO_MAX_CLASSES) ctrl->bias[tid] = tid < n_classes ? pdg.bias[tid] : 0.0f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = ctrl->tmem_base;

  if (warp == kLoaderWarp) {
    // ===================== loader: weights (bulk copy) + L2 prefetch of crop rows
    constexpr int kPrefetchGroups = 3;
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      RowMeta mr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) mr[r] = load_meta(p, list_in, base, tile * kTileM + lane * 4 + r, count);
      auto prefetch_group = [&](int g) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (!mr[r].valid) continue;
          const int sy = mr[r].y0 + (((2 * g + 1) * mr[r].h) >> 7);
          const uint8_t* row = p.frames + mr[r].frame_off + static_cast<uint32_t>(sy) * (p.frame_w * 3);
          const uint32_t a = (3u * mr[r].x0) & ~15u;
          const uint32_t e = (3u * (mr[r].x0 + mr[r].w) + 15u) & ~15u;
          const uint32_t row_bytes = static_cast<uint32_t>(p.frame_w * 3);
          prefetch_l2(row + a, min(e, row_bytes) - a);
        }
      };
      for (int g = 0; g < kPrefetchGroups; ++g) prefetch_group(g);
      for (int g = 0; g < kGroups; ++g, ++it) {
        if (g + kPrefetchGroups < kGroups) prefetch_group(g + kPrefetchGroups);
        const uint32_t s = it % S, ph = (it / S) & 1u;
        if (lane == 0) {
          mbar_wait(&ctrl->empty[s], ph ^ 1u);
          uint8_t* bdst = smem + s * stage_bytes + kAStageBytes;
          mbar_arrive_expect_tx(&ctrl->full_b[s], b_stage_bytes);
          bulk_g2s(bdst, w_tiled + static_cast<uint64_t>(g) * b_stage_bytes, b_stage_bytes, &ctrl->full_b[s]);
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (single thread)
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(kTileM, static_cast<uint32_t>(n_pad));
      uint32_t it = 0, tl = 0;
      for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl) {
        const uint32_t acc = tl & 1u, aph = (tl >> 1) & 1u;
        mbar_wait(&ctrl->tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * static_cast<uint32_t>(n_alloc);
        for (int g = 0; g < kGroups; ++g, ++it) {
          const uint32_t s = it % S, ph = (it / S) & 1u;
          mbar_wait(&ctrl->full_a[s], ph);
          mbar_wait(&ctrl->full_b[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + s * stage_bytes);
          const uint32_t b_base = a_base + kAStageBytes;
#pragma unroll
          for (int kb = 0; kb < kKBlocksPerGroup; ++kb) {
#pragma unroll
            for (int kk = 0; kk < kKBlock / 16; ++kk) {
              const uint64_t ad = desc_sw128(a_base + kb * (kTileM * 128) + kk * 32);
              const uint64_t bd = desc_sw128(b_base + kb * (n_pad * 128) + kk * 32);
              tc_mma_bf16(d_tmem, ad, bd, idesc, (g | kb | kk) != 0 ? 1u : 0u);
            }
          }
          tc_commit(&ctrl->empty[s]);
        }
        tc_commit(&ctrl->tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= kConvWarp0) {
    // ===================== converters: gather + u8->bf16 + swizzled st.shared
    const int cw = warp - kConvWarp0;  // rows m = cw + 8*i, i = 0..15
    constexpr int kRows = kTileM / kConvWarps;  // 16
    constexpr int kBatch = 8;
    const uint32_t row_pitch = static_cast<uint32_t>(p.frame_w * 3);
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      // lane i < 16 holds the metadata of row cw + 8*i
      RowMeta my = load_meta(p, list_in, base, tile * kTileM + cw + kConvWarps * (lane & 15), count);
      if (lane >= kRows) my.valid = 0;
      for (int g = 0; g < kGroups; ++g, ++it) {
        const uint32_t s = it % S, ph = (it / S) & 1u;
        mbar_wait(&ctrl->empty[s], ph ^ 1u);
        uint8_t* a_stage = smem + s * stage_bytes;
#pragma unroll
        for (int i0 = 0; i0 < kRows; i0 += kBatch) {
          uint32_t w00[kBatch], w01[kBatch], w10[kBatch], w11[kBatch], sh0[kBatch], sh1[kBatch];
          int valid[kBatch];
#pragma unroll
          for (int b = 0; b < kBatch; ++b) {
            const int src = i0 + b;
            valid[b] = __shfl_sync(0xFFFFFFFFu, my.valid, src);
            const uint32_t foff = __shfl_sync(0xFFFFFFFFu, my.frame_off, src);
            const int x0 = __shfl_sync(0xFFFFFFFFu, my.x0, src);
            const int y0 = __shfl_sync(0xFFFFFFFFu, my.y0, src);
            const int w = __shfl_sync(0xFFFFFFFFu, my.w, src);
            const int h = __shfl_sync(0xFFFFFFFFu, my.h, src);
            w00[b] = w01[b] = w10[b] = w11[b] = 0;
            sh0[b] = sh1[b] = 0;
            if (valid[b]) {
              const int sy = y0 + (((2 * g + 1) * h) >> 7);
              const uint8_t* row = p.frames + foff + static_cast<uint32_t>(sy) * row_pitch;
              const int dx0 = 2 * lane;
              const int sx0 = x0 + (((2 * dx0 + 1) * w) >> 7);
              const int sx1 = x0 + (((2 * dx0 + 3) * w) >> 7);
              const uint32_t o0 = 3u * sx0, o1 = 3u * sx1;
              w00[b] = ldg32(row + (o0 & ~3u));
              if ((o0 & 3u) > 1u) w01[b] = ldg32(row + (o0 & ~3u) + 4);
              w10[b] = ldg32(row + (o1 & ~3u));
              if ((o1 & 3u) > 1u) w11[b] = ldg32(row + (o1 & ~3u) + 4);
              sh0[b] = 8u * (o0 & 3u);
              sh1[b] = 8u * (o1 & 3u);
            }
          }
#pragma unroll
          for (int b = 0; b < kBatch; ++b) {
            if (!valid[b]) continue;
            const int m = cw + kConvWarps * (i0 + b);
            const uint32_t px0 = __funnelshift_r(w00[b], w01[b], sh0[b]);
            const uint32_t px1 = __funnelshift_r(w10[b], w11[b], sh1[b]);
            uint32_t e[6];
            e[0] = bf16_bits_of_byte(px0 & 0xFF);
            e[1] = bf16_bits_of_byte((px0 >> 8) & 0xFF);
            e[2] = bf16_bits_of_byte((px0 >> 16) & 0xFF);
            e[3] = bf16_bits_of_byte(px1 & 0xFF);
            e[4] = bf16_bits_of_byte((px1 >> 8) & 0xFF);
            e[5] = bf16_bits_of_byte((px1 >> 16) & 0xFF);
            const uint32_t row_off = static_cast<uint32_t>(m >> 3) * 1024u + static_cast<uint32_t>(m & 7) * 128u;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const uint32_t el = 6u * lane + 2u * q;    // element within the 192-element crop row
              const uint32_t kb = el >> 6;
              const uint32_t byte = (el & 63u) * 2u;
              const uint32_t chunk = (byte >> 4) ^ static_cast<uint32_t>(m & 7);
              const uint32_t off = kb * (kTileM * 128u) + row_off + (chunk << 4) + (byte & 15u);
              *reinterpret_cast<uint32_t*>(a_stage + off) = e[2 * q] | (e[2 * q + 1] << 16);
            }
            if (p.dbg_crops) {
              const uint32_t pos = tile * kTileM + m;
              uint16_t* d = p.dbg_crops + static_cast<uint64_t>(pos) * kFeatures + g * 192 + 6 * lane;
#pragma unroll
              for (int j = 0; j < 6; ++j) d[j] = static_cast<uint16_t>(e[j]);
            }
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctrl->full_a[s]);
      }
    }
  } else {
    // ===================== epilogue warps 0..3 (TMEM lane quadrant = warp)
    const int q = warp;
    uint32_t n_in = 0, n_pass = 0, tl = 0;
    for (uint32_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl) {
      const uint32_t acc = tl & 1u, aph = (tl >> 1) & 1u;
      mbar_wait(&ctrl->tfull[acc], aph);
      tc_fence_after();
      const int m = q * 32 + lane;
      const uint32_t pos = tile * kTileM + m;
      const bool valid = pos < count;
      float best = -3.402823466e38f;
      int bi = 0;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * static_cast<uint32_t>(n_alloc);
      for (int c0 = 0; c0 < n_pad; c0 += 16) {
        uint32_t v[16];
        tc_ld_32x32b_x16(taddr + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int c = c0 + j;
          if (c < n_classes) {
            const float z = __uint_as_float(v[j]) + ctrl->bias[c];
            if (z > best) {  // strict: lowest index wins ties (R12)
              best = z;
              bi = c;
            }
            if (p.dbg_logits && valid) p.dbg_logits[static_cast<uint64_t>(pos) * n_classes + c] = z;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->tempty[acc]);
      const bool verdict = valid && (bi == target);
      const uint32_t bv = __ballot_sync(0xFFFFFFFFu, verdict);
      const uint32_t bvalid = __ballot_sync(0xFFFFFFFFu, valid);
      if (lane == 0 && bvalid) bits_out[tile * (kTileM / 32) + q] = bv;
      if (p.dbg_verdict && valid) p.dbg_verdict[pos] = verdict ? 1 : 0;
      n_in += __popc(bvalid);
      n_pass += __popc(bv);
    }
    if (p.collect_stats && lane == 0) {
      atomicAdd(&st->d_in[pred], static_cast<unsigned long long>(n_in));
      atomicAdd(&st->d_pass[pred], static_cast<unsigned long long>(n_pass));
    }
  }

  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols) : "memory");
  }
  if (tid == 0 && p.collect_stats) {
    atomicAdd(&st->d_cost[pred], static_cast<unsigned long long>(clock64() - t_start));
  }
}
