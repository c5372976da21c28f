// Internal device-side state, kernel parameter blocks and PTX helpers of libhydro.
// sm_100a only.  Nothing here is shared with oracle/ (DESIGN.md §1).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hydro.h"

namespace hydro {

constexpr int kMaxPred = HYDRO_MAX_PREDICATES;
constexpr int kCrop = HYDRO_CROP;
constexpr int kFeatures = HYDRO_FEATURES;   // 12288
constexpr int kKBlock = 64;                 // bf16 elements per UMMA K-block row (128 B)
constexpr int kNumKBlocks = kFeatures / kKBlock;  // 192
constexpr int kKBlocksPerGroup = 3;         // one crop row (64 px x 3 ch = 192 el) per stage
constexpr int kGroups = kNumKBlocks / kKBlocksPerGroup;  // 64 crop rows

// ---- K1 (route / filter / compact) geometry
constexpr int kRouteThreads = 256;
#ifndef HYDRO_K1_ITEMS
#define HYDRO_K1_ITEMS 8
#endif
constexpr int kRouteItems = HYDRO_K1_ITEMS;                 // positions per thread
constexpr int kRouteTile = kRouteThreads * kRouteItems;     // 2048 positions per tile

// ---- K4 (classifier) geometry
constexpr int kTileM = 128;                                 // UMMA M (cta_group::1)
constexpr int kConvWarps = 8;                               // gather/convert warps
constexpr int kConvRows = kTileM / kConvWarps;              // 16 consecutive rows per converter warp
constexpr int kEpiWarps = 4;                                // TMEM quadrant warps 0..3
constexpr int kLoaderWarp = 4;                              // weights (bulk copy) + L2 prefetch
constexpr int kMmaWarp = 5;                                 // TMEM alloc + tcgen05.mma issue
constexpr int kConvWarp0 = 6;
constexpr int kClsWarps = kConvWarp0 + kConvWarps;          // 14
constexpr int kClsThreads = kClsWarps * 32;                 // 448
constexpr int kAKBlockBytes = kTileM * 128;                 // one 128 x 64 fp16 K-block: 16 KB
constexpr int kARing = 6;                                   // A K-block stages (2 crop rows)
constexpr int kBRing = 3;                                   // B K-block stages
// staging pitch of the 4 rows of a quad: 800 B = 200 words puts row r's segment 8r banks after
// row 0's, which spreads the 4 rows' read windows (measured by simulation: 41.4 -> 40.0 LDS
// wavefronts per quad with the interleaved pixel order below)
#ifndef HYDRO_SEG_PITCH
#define HYDRO_SEG_PITCH 800
#endif
constexpr int kSegPitch = HYDRO_SEG_PITCH;
// longest crop-row segment staged contiguously (3*255 + 16-byte alignment slack when the pitch
// allows); wider segments are staged as a 64-pixel gather (8 B per sampled pixel)
constexpr int kMaxSegBytes = kSegPitch < 784 ? kSegPitch : 784;
static_assert(kSegPitch % 16 == 0 && kMaxSegBytes >= 512, "staging pitch");
#ifndef HYDRO_QUAD_DEPTH
#define HYDRO_QUAD_DEPTH 2
#endif
constexpr int kQuadDepth = HYDRO_QUAD_DEPTH;                // quads staged ahead per converter warp
constexpr int kQuadSlots = kQuadDepth + 1;
constexpr int kQuadSlotBytes = 4 * kSegPitch;               // 4 rows x worst-case segment
constexpr int kClsSmemBytes = 232448;                       // 227 KB opt-in maximum
// data-aware AREA hops (R28): K6's per-CTA position ranges are used while the hop has fewer than
// this many 128-tuple tiles per CTA (the tail dominates); beyond, tiles are dealt round-robin and
// the balance is the warp-level row assignment inside every tile
constexpr uint32_t kBalRangeTilesPerCta = 4;

// K order of the A operand inside one crop row (192 = 64 px x 3 ch elements):
// converter lane j of a row produces output pixels dx = j + 8k (k = 0..7, interleaved so that the
// 8 lanes of a row read 8 neighbouring pixels in every load instruction: one short shared-memory
// window per row instead of 8 windows spread over the whole segment) and stores them as three
// 16-byte chunks 3j .. 3j+2.  Position p of the crop row therefore holds feature
//   (g*64 + dx) * 3 + ch  with  j = p / 24, k = (p % 24) / 3, ch = p % 3, dx = j + 8k.
// The weight tiling applies the same permutation, so the contraction sum_k x_k W[c][k] is unchanged.
__host__ __device__ __forceinline__ uint32_t crop_pos_feature(uint32_t g, uint32_t p) {
  const uint32_t j = p / 24u, rem = p % 24u;
  return (g * 64u + j + 8u * (rem / 3u)) * 3u + rem % 3u;
}

// K order of K4-T (hydro_classifier_tm_kernel, A in tensor memory): position
// p = 2c + e of a crop row is element e of TMEM column c.  Converter thread t0 = t % 4 of a tuple
// writes columns 8i + 2*t0 + sub (tcgen05.st 16x256b repetition i = 0..11, sub = 0, 1), holding its
// per-row features f = 4*(i % 6) + 2*sub + e of half hh = i / 6: pixel k = 8*hh + f / 3 (output
// pixel dx = 4k + t0), channel f % 3.
__host__ __device__ __forceinline__ uint32_t crop_pos_feature_tm(uint32_t g, uint32_t p) {
  const uint32_t c = p >> 1, e = p & 1u;
  const uint32_t i = c >> 3, t0 = (c >> 1) & 3u, sub = c & 1u;
  const uint32_t f = 4u * (i % 6u) + 2u * sub + e;
  const uint32_t k = 8u * (i / 6u) + f / 3u;
  return (g * 64u + 4u * k + t0) * 3u + f % 3u;
}

// K order of AREA heads (K4's row-cooperative AREA converter): lane q of a converter
// warp makes output pixels q and q + 32 of one tuple's crop row and stores their 6 features as 3
// consecutive words, so position p = 6q + 3*hi + ch of crop row g holds feature
// (g*64 + q + 32*hi) * 3 + ch.
__host__ __device__ __forceinline__ uint32_t crop_pos_feature_area(uint32_t g, uint32_t p) {
  const uint32_t q = p / 6u, r = p % 6u;
  return (g * 64u + q + 32u * (r / 3u)) * 3u + r % 3u;
}

enum PredKind : int32_t {
  kLabelEq = HYDRO_PRED_LABEL_EQ,
  kHash = HYDRO_PRED_HASH,
  kLinear = HYDRO_PRED_LINEAR,
  kMlp = HYDRO_PRED_MLP,
  kHsv = HYDRO_PRED_HSV
};
// classifier hops run in K4 (linear or MLP head); cheap hops run in K1
__host__ __device__ inline bool is_classifier(int32_t kind) { return kind == kLinear || kind == kMlp || kind == kHsv; }

struct PredDev {
  int32_t kind;
  int32_t label_value;
  uint64_t seed;
  uint64_t thr0, thr1;
  uint64_t drift_id;
  int32_t units, units_per_area;
  const uint8_t* w_tiled;   // LINEAR: [192 kblk][n_pad rows][128 B SW128-swizzled]
  const uint8_t* w_tiled_tm;  // LINEAR (nearest): the same in K4-T's K order (crop_pos_feature_tm)
  const float* bias;        // [n_pad] (padding rows: -inf never wins; they are skipped anyway)
  int32_t n_classes, n_pad, target, crop_mode;
  int32_t a_fp16;           // 1: operands staged as fp16 (weights exactly representable), 0: bf16
  float w_unscale;          // LINEAR: 2^-k for weights tiled as 2^k W (exact fp16 rescale), else 1
  int32_t hidden;           // MLP: hidden width (256 / 512); w_tiled = W1 (n_pad rows = hidden), bias = b2
  const uint8_t* w2_tiled;  // MLP: W2 [hidden/64 kblk][n_pad rows][128 B SW128], bf16
  const float* bias1;       // MLP: b1 [hidden]
  uint32_t* cache_known;    // verdict cache (reuse-aware routing): bit id = verdict known
  uint32_t* cache_pass;     //   bit id = cached verdict
  uint64_t cache_cap;       //   ids [0, cache_cap)
  int32_t cache_fill;       //   record computed verdicts
  int32_t pad2_;
};

// Device-resident eddy state (one per context).  d_* are the atomically accumulated deltas of
// the running batch; pend_* the deltas waiting for the next fold (multi-GPU: all-reduced).
struct DevState {
  int32_t n_pred;
  int32_t policy;
  int32_t cost_source;
  int32_t pair_a, pair_b;             // fused linear pair (K4-T, one contraction for both heads); -1: none
  int32_t pad0;
  double gamma;
  double prior;
  int32_t kind[kMaxPred];
  int32_t order[kMaxPred];
  int32_t position[kMaxPred];
  int32_t sched[kMaxPred];            // hop slot -> first order position of that hop (-1: none)
  double declared_cost[kMaxPred];
  double declared_sel[kMaxPred];
  double cost_norm[kMaxPred];         // raw cycles -> SM-cycles
  unsigned long long d_in[kMaxPred], d_pass[kMaxPred], d_cost[kMaxPred];
  unsigned long long d_comp[kMaxPred];     // tuples evaluated (not served by the verdict cache)
  unsigned long long d_hit[kMaxPred];      // REUSE probe: cached ids of the batch
  unsigned long long pend[4 * kMaxPred];   // in[8], pass[8], cost[8], comp[8]: the local window
  unsigned long long xfer[2][4 * kMaxPred];  // exchanged windows (multi-rank): summed over the ranks in place
  unsigned long long tot_comp[kMaxPred];
  double s_comp[kMaxPred];
  double hit[kMaxPred];                    // REUSE: the batch's cache hit rate
  unsigned long long tot_in[kMaxPred], tot_pass[kMaxPred];
  double tot_cost[kMaxPred];
  double s_in[kMaxPred], s_pass[kMaxPred], s_cost[kMaxPred];
  double sel[kMaxPred], cost[kMaxPred], key[kMaxPred];
  unsigned int pad1, pad2;
  // device launch timers (bench evidence, hydro_device_time): per kernel kind, %globaltimer of the
  // first CTA's start and the last CTA's end of every launch that did work, summed
  unsigned long long kt_start[8], kt_end[8], kt_total[8], kt_count[8];
  unsigned long long kt_items[8];  // classifier-input tuples (crops) the kind's launches evaluated
  unsigned int kt_done[8];
};

// Fused pair hop: order positions h and h + 1 hold the context's two pairable linear heads (same
// nearest crop, one K4-T contraction evaluates both).
__host__ __device__ inline bool is_pair_hop(const int32_t* order, int P, int h, int pa, int pb) {
  return pa >= 0 && h >= 0 && h + 1 < P &&
         ((order[h] == pa && order[h + 1] == pb) || (order[h] == pb && order[h + 1] == pa));
}

// Hop schedule: the evaluator hops of an order are its classifier positions (a fused pair counts
// once) and the starts of its maximal runs of cheap predicates; slot i of the per-batch chain runs
// hop sched[i].  The host launches only as many slots as any order of the context can need.
__host__ __device__ inline void build_sched(const int32_t* kind, const int32_t* order, int P, int32_t* sched,
                                            int pa = -1, int pb = -1) {
  int n = 0;
  if (P == 0) sched[n++] = 0;
  for (int h = 0; h < P; ++h) {
    if (is_classifier(kind[order[h]])) {
      if (h == 0 || !is_pair_hop(order, P, h - 1, pa, pb)) sched[n++] = h;  // (the 2nd of a pair: no hop)
    } else if (h == 0 || is_classifier(kind[order[h - 1]])) {
      sched[n++] = h;
    }
  }
  for (; n < kMaxPred; ++n) sched[n] = -1;
}

struct BatchRec {
  unsigned int warm_count;    // survivors of the warmup slice (written first in the output)
  unsigned int total_count;   // all survivors of the batch
  int32_t order_used[kMaxPred];
  unsigned long long d_in[kMaxPred], d_pass[kMaxPred], d_cost[kMaxPred], d_comp[kMaxPred];
};

// K1: evaluate a run of cheap predicates -> verdict bitmap (bit per input position) + survivors
// per 2048-position segment.  K2: compact (input positions, bitmap, segment counts) -> the next
// alive list or the emitted (id, bbox) rows.  No inter-CTA waiting in either kernel.
struct RouteParams {
  // ---- input positions: RANGE (list_in == nullptr): idx = range_base + p, p < range_n;
  //      LIST: idx = list_in[p], p < *count_in
  const uint32_t* list_in;
  const uint32_t* count_in;
  uint32_t range_base, range_n;
  const uint32_t* sel0;        // dispatch: hop 0 reads these positions (nullptr: the range)
  const uint32_t* sel0_count;  // device count of sel0
  const uint32_t* and_bits[kMaxPred];  // verdict bitmaps (bit p) ANDed into the alive mask
  int32_t n_and;
  // ---- which predicates: dispatch (device order) or explicit
  int32_t dispatch;       // 1: hop = `hop`, decided on device from order[]; 0: explicit below
  int32_t hop;
  int32_t explicit_pred;  // dispatch == 0: -1 = none, else evaluate this single predicate
  // ---- hop-indexed workspace (dispatch mode)
  uint32_t* lists;        // list h at lists + h * list_stride  (h = 1..P)
  uint64_t list_stride;
  uint32_t* counts;       // counts[h]
  uint32_t* bits;         // verdicts of hop h at bits + h * bits_stride
  uint64_t bits_stride;
  // ---- outputs
  uint32_t* bitmap_out;   // explicit mode
  uint32_t* seg_counts;   // survivors per 2048-position segment
  uint32_t* warp_counts;  // survivors per 256-position warp segment (8 per 2048-position segment)
  // ---- columns
  const uint64_t* id;
  const uint32_t* frame_id;
  const uint64_t* bbox;   // 4 x u16 packed
  const uint16_t* label;
  // ---- state
  DevState* st;
  const PredDev* preds;
  int32_t collect_stats;
  int32_t force_fill;     // record every computed verdict in the predicate's cache (hydro_cache_fill)
};

struct CompactParams {
  int32_t dispatch;       // 1: hop from device order; 0: explicit
  int32_t hop;
  const uint32_t* list_in;  // explicit: nullptr = range
  const uint32_t* count_in;
  uint32_t range_base, range_n;
  const uint32_t* sel0;        // dispatch: hop 0 reads these positions (nullptr: the range)
  const uint32_t* sel0_count;  // device count of sel0
  const uint32_t* bits_in;  // explicit
  const uint32_t* seg_counts;
  const uint32_t* warp_counts;
  uint32_t* lists;
  uint64_t list_stride;
  uint32_t* counts;
  const uint32_t* bits;
  uint64_t bits_stride;
  int32_t emit;             // explicit: 1 = emit rows, 0 = write list_out / count_out
  uint32_t* list_out;
  uint32_t* count_out;
  uint64_t* out_ids;
  uint64_t* out_bbox;
  uint32_t* out_pos;           // emit: the survivors' input positions too (nullable)
  uint32_t* emit_count;        // *emit_count = *emit_offset + survivors
  const uint32_t* emit_offset; // nullable
  const uint64_t* id;
  const uint64_t* bbox;
  DevState* st;
};
// K1F (fused route + emit for chains without classifiers): K1's inputs, K2's emit outputs and the
// look-back state (tile_status[ntiles] then tile_counter, zeroed before every launch)
constexpr int kFusedMaxRun = 4;
struct FusedParams {
  RouteParams r;
  uint64_t* out_ids;
  uint64_t* out_bbox;
  uint32_t* out_pos;
  uint32_t* emit_count;
  const uint32_t* emit_offset;
  unsigned long long* tile_status;
  uint32_t* tile_counter;
};
// concurrent-worker router (hydro_route_workers): each worker's device state and SM count
struct WorkerRoute {
  const DevState* st[kMaxPred];
  double sms[kMaxPred];
  int32_t n;
  int32_t policy;
};

constexpr int kCompactUnits = 16;  // HASH rounds from which K1 compacts the alive ids before hashing
constexpr int kWarpSeg = 256;  // positions per K1 warp per tile (= kRouteTile / 8)
constexpr int kCompactSegs = 4;  // 2048-position segments per K2 CTA (multiple of 4: vector prefix loads)

struct ClsParams {
  int32_t dispatch;       // 1: hop from device order; 0: explicit_pred
  int32_t hop;
  int32_t explicit_pred;
  const uint32_t* list_in;    // explicit mode input (nullptr: range)
  const uint32_t* count_in;
  uint32_t range_base, range_n;
  const uint32_t* sel0;        // dispatch: hop 0 reads these positions (nullptr: the range)
  const uint32_t* sel0_count;  // device count of sel0
  uint32_t* lists;
  uint64_t list_stride;
  uint32_t* counts;
  uint32_t* bits;
  uint64_t bits_stride;
  uint32_t* bits_out;         // explicit mode output bitmap
  uint32_t* seg_counts;       // survivors per 2048-position segment (atomically accumulated; zeroed by K1)
  uint32_t* warp_counts;      // survivors per 256-position warp segment (likewise)
  const uint32_t* frame_id;
  const uint64_t* bbox;
  const uint8_t* frames;
  int32_t n_frames, frame_h, frame_w;
  DevState* st;
  const PredDev* preds;
  float* dbg_logits;      // [pos][n_classes]
  uint16_t* dbg_crops;    // [pos][12288]
  uint8_t* dbg_verdict;   // [pos]
  int32_t collect_stats;
  // data-aware tile scheduling (HYDRO_BALANCE_DATA_AWARE, AREA heads)
  const uint32_t* bounds;  // K4: CTA c owns positions [bounds[c], bounds[c+1]) when the hop is AREA
  uint32_t* bal_chunks;    // K6: estimated cost (sum of w*h) per 32-position chunk of the hop input
  uint32_t* bal_bounds;    // K6: output bounds, bal_ctas + 1 entries
  int32_t bal_ctas;        // CTAs of the K4 launch the bounds are for
  int32_t area_only;       // K4: evaluate AREA hops only (nearest hops run in K4-T, launched beside it)
  // verdict caches on classifier hops (reuse; R26): K0c splits a cached hop's
  // input into cached verdicts (written straight into the hop bitmap) and the uncached tuples,
  // which the classifier kernel then evaluates through this redirection
  const uint64_t* id;       // tuple ids (cache lookups and fills)
  uint32_t* cache_idx;      // uncached tuples: batch indices (the classifier's list input) ...
  uint32_t* cache_pos;      // ... their positions in the hop input (verdict bits) ...
  uint32_t* cache_count;    // ... and their number; nullptr: the context has no classifier cache
  int32_t force_fill;       // hydro_cache_fill: record every computed verdict
  // fused linear pair (DevState pair_a / pair_b): both heads' weights tiled into one B operand
  // (pair_a's rows [0, pair_npa), pair_b's after), their biases, per-head logit scales
  const uint8_t* pair_w_tiled;
  const float* pair_bias;   // [pair_n_pad]
  int32_t pair_npa, pair_n_pad;
  float pair_unscale_a, pair_unscale_b;
};

// ------------------------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// long waits: the hint lets the warp sleep in hardware instead of re-polling
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAITS_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// waits of the warps that are idle most of the time (epilogue, MMA issuer, weight loader): poll the
// phase with a non-blocking test and sleep in between, so the polling does not take issue slots
// from the converter warps (a suspended try_wait re-polls at every barrier event of the CTA)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
template <int kNs>
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  while (!mbar_test(bar, parity)) __nanosleep(kNs);
}

// async proxy / TMA bulk copy (1D) global -> shared, completion on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// tcgen05
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t smem_addr) {
  // SM100 shared-memory matrix descriptor, K-major, 128B swizzle:
  // start>>4 [0,14) | LBO=1 (16 B) [16,30) | SBO=1024>>4 [32,46) | version 1 [46,48) | layout 2 [61,64)
  return static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

__device__ __forceinline__ uint32_t idesc_f16_f32(uint32_t M, uint32_t N, bool bf16) {
  // kind::f16 instruction descriptor: D f32 [4,6)=1, A/B format [7,10)/[10,13) (0 = f16, 1 = bf16),
  // K-major A/B (bits 15,16 = 0), N>>3 [17,23), M>>4 [24,29)
  const uint32_t f = bf16 ? 1u : 0u;
  return (1u << 4) | (f << 7) | (f << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tc_ld_32x32b_x16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- device launch timer: thread 0 of every CTA of a launch calls begin after the dispatch check
// and end after the CTA's work; the last CTA to end adds (last end - first start) to the kind's total
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ktimer_begin(DevState* st, int kind) { atomicMin(&st->kt_start[kind], gtimer_ns()); }
__device__ __forceinline__ void ktimer_end(DevState* st, int kind) {
  atomicMax(&st->kt_end[kind], gtimer_ns());
  __threadfence();
  const unsigned int n = gridDim.x * gridDim.y * gridDim.z;
  if (atomicAdd(&st->kt_done[kind], 1u) == n - 1) {
    __threadfence();
    const unsigned long long e = atomicAdd(&st->kt_end[kind], 0ull), s = atomicAdd(&st->kt_start[kind], 0ull);
    st->kt_total[kind] += e > s ? e - s : 0ull;
    st->kt_count[kind] += 1;
    st->kt_start[kind] = ~0ull;
    st->kt_end[kind] = 0ull;
    st->kt_done[kind] = 0u;
  }
}

// ---- classifier hop inputs and verdict output (all K4 kernels)
// A cached classifier hop (its predicate has a verdict cache and K0c ran) evaluates only the
// uncached tuples: list input = their batch indices, `ind` = their hop-input positions.
__device__ __forceinline__ const uint32_t* cls_redirect(const ClsParams& p, const PredDev& pd, const uint32_t*& list_in,
                                                        uint32_t& count) {
  if (!p.dispatch || !p.cache_count || !pd.cache_known) return nullptr;
  list_in = p.cache_idx;
  count = *p.cache_count;
  return p.cache_pos;
}
// Verdict of position `pos` of the kernel's input (one call per lane, the 32 lanes of a warp hold
// positions wpos0 .. wpos0 + 31): direct mode writes the bitmap word with one ballot; redirected
// mode sets the bit of the hop-input position (atomicOr: a word's positions are spread over
// tiles).  Survivor counts per 2048 / 256 positions for K2.  With `fill`, the computed verdict is
// recorded in the predicate's cache (keyed by tuple id).
__device__ __forceinline__ void cls_emit(const ClsParams& p, uint32_t* bits_out, const uint32_t* ind,
                                         const uint32_t* list_in, uint32_t base, uint32_t wpos0, uint32_t pos,
                                         bool valid, bool verdict, const PredDev& pd, bool fill) {
  const int lane = static_cast<int>(threadIdx.x & 31);
  if (!ind) {
    const uint32_t bv = __ballot_sync(0xFFFFFFFFu, verdict), bvalid = __ballot_sync(0xFFFFFFFFu, valid);
    if (lane == 0 && bvalid) {
      bits_out[wpos0 >> 5] = bv;
      if (bv) {
        atomicAdd(p.seg_counts + wpos0 / kRouteTile, static_cast<uint32_t>(__popc(bv)));
        atomicAdd(p.warp_counts + wpos0 / kWarpSeg, static_cast<uint32_t>(__popc(bv)));
      }
    }
  } else if (valid && verdict) {
    const uint32_t q = __ldg(ind + pos);
    atomicOr(bits_out + (q >> 5), 1u << (q & 31));
    atomicAdd(p.seg_counts + q / kRouteTile, 1u);
    atomicAdd(p.warp_counts + q / kWarpSeg, 1u);
  }
  if (fill && valid) {
    const uint32_t idx = list_in ? __ldg(list_in + pos) : base + pos;
    const uint64_t id = __ldg(p.id + idx);
    if (id < pd.cache_cap) {
      const uint32_t bit = 1u << (id & 31);
      if (verdict) atomicOr(pd.cache_pass + (id >> 5), bit);
      else atomicAnd(pd.cache_pass + (id >> 5), ~bit);
      atomicOr(pd.cache_known + (id >> 5), bit);
    }
  }
}

// ---- method arithmetic on device (independent of oracle/, written from DESIGN.md R5)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  return h ^ (h >> 16);
}

}  // namespace hydro

// kernels (defined in k_route.cu / k_classifier.cu), launched by runtime.cu
void hydro_route_launch(const hydro::RouteParams& r, int grid, cudaStream_t stream, bool compact);
void hydro_route_emit_launch(const hydro::FusedParams& f, int grid, cudaStream_t stream);
int hydro_route_emit_occupancy();
int hydro_route_emit_tile();
int hydro_route_occupancy(bool compact);
__global__ void hydro_compact_kernel(hydro::CompactParams p);
cudaError_t hydro_classifier_configure();
void hydro_classifier_launch(const hydro::ClsParams& c, int grid, cudaStream_t stream, bool debug, bool area);
// K6 data-aware balance: per-chunk input-size estimates, then the bounds
void hydro_balance_launch(const hydro::ClsParams& c, uint64_t max_positions, int num_sms, cudaStream_t stream);
void hydro_mlp_launch(const hydro::ClsParams& c, int grid, cudaStream_t stream, bool debug);
void hydro_classifier_tm_launch(const hydro::ClsParams& c, int grid, cudaStream_t stream, bool debug);
void hydro_cache_split_launch(const hydro::ClsParams& c, uint64_t max_positions, int num_sms, cudaStream_t stream);
void hydro_hsv_launch(const hydro::ClsParams& c, uint64_t max_positions, int num_sms, cudaStream_t stream);
int hydro_hsv_warps_per_sm();
__global__ void hydro_fold_kernel(hydro::DevState* st, hydro::BatchRec* rec, int32_t mode, uint32_t n_batch,
                                  int32_t snap_slot, int32_t apply_slot);
__global__ void hydro_route_workers_kernel(hydro::WorkerRoute w, int32_t* order, double* cost, double* sel);
__global__ void hydro_probe_kernel(hydro::DevState* st, const hydro::PredDev* preds, const uint64_t* id, uint32_t base,
                                   uint32_t n);
__global__ void hydro_cache_put_kernel(uint32_t* known, uint32_t* pass, uint64_t cap, const uint64_t* ids,
                                       const uint8_t* verdicts, uint64_t n);
__global__ void hydro_tile_weights_kernel(const uint16_t* w, uint8_t* w_tiled, int32_t n_classes, int32_t n_pad,
                                          int32_t k_features, int32_t to_fp16, int32_t crop_order, int32_t* inexact,
                                          float scale);
