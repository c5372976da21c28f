// libhydro host runtime: the C ABI of include/hydro.h.
//
// Per routing batch the runtime enqueues a FIXED launch skeleton on the
// context stream; which predicate each hop evaluates is decided on the device from the order
// the previous fold wrote (no host synchronisation inside a batch):
//   [first batch] warmup slice: every predicate on the slice (bitmaps) -> AND + emit -> fold
//   for hop h = 0 .. P-1:   K1(h)  route/compact (cheap predicates, bitmap of hop h-1)
//                           K4(h)  classifier hop (exits unless order[h] is LINEAR)
//   K1(P)   final compaction + emit of (id, bbox) in input order
//   K5      fold (+ NCCL all-reduce of the deltas when world > 1)
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "hydro_internal.cuh"

using namespace hydro;

static thread_local std::string g_last_error;

// Driver-API entry points for green contexts, resolved through the runtime (cudaGetDriverEntryPoint)
// so the library keeps no link-time dependency on libcuda (it still loads on a machine without a
// driver; only sm_groups > 1 needs them).
struct GreenApi {
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetDevResource) getDevResource = nullptr;
  decltype(&cuDevSmResourceSplitByCount) splitByCount = nullptr;
  decltype(&cuDevResourceGenerateDesc) generateDesc = nullptr;
  decltype(&cuGreenCtxCreate) ctxCreate = nullptr;
  decltype(&cuGreenCtxStreamCreate) streamCreate = nullptr;
  decltype(&cuGreenCtxDestroy) ctxDestroy = nullptr;
  decltype(&cuGetErrorString) errorString = nullptr;
  bool ok = false;
};
static const GreenApi& green_api() {
  static GreenApi g = [] {
    GreenApi a;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      // the ABI version of the prototypes in the cuda.h this file is compiled against
      return cudaGetDriverEntryPointByVersion(name, fn, CUDA_VERSION, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess;
    };
    a.ok = get("cuDeviceGet", reinterpret_cast<void**>(&a.deviceGet)) &&
           get("cuDeviceGetDevResource", reinterpret_cast<void**>(&a.getDevResource)) &&
           get("cuDevSmResourceSplitByCount", reinterpret_cast<void**>(&a.splitByCount)) &&
           get("cuDevResourceGenerateDesc", reinterpret_cast<void**>(&a.generateDesc)) &&
           get("cuGreenCtxCreate", reinterpret_cast<void**>(&a.ctxCreate)) &&
           get("cuGreenCtxStreamCreate", reinterpret_cast<void**>(&a.streamCreate)) &&
           get("cuGreenCtxDestroy", reinterpret_cast<void**>(&a.ctxDestroy)) &&
           get("cuGetErrorString", reinterpret_cast<void**>(&a.errorString));
    return a;
  }();
  return g;
}

static bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && e[0] == '1';
}

static hydro_status set_err(hydro_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

#define CU(expr)                                                                                   \
  do {                                                                                             \
    cudaError_t _e = (expr);                                                                       \
    if (_e != cudaSuccess) {                                                                       \
      return ctx_fail(ctx, HYDRO_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));       \
    }                                                                                              \
  } while (0)

namespace {

struct PredHost {
  hydro_predicate_desc desc;
  uint8_t* w_tiled = nullptr;
  uint8_t* w_tiled_tm = nullptr;  // nearest LINEAR heads: K4-T's K order
  float* bias = nullptr;
  int n_pad = 0;
  int a_fp16 = 0;
  int w_scale_log2 = 0;  // LINEAR: weights tiled as 2^k W (fp16-exact), logits scaled back by 2^-k
  uint8_t* w2_tiled = nullptr;  // MLP layer 2
  float* bias1 = nullptr;       // MLP layer 1 bias
  uint32_t* cache_known = nullptr;  // verdict cache (reuse-aware routing)
  uint32_t* cache_pass = nullptr;
  uint64_t cache_cap = 0;
  int cache_fill = 0;
};

struct Slot {
  bool busy = false;
  int64_t batch_id = -1;
  int64_t n = 0;
  int64_t warm_n = 0;
  cudaEvent_t done = nullptr;
  cudaEvent_t uploaded = nullptr;
  uint64_t* out_ids = nullptr;
  uint64_t* out_bbox = nullptr;
  uint32_t* out_pos = nullptr;  // the survivors' input positions (hydro_batch_output)
  BatchRec* rec = nullptr;
  BatchRec rec_host{};
  bool rec_valid = false;
  // staging for host input
  uint64_t* s_id = nullptr;
  uint32_t* s_frame = nullptr;
  uint64_t* s_bbox = nullptr;
  uint16_t* s_label = nullptr;
};

struct TimedLaunch {
  cudaEvent_t a, b;
  int kind;
};

}  // namespace

struct hydro_ctx {
  hydro_config cfg{};
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host -> device uploads of batch k+1 overlap batch k
  bool own_stream = false;
  CUgreenCtx green = nullptr;  // sm_groups > 1: the SM partition the context's stream runs on
  int num_sms = 0;
  int k1_occ = 1;
  bool k1_compact = false;  // a HASH predicate expensive enough for K1's compaction path
  std::vector<PredHost> preds;
  bool frozen = false;
  bool warmup_pending = true;
  hydro_status sticky = HYDRO_OK;
  std::string sticky_msg;
  // device state
  DevState* st = nullptr;
  PredDev* preds_dev = nullptr;
  uint32_t* lists = nullptr;
  uint64_t list_stride = 0;
  uint32_t* counts = nullptr;
  uint32_t* bits = nullptr;
  uint64_t bits_stride = 0;
  uint32_t* warm_bits = nullptr;
  uint32_t* seg_counts = nullptr;  // [max_segs] segment counts, then [8 * max_segs] warp counts
  unsigned long long* fused_status = nullptr;  // K1F look-back: [max_segs] tile words, then the tile counter
  uint64_t max_segs = 0;
  uint32_t* warm_and = nullptr;
  uint32_t* bal_chunks = nullptr;  // K6 (data-aware balance): chunk cost estimates
  uint32_t* bal_bounds = nullptr;  // K6: per-CTA position bounds of the current AREA hop
  int bal_last_ctas = 0;           // CTAs of the last data-aware K4 launch
  uint32_t* zero_word = nullptr;
  std::vector<Slot> slots;
  int64_t next_batch = 0;
  int64_t launches = 0;
  int64_t since_sync = 0;
  ncclComm_t comm = nullptr;
  // statistics exchange between ranks (a11): NCCL on a side stream or the HOST callback
  bool exchange = false;
  cudaStream_t xchg_stream = nullptr;
  cudaEvent_t xchg_ready[2] = {nullptr, nullptr}, xchg_done[2] = {nullptr, nullptr};
  uint64_t* host_xfer = nullptr;  // pinned, HOST transport
  int xchg_next = 0;              // slot of the next snapshot
  int xchg_outstanding = -1;      // slot exchanged at the last sync point, not folded yet
  // green-context workers run on a library stream: it waits on the caller's stream per submit
  cudaStream_t user_stream = nullptr;
  cudaEvent_t user_ev = nullptr;
  int32_t fixed_order[kMaxPred];
  bool fixed_order_set = false;
  bool has_area = false;
  bool has_nearest_linear = false;  // a nearest LINEAR head (K4-T) next to an AREA head (K4)
  bool k4_legacy = false;
  int pair_a = -1, pair_b = -1;   // fused linear pair (pred ids), see freeze()
  int pair_npa = 0, pair_n_pad = 0;
  uint8_t* pair_w_tiled = nullptr;
  float* pair_bias = nullptr;
  uint32_t* cache_idx = nullptr;    // K0c: uncached tuples of a cached classifier hop (batch indices)
  uint32_t* cache_pos = nullptr;    //      and their hop-input positions
  uint32_t* cache_count = nullptr;  //      their number (nullptr: no classifier cache)  // HYDRO_K4_LEGACY=1: nearest heads on the shared-memory-A kernel (A/B runs)
  bool has_linear = false, has_mlp = false, has_hsv = false;
  std::vector<PredDev> pd_host;  // the device predicate table as uploaded at freeze
  // timing
  bool timing = false;
  std::vector<TimedLaunch> timed;
  std::vector<cudaEvent_t> event_pool;
};

static hydro_status ctx_fail(hydro_ctx* ctx, hydro_status s, const std::string& msg) {
  if (ctx && (s == HYDRO_ECUDA || s == HYDRO_ENCCL) && ctx->sticky == HYDRO_OK) {
    ctx->sticky = s;
    ctx->sticky_msg = msg;
  }
  return set_err(s, msg);
}

static hydro_status check_sticky(hydro_ctx* ctx) {
  if (ctx->sticky != HYDRO_OK) return set_err(ctx->sticky, ctx->sticky_msg);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_fail(ctx, HYDRO_ECUDA, std::string("async CUDA error: ") + cudaGetErrorString(e));
  return HYDRO_OK;
}

static cudaEvent_t get_event(hydro_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

template <typename F>
static hydro_status timed_launch(hydro_ctx* ctx, int kind, F&& launch) {
  TimedLaunch tl{};
  if (ctx->timing) {
    tl.a = get_event(ctx);
    tl.b = get_event(ctx);
    tl.kind = kind;
    cudaEventRecord(tl.a, ctx->stream);
  }
  launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_fail(ctx, HYDRO_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  ctx->launches += 1;
  if (ctx->timing) {
    cudaEventRecord(tl.b, ctx->stream);
    ctx->timed.push_back(tl);
  }
  return HYDRO_OK;
}

static int next_pow2_pad(int c) {  // n_pad: multiple of 16 >= c
  return ((c + 15) / 16) * 16;
}

// Copies W [rows][k_features] (bf16; host or device) and re-lays it out as the swizzled K-block
// image the classifier kernels bulk-copy (n_pad rows per K-block).  try_fp16: re-encode as fp16
// when every weight is exactly representable (*fp16 = 1), else keep bf16 (*fp16 = 0).
// k = 15 - floor(log2 max|w|) over a bf16 weight matrix (host or device; 0 if all zero): the
// power-of-two rescale that puts the largest weight just below fp16's maximum exponent
static int fp16_scale_log2(hydro_ctx* ctx, const uint16_t* w, bool on_device, size_t n) {
  std::vector<uint16_t> h;
  const uint16_t* src = w;
  if (on_device) {
    h.resize(n);
    if (cudaMemcpy(h.data(), w, n * sizeof(uint16_t), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
    src = h.data();
  }
  (void)ctx;
  int emax = -1000;
  for (size_t i = 0; i < n; ++i) {
    const uint32_t e = (src[i] >> 7) & 0xFFu;
    if ((src[i] & 0x7FFFu) == 0 || e == 0 || e == 0xFFu) continue;  // zeros, subnormals, inf / NaN
    emax = std::max(emax, static_cast<int>(e) - 127);
  }
  return emax == -1000 ? 0 : 15 - emax;
}

static hydro_status tile_weights(hydro_ctx* ctx, const uint16_t* w, bool on_device, int rows, int n_pad,
                                 int k_features, bool try_fp16, uint8_t** out, int* fp16, int order,
                                 float scale = 1.0f);

// ------------------------------------------------------------------------------------------

extern "C" {

const char* hydro_version(void) { return "hydro-b200 0.1 (sm_100a)"; }
const char* hydro_last_error(void) { return g_last_error.c_str(); }

hydro_status hydro_config_default(hydro_config* cfg) {
  if (!cfg) return set_err(HYDRO_EINVAL, "cfg is NULL");
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->device = 0;
  cfg->stream = nullptr;
  cfg->policy = HYDRO_POLICY_SCORE;
  cfg->cost_source = HYDRO_COST_MEASURED;
  cfg->decay_gamma = 0.5;
  cfg->prior_selectivity = 0.5;
  cfg->warmup_tuples = 65536;
  cfg->max_batch_tuples = 1 << 20;
  cfg->max_inflight = 4;
  cfg->rank = 0;
  cfg->world = 1;
  cfg->sync_every = 1;
  return HYDRO_OK;
}

hydro_status hydro_nccl_unique_id(void* out128) {
  if (!out128) return set_err(HYDRO_EINVAL, "out128 is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_err(HYDRO_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
  return HYDRO_OK;
}

hydro_status hydro_create(const hydro_config* cfg, hydro_ctx** out) {
  if (!cfg || !out) return set_err(HYDRO_EINVAL, "NULL argument");
  hydro_ctx* ctx = nullptr;
  if (cfg->max_batch_tuples < 1 || cfg->max_batch_tuples > (1 << 30))
    return set_err(HYDRO_EINVAL, "max_batch_tuples must be in [1, 2^30]");
  if (cfg->max_inflight < 1 || cfg->max_inflight > 64) return set_err(HYDRO_EINVAL, "max_inflight in [1, 64]");
  if (!(cfg->decay_gamma > 0.0 && cfg->decay_gamma <= 1.0)) return set_err(HYDRO_EINVAL, "decay_gamma in (0, 1]");
  if (!(cfg->prior_selectivity >= 0.0 && cfg->prior_selectivity <= 1.0))
    return set_err(HYDRO_EINVAL, "prior_selectivity in [0, 1]");
  if (cfg->policy < 0 || cfg->policy > HYDRO_POLICY_REUSE) return set_err(HYDRO_EINVAL, "unknown policy");
  if (cfg->cost_source < 0 || cfg->cost_source > 1) return set_err(HYDRO_EINVAL, "unknown cost_source");
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return set_err(HYDRO_EINVAL, "bad rank/world");
  if (cfg->transport != HYDRO_TRANSPORT_NCCL && cfg->transport != HYDRO_TRANSPORT_HOST)
    return set_err(HYDRO_EINVAL, "unknown transport");
  if (cfg->transport == HYDRO_TRANSPORT_HOST && !cfg->allreduce_fn)
    return set_err(HYDRO_EINVAL, "HOST transport needs allreduce_fn");
  if (cfg->world > 1 && cfg->transport == HYDRO_TRANSPORT_NCCL && !cfg->nccl_unique_id)
    return set_err(HYDRO_EINVAL, "world > 1 needs nccl_unique_id (NCCL transport)");
  if (cfg->world > 1 && cfg->policy == HYDRO_POLICY_REUSE)
    return set_err(HYDRO_EINVAL, "REUSE orders each batch by its own cache hit rate: single rank only");
  if (cfg->sync_every < 1) return set_err(HYDRO_EINVAL, "sync_every >= 1");
  if (cfg->balance != HYDRO_BALANCE_ROUND_ROBIN && cfg->balance != HYDRO_BALANCE_DATA_AWARE)
    return set_err(HYDRO_EINVAL, "unknown balance mode");
  if (cfg->max_sms < 0) return set_err(HYDRO_EINVAL, "max_sms >= 0");
  if (cfg->sm_groups < 0 || (cfg->sm_groups > 1 && (cfg->sm_group < 0 || cfg->sm_group >= cfg->sm_groups)))
    return set_err(HYDRO_EINVAL, "sm_group must be in [0, sm_groups)");
  if (cfg->frames) {
    if (cfg->n_frames < 1 || cfg->frame_h < 1 || cfg->frame_w < 1 || (cfg->frame_w % 16) != 0 ||
        cfg->frame_h > 65535 || cfg->frame_w > 65535)
      return set_err(HYDRO_EINVAL, "frame pool: n_frames, frame_h >= 1; frame_w % 16 == 0; dims <= 65535");
    if ((reinterpret_cast<uintptr_t>(cfg->frames) & 15u) != 0) return set_err(HYDRO_EINVAL, "frames must be 16-byte aligned");
    if (static_cast<double>(cfg->n_frames) * cfg->frame_h * cfg->frame_w * 3 >= 68719476736.0)
      return set_err(HYDRO_EINVAL, "frame pool must be < 64 GiB");  // row offsets in 16-byte units (u32)
  }
  ctx = new hydro_ctx();
  ctx->cfg = *cfg;
  CU(cudaSetDevice(cfg->device));
  CU(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cfg->device));
  if (cfg->max_sms > 0) ctx->num_sms = std::min(ctx->num_sms, static_cast<int>(cfg->max_sms));  // SM budget
  if (cfg->sm_groups > 1) {
    // a worker on its own SM partition (CUDA green context): group sm_group of an even split
    const GreenApi& G = green_api();
    CUdevice dev;
    CUdevResource all, rem;
    std::vector<CUdevResource> groups(static_cast<size_t>(cfg->sm_groups));
    unsigned int ng = static_cast<unsigned int>(cfg->sm_groups);
    CUdevResourceDesc desc;
    CUstream gs = nullptr;
    CUresult r = G.ok ? CUDA_SUCCESS : CUDA_ERROR_NOT_SUPPORTED;
    const char* step = "driver entry points";
    if (r == CUDA_SUCCESS) r = G.deviceGet(&dev, cfg->device), step = "cuDeviceGet";
    if (r == CUDA_SUCCESS) r = G.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM), step = "cuDeviceGetDevResource";
    // even split; the SM count of a group a multiple of 8 (the co-scheduling granularity)
    const unsigned int per = r == CUDA_SUCCESS ? (all.sm.smCount / static_cast<unsigned int>(cfg->sm_groups)) & ~7u : 0u;
    if (r == CUDA_SUCCESS) r = G.splitByCount(groups.data(), &ng, &all, &rem, 0, per), step = "cuDevSmResourceSplitByCount";
    if (r == CUDA_SUCCESS && ng <= static_cast<unsigned int>(cfg->sm_group)) r = CUDA_ERROR_INVALID_VALUE, step = "group count";
    if (r == CUDA_SUCCESS) r = G.generateDesc(&desc, &groups[cfg->sm_group], 1), step = "cuDevResourceGenerateDesc";
    if (r == CUDA_SUCCESS) r = G.ctxCreate(&ctx->green, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM), step = "cuGreenCtxCreate";
    if (r == CUDA_SUCCESS) r = G.streamCreate(&gs, ctx->green, CU_STREAM_NON_BLOCKING, 0), step = "cuGreenCtxStreamCreate";
    if (r != CUDA_SUCCESS) {
      const char* msg = nullptr;
      if (G.errorString) G.errorString(r, &msg);
      hydro_status s = set_err(HYDRO_ECUDA, std::string("green context SM partition (") + step + "): " +
                                                (msg ? msg : "driver API unavailable"));
      hydro_destroy(ctx);
      return s;
    }
    ctx->stream = reinterpret_cast<cudaStream_t>(gs);
    ctx->own_stream = true;
    if (cfg->stream) {  // keep the caller's stream order: every submit waits on it
      ctx->user_stream = static_cast<cudaStream_t>(cfg->stream);
      CU(cudaEventCreateWithFlags(&ctx->user_ev, cudaEventDisableTiming));
    }
    ctx->num_sms = std::min(ctx->num_sms, static_cast<int>(groups[cfg->sm_group].sm.smCount));
  } else if (cfg->stream) {
    ctx->stream = static_cast<cudaStream_t>(cfg->stream);
  } else {
    CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  ctx->k1_occ = hydro_route_occupancy(false);
  CU(hydro_classifier_configure());
  {
    const char* e = getenv("HYDRO_K4_LEGACY");
    ctx->k4_legacy = e && e[0] == '1';
  }
  CU(cudaMalloc(&ctx->st, sizeof(DevState)));
  CU(cudaMemset(ctx->st, 0, sizeof(DevState)));
  CU(cudaMalloc(&ctx->preds_dev, sizeof(PredDev) * kMaxPred));
  CU(cudaMalloc(&ctx->zero_word, 16));
  CU(cudaMemset(ctx->zero_word, 0, 16));
  if (cfg->transport == HYDRO_TRANSPORT_HOST) {
    ctx->exchange = true;
    CU(cudaMallocHost(&ctx->host_xfer, sizeof(uint64_t) * 4 * kMaxPred));
  } else if (cfg->nccl_unique_id) {  // world > 1, or world == 1 with an id: exercise the NCCL merge path
    ctx->exchange = true;
    CU(cudaStreamCreateWithFlags(&ctx->xchg_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CU(cudaEventCreateWithFlags(&ctx->xchg_ready[i], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&ctx->xchg_done[i], cudaEventDisableTiming));
    }
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_unique_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&ctx->comm, cfg->world, id, cfg->rank);
    if (r != ncclSuccess) {
      hydro_status s = set_err(HYDRO_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      hydro_destroy(ctx);
      return s;
    }
  }
  ctx->warmup_pending = (cfg->warmup_tuples > 0) && (cfg->policy == HYDRO_POLICY_SCORE ||
                                                     cfg->policy == HYDRO_POLICY_COST ||
                                                     cfg->policy == HYDRO_POLICY_SELECTIVITY ||
                                                     cfg->policy == HYDRO_POLICY_REUSE);
  *out = ctx;
  return HYDRO_OK;
}

hydro_status hydro_add_predicate(hydro_ctx* ctx, const hydro_predicate_desc* d, int32_t* pred_id) {
  if (!ctx || !d) return set_err(HYDRO_EINVAL, "NULL argument");
  if (ctx->frozen) return set_err(HYDRO_ESTATE, "add_predicate after the first submit");
  if (static_cast<int>(ctx->preds.size()) >= kMaxPred) return set_err(HYDRO_EINVAL, "too many predicates (max 8)");
  if (!(d->declared_cost >= 0.0) || !(d->declared_selectivity >= 0.0 && d->declared_selectivity <= 1.0))
    return set_err(HYDRO_EINVAL, "declared_cost >= 0, declared_selectivity in [0, 1]");
  PredHost ph;
  ph.desc = *d;
  if (d->kind == HYDRO_PRED_LABEL_EQ) {
    if (d->label_value < 0 || d->label_value > 65535) return set_err(HYDRO_EINVAL, "label_value out of u16 range");
  } else if (d->kind == HYDRO_PRED_HASH) {
    if (d->threshold[0] > (1ull << 32) || d->threshold[1] > (1ull << 32))
      return set_err(HYDRO_EINVAL, "threshold must be <= 2^32");
    if (d->units < 0 || d->units_per_area < 0) return set_err(HYDRO_EINVAL, "units must be >= 0");
  } else if (d->kind == HYDRO_PRED_HSV) {
    if (!ctx->cfg.frames) return set_err(HYDRO_EINVAL, "HSV predicate needs the frame pool in hydro_config");
    if (d->target < 0 || d->target > 9) return set_err(HYDRO_EINVAL, "HSV target is a colour class in [0, 9]");
    if (d->crop_mode != HYDRO_CROP_NEAREST) return set_err(HYDRO_EINVAL, "HSV supports HYDRO_CROP_NEAREST only");
    ph.desc.n_classes = 10;
    ctx->has_hsv = true;
  } else if (d->kind == HYDRO_PRED_MLP) {
    if (!ctx->cfg.frames) return set_err(HYDRO_EINVAL, "MLP predicate needs the frame pool in hydro_config");
    if (d->n_classes < 2 || d->n_classes > HYDRO_MAX_CLASSES) return set_err(HYDRO_EINVAL, "n_classes in [2, 128]");
    if (d->target < 0 || d->target >= d->n_classes) return set_err(HYDRO_EINVAL, "target outside [0, n_classes)");
    if (d->hidden != 256 && d->hidden != 512) return set_err(HYDRO_EINVAL, "MLP hidden must be 256 or 512");
    if (!d->weight_bf16 || !d->bias || !d->weight2_bf16 || !d->bias2)
      return set_err(HYDRO_EINVAL, "MLP needs weight_bf16, bias, weight2_bf16 and bias2");
    if (d->crop_mode != HYDRO_CROP_NEAREST) return set_err(HYDRO_EINVAL, "MLP supports HYDRO_CROP_NEAREST only");
    const int C = d->n_classes, H = d->hidden;
    ph.n_pad = next_pow2_pad(C);
    const cudaMemcpyKind kind = d->weights_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    hydro_status st = tile_weights(ctx, d->weight_bf16, d->weights_on_device != 0, H, H, kFeatures, true, &ph.w_tiled,
                                   &ph.a_fp16, 1);
    if (st != HYDRO_OK) return st;
    int w2_fp16 = 0;
    st = tile_weights(ctx, d->weight2_bf16, d->weights_on_device != 0, C, ph.n_pad, H, false, &ph.w2_tiled, &w2_fp16,
                      0);
    if (st != HYDRO_OK) return st;
    CU(cudaMalloc(&ph.bias, sizeof(float) * HYDRO_MAX_CLASSES));
    CU(cudaMemsetAsync(ph.bias, 0, sizeof(float) * HYDRO_MAX_CLASSES, ctx->stream));
    CU(cudaMemcpyAsync(ph.bias, d->bias2, sizeof(float) * C, kind, ctx->stream));
    CU(cudaMalloc(&ph.bias1, sizeof(float) * H));
    CU(cudaMemcpyAsync(ph.bias1, d->bias, sizeof(float) * H, kind, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->has_mlp = true;
  } else if (d->kind == HYDRO_PRED_LINEAR) {
    if (!ctx->cfg.frames) return set_err(HYDRO_EINVAL, "LINEAR predicate needs the frame pool in hydro_config");
    if (d->n_classes < 2 || d->n_classes > HYDRO_MAX_CLASSES) return set_err(HYDRO_EINVAL, "n_classes in [2, 128]");
    if (d->target < 0 || d->target >= d->n_classes) return set_err(HYDRO_EINVAL, "target outside [0, n_classes)");
    if (!d->weight_bf16 || !d->bias) return set_err(HYDRO_EINVAL, "LINEAR needs weight_bf16 and bias");
    if (d->crop_mode != HYDRO_CROP_NEAREST && d->crop_mode != HYDRO_CROP_AREA)
      return set_err(HYDRO_EINVAL, "crop_mode must be HYDRO_CROP_NEAREST or HYDRO_CROP_AREA");
    const int C = d->n_classes;
    ph.n_pad = next_pow2_pad(C);
    // K order of w_tiled: K4's (crop_pos_feature; AREA heads: the AREA converter's order)
    const int k4_order = d->crop_mode == HYDRO_CROP_AREA ? 3 : 1;
    // stage operands as fp16 when every weight is exactly representable (u8 pixels always are):
    // same products, cheaper u8 -> fp16 operand construction in K4
    hydro_status st = tile_weights(ctx, d->weight_bf16, d->weights_on_device != 0, C, ph.n_pad, kFeatures, true,
                                   &ph.w_tiled, &ph.a_fp16, k4_order);
    if (st != HYDRO_OK) return st;
    const char* no_scale = getenv("HYDRO_NO_FP16_SCALE");  // test hook: keep general heads on bf16 operands
    if (!ph.a_fp16 && !(no_scale && no_scale[0] == '1')) {
      // a general bf16 head: scaled by 2^k so that its largest weight sits at the top of fp16's
      // range, every weight is fp16-exact when the head spans <= 32 binades (products and fp32
      // sums are then exactly 2^k times the bf16 ones; the epilogue multiplies by 2^-k)
      const int k = fp16_scale_log2(ctx, d->weight_bf16, d->weights_on_device != 0, static_cast<size_t>(C) * kFeatures);
      if (k != 0 && k > -100 && k < 100) {
        uint8_t* w2 = nullptr;
        int ok = 0;
        st = tile_weights(ctx, d->weight_bf16, d->weights_on_device != 0, C, ph.n_pad, kFeatures, true, &w2, &ok, k4_order,
                          std::ldexp(1.0f, k));
        if (st != HYDRO_OK) return st;
        if (ok) {
          cudaFree(ph.w_tiled);
          ph.w_tiled = w2;
          ph.a_fp16 = 1;
          ph.w_scale_log2 = k;
        } else {
          cudaFree(w2);
        }
      }
    }
    if (d->crop_mode == HYDRO_CROP_NEAREST) {  // K4-T's copy (same operand type and scale)
      int fp16_tm = 0;
      st = tile_weights(ctx, d->weight_bf16, d->weights_on_device != 0, C, ph.n_pad, kFeatures, ph.a_fp16 != 0,
                        &ph.w_tiled_tm, &fp16_tm, 2, std::ldexp(1.0f, ph.w_scale_log2));
      if (st != HYDRO_OK) return st;
    }
    CU(cudaMalloc(&ph.bias, sizeof(float) * HYDRO_MAX_CLASSES));
    CU(cudaMemsetAsync(ph.bias, 0, sizeof(float) * HYDRO_MAX_CLASSES, ctx->stream));
    CU(cudaMemcpyAsync(ph.bias, d->bias, sizeof(float) * C,
                       d->weights_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->has_linear = true;
  } else {
    return set_err(HYDRO_EINVAL, "unknown predicate kind");
  }
  if (d->kind == HYDRO_PRED_LINEAR && d->crop_mode == HYDRO_CROP_AREA) ctx->has_area = true;
  if (d->kind == HYDRO_PRED_LINEAR && d->crop_mode == HYDRO_CROP_NEAREST) ctx->has_nearest_linear = true;
  ctx->preds.push_back(ph);
  if (pred_id) *pred_id = static_cast<int32_t>(ctx->preds.size() - 1);
  return HYDRO_OK;
}

}  // extern "C"

static hydro_status tile_weights(hydro_ctx* ctx, const uint16_t* w, bool on_device, int rows, int n_pad,
                                 int k_features, bool try_fp16, uint8_t** out, int* fp16, int order,
                                 float scale) {
  const size_t wbytes = static_cast<size_t>(rows) * k_features * 2;
  uint16_t* wdev = nullptr;
  CU(cudaMalloc(&wdev, wbytes));
  CU(cudaMemcpyAsync(wdev, w, wbytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMalloc(out, static_cast<size_t>(k_features / kKBlock) * n_pad * 128));
  CU(cudaMemsetAsync(ctx->zero_word + 1, 0, sizeof(int32_t), ctx->stream));
  int32_t* inexact = reinterpret_cast<int32_t*>(ctx->zero_word + 1);
  int32_t bad = 1;
  if (try_fp16) {
    hydro_tile_weights_kernel<<<512, 256, 0, ctx->stream>>>(wdev, *out, rows, n_pad, k_features, 1, k_features == kFeatures ? order : 0, inexact, scale);
    ctx->launches += 1;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&bad, inexact, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  *fp16 = bad ? 0 : 1;
  if (bad) {
    hydro_tile_weights_kernel<<<512, 256, 0, ctx->stream>>>(wdev, *out, rows, n_pad, k_features, 0, k_features == kFeatures ? order : 0, inexact, scale);
    ctx->launches += 1;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(ctx->stream));
  }
  CU(cudaFree(wdev));
  return HYDRO_OK;
}

extern "C" {

hydro_status hydro_cache_enable(hydro_ctx* ctx, int32_t k, uint64_t id_capacity, int32_t fill) {
  if (!ctx) return set_err(HYDRO_EINVAL, "NULL argument");
  if (ctx->frozen) {  // allowed between batches once nothing is in flight
    for (const Slot& sl : ctx->slots)
      if (sl.busy) return set_err(HYDRO_ESTATE, "cache_enable with uncollected batches in flight");
  }
  if (k < 0 || k >= static_cast<int32_t>(ctx->preds.size())) return set_err(HYDRO_EINVAL, "bad pred id");
  PredHost& ph = ctx->preds[k];
  if (ph.cache_known) return set_err(HYDRO_EINVAL, "cache already enabled");
  if (k == ctx->pair_a || k == ctx->pair_b) {  // a cached head leaves the fused pair (K0c splits its hop)
    ctx->pair_a = ctx->pair_b = -1;
    if (ctx->frozen) {
      const int32_t none[2] = {-1, -1};
      CU(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->st) + offsetof(DevState, pair_a), none, sizeof(none),
                         cudaMemcpyHostToDevice, ctx->stream));
      int32_t kind[kMaxPred], order[kMaxPred], sched[kMaxPred];
      const int P = static_cast<int>(ctx->preds.size());
      CU(cudaMemcpyAsync(order, reinterpret_cast<char*>(ctx->st) + offsetof(DevState, order), sizeof(order),
                         cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      for (int i = 0; i < P; ++i) kind[i] = ctx->preds[i].desc.kind;
      build_sched(kind, order, P, sched);
      CU(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->st) + offsetof(DevState, sched), sched, sizeof(sched),
                         cudaMemcpyHostToDevice, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
    }
  }
  if (is_classifier(ph.desc.kind) && !ctx->cache_count) {  // K0c's split lists (one set: hops run in order)
    const size_t cap = static_cast<size_t>(ctx->cfg.max_batch_tuples) + 64;
    CU(cudaMalloc(&ctx->cache_idx, cap * sizeof(uint32_t)));
    CU(cudaMalloc(&ctx->cache_pos, cap * sizeof(uint32_t)));
    CU(cudaMalloc(&ctx->cache_count, sizeof(uint32_t)));
  }
  if (id_capacity == 0 || id_capacity > (1ull << 34)) return set_err(HYDRO_EINVAL, "id_capacity in [1, 2^34]");
  const size_t words = static_cast<size_t>((id_capacity + 31) / 32);
  CU(cudaMalloc(&ph.cache_known, words * 4));
  CU(cudaMalloc(&ph.cache_pass, words * 4));
  CU(cudaMemsetAsync(ph.cache_known, 0, words * 4, ctx->stream));
  CU(cudaMemsetAsync(ph.cache_pass, 0, words * 4, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ph.cache_cap = id_capacity;
  ph.cache_fill = fill ? 1 : 0;
  if (ctx->frozen) {  // refresh the device predicate table entry
    PredDev& q = ctx->pd_host[k];
    q.cache_known = ph.cache_known;
    q.cache_pass = ph.cache_pass;
    q.cache_cap = ph.cache_cap;
    q.cache_fill = ph.cache_fill;
    CU(cudaMemcpy(ctx->preds_dev + k, &q, sizeof(PredDev), cudaMemcpyHostToDevice));
  }
  return HYDRO_OK;
}

hydro_status hydro_cache_put(hydro_ctx* ctx, int32_t k, const uint64_t* ids, const uint8_t* verdicts, int64_t n,
                             int32_t on_device) {
  if (!ctx) return set_err(HYDRO_EINVAL, "NULL argument");
  if (k < 0 || k >= static_cast<int32_t>(ctx->preds.size())) return set_err(HYDRO_EINVAL, "bad pred id");
  PredHost& ph = ctx->preds[k];
  if (!ph.cache_known) return set_err(HYDRO_EINVAL, "no verdict cache on this predicate (hydro_cache_enable)");
  if (n < 0 || (n > 0 && (!ids || !verdicts))) return set_err(HYDRO_EINVAL, "bad ids / verdicts");
  if (n == 0) return HYDRO_OK;
  const uint64_t* d_ids = ids;
  const uint8_t* d_v = verdicts;
  uint64_t* tmp_ids = nullptr;
  uint8_t* tmp_v = nullptr;
  if (!on_device) {
    CU(cudaMalloc(&tmp_ids, sizeof(uint64_t) * n));
    CU(cudaMalloc(&tmp_v, static_cast<size_t>(n)));
    CU(cudaMemcpyAsync(tmp_ids, ids, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(tmp_v, verdicts, static_cast<size_t>(n), cudaMemcpyHostToDevice, ctx->stream));
    d_ids = tmp_ids;
    d_v = tmp_v;
  }
  hydro_cache_put_kernel<<<256, 256, 0, ctx->stream>>>(ph.cache_known, ph.cache_pass, ph.cache_cap, d_ids, d_v,
                                                        static_cast<uint64_t>(n));
  ctx->launches += 1;
  CU(cudaGetLastError());
  if (!on_device) {
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaFree(tmp_ids));
    CU(cudaFree(tmp_v));
  }
  return HYDRO_OK;
}

hydro_status hydro_set_fixed_order(hydro_ctx* ctx, const int32_t* order, int32_t n) {
  if (!ctx || !order) return set_err(HYDRO_EINVAL, "NULL argument");
  const int P = static_cast<int>(ctx->preds.size());
  if (n != P) return set_err(HYDRO_EINVAL, "order length != number of predicates");
  std::vector<int> seen(P, 0);
  for (int i = 0; i < P; ++i) {
    if (order[i] < 0 || order[i] >= P || seen[order[i]]) return set_err(HYDRO_EINVAL, "order is not a permutation");
    seen[order[i]] = 1;
  }
  for (int i = 0; i < P; ++i) ctx->fixed_order[i] = order[i];
  ctx->fixed_order_set = true;
  if (ctx->frozen) {  // update the device order in stream order
    int32_t pos[kMaxPred];
    for (int i = 0; i < P; ++i) pos[order[i]] = i;
    CU(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->st) + offsetof(DevState, order), ctx->fixed_order, sizeof(int32_t) * P, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->st) + offsetof(DevState, position), pos, sizeof(int32_t) * P, cudaMemcpyHostToDevice, ctx->stream));
    int32_t kind[kMaxPred], sched[kMaxPred];
    for (int i = 0; i < P; ++i) kind[i] = ctx->preds[i].desc.kind;
    build_sched(kind, ctx->fixed_order, P, sched, ctx->pair_a, ctx->pair_b);
    CU(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->st) + offsetof(DevState, sched), sched, sizeof(sched), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  return HYDRO_OK;
}

static hydro_status freeze(hydro_ctx* ctx) {
  if (ctx->frozen) return HYDRO_OK;
  const int P = static_cast<int>(ctx->preds.size());
  const uint64_t maxb = static_cast<uint64_t>(ctx->cfg.max_batch_tuples);
  // host-side initial state
  DevState h{};
  h.n_pred = P;
  h.policy = ctx->cfg.policy;
  h.cost_source = ctx->cfg.cost_source;
  h.gamma = ctx->cfg.decay_gamma;
  h.prior = ctx->cfg.prior_selectivity;
  for (const PredHost& ph : ctx->preds)
    if (ph.desc.kind == HYDRO_PRED_HASH && ph.desc.units >= kCompactUnits && ph.desc.units_per_area <= 0)
      ctx->k1_compact = true;
  ctx->k1_occ = hydro_route_occupancy(ctx->k1_compact);
  const double k1_norm = 1.0 / (256.0 * static_cast<double>(ctx->k1_occ) * (kRouteThreads / 32));
  std::vector<PredDev> pd(kMaxPred);
  for (int k = 0; k < P; ++k) {
    const hydro_predicate_desc& d = ctx->preds[k].desc;
    h.kind[k] = d.kind;
    h.declared_cost[k] = d.declared_cost;
    h.declared_sel[k] = d.declared_selectivity;
    h.cost_norm[k] = d.kind == HYDRO_PRED_HSV ? 1.0 / hydro_hsv_warps_per_sm() : (is_classifier(d.kind) ? 1.0 : k1_norm);
    PredDev& q = pd[k];
    q.kind = d.kind;
    q.label_value = d.label_value;
    q.seed = d.seed;
    q.thr0 = d.threshold[0];
    q.thr1 = d.threshold[1];
    q.drift_id = d.drift_id;
    q.units = d.units;
    q.units_per_area = d.units_per_area;
    q.w_tiled = ctx->preds[k].w_tiled;
    q.w_tiled_tm = ctx->preds[k].w_tiled_tm;
    q.bias = ctx->preds[k].bias;
    q.n_classes = d.n_classes;
    q.n_pad = ctx->preds[k].n_pad;
    q.target = d.target;
    q.crop_mode = d.crop_mode;
    q.a_fp16 = ctx->preds[k].a_fp16;
    q.w_unscale = std::ldexp(1.0f, -ctx->preds[k].w_scale_log2);
    q.hidden = d.hidden;
    q.w2_tiled = ctx->preds[k].w2_tiled;
    q.bias1 = ctx->preds[k].bias1;
    q.cache_known = ctx->preds[k].cache_known;
    q.cache_pass = ctx->preds[k].cache_pass;
    q.cache_cap = ctx->preds[k].cache_cap;
    q.cache_fill = ctx->preds[k].cache_fill;
  }
  // initial order: declared statistics (SCORE/COST/SEL before warmup; STATIC), or add order
  for (int k = 0; k < P; ++k) {
    double c = h.declared_cost[k], s = h.declared_sel[k];
    double key;
    if (h.policy == HYDRO_POLICY_COST || h.policy == HYDRO_POLICY_REUSE) key = c;  // REUSE: hit rates per batch
    else if (h.policy == HYDRO_POLICY_SELECTIVITY) key = s;
    else key = (c == 0.0) ? 0.0 : (s >= 1.0 ? INFINITY : c / (1.0 - s));
    h.key[k] = key;
    h.sel[k] = s;
    h.cost[k] = c;
    h.order[k] = k;
  }
  if (h.policy == HYDRO_POLICY_FIXED_ORDER) {
    if (ctx->fixed_order_set)
      for (int i = 0; i < P; ++i) h.order[i] = ctx->fixed_order[i];
  } else {
    std::stable_sort(h.order, h.order + P, [&](int a, int b) { return h.key[a] < h.key[b]; });
  }
  for (int i = 0; i < P; ++i) h.position[h.order[i]] = i;
  // fused linear pair (K4-T evaluates both heads in one contraction when the order puts them next
  // to each other): two nearest LINEAR heads with the same operand type, N_a + N_b <= 144, no
  // verdict cache, K4-T in use (not HYDRO_K4_LEGACY / HYDRO_NO_PAIR; AREA heads never pair)
  ctx->pair_a = ctx->pair_b = -1;
  if (!ctx->k4_legacy && !getenv_flag("HYDRO_NO_PAIR")) {
    int la = -1, lb = -1;
    for (int k = 0; k < P; ++k) {
      const PredHost& ph = ctx->preds[k];
      if (ph.desc.kind != HYDRO_PRED_LINEAR || ph.desc.crop_mode != HYDRO_CROP_NEAREST || ph.cache_known) continue;
      if (la < 0) la = k;
      else if (lb < 0) lb = k;
    }
    if (lb >= 0) {
      const PredHost& A = ctx->preds[la];
      const PredHost& B = ctx->preds[lb];
      const int npa = A.n_pad, npb = B.n_pad, C_a = A.desc.n_classes, C_b = B.desc.n_classes;
      if (A.a_fp16 == B.a_fp16 && npa + npb <= 144 && npa % 16 == 0 && npb % 16 == 0) {
        const size_t pitch = static_cast<size_t>(npa + npb) * 128;
        CU(cudaMalloc(&ctx->pair_w_tiled, pitch * (kFeatures / kKBlock)));
        CU(cudaMemcpy2DAsync(ctx->pair_w_tiled, pitch, A.w_tiled_tm, static_cast<size_t>(npa) * 128,
                             static_cast<size_t>(npa) * 128, kFeatures / kKBlock, cudaMemcpyDeviceToDevice, ctx->stream));
        CU(cudaMemcpy2DAsync(ctx->pair_w_tiled + static_cast<size_t>(npa) * 128, pitch, B.w_tiled_tm,
                             static_cast<size_t>(npb) * 128, static_cast<size_t>(npb) * 128, kFeatures / kKBlock,
                             cudaMemcpyDeviceToDevice, ctx->stream));
        CU(cudaMalloc(&ctx->pair_bias, sizeof(float) * 144));
        CU(cudaMemsetAsync(ctx->pair_bias, 0, sizeof(float) * 144, ctx->stream));
        CU(cudaMemcpyAsync(ctx->pair_bias, A.bias, sizeof(float) * C_a, cudaMemcpyDeviceToDevice, ctx->stream));
        CU(cudaMemcpyAsync(ctx->pair_bias + npa, B.bias, sizeof(float) * C_b, cudaMemcpyDeviceToDevice, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        ctx->pair_a = la;
        ctx->pair_b = lb;
        ctx->pair_npa = npa;
        ctx->pair_n_pad = npa + npb;
      }
    }
  }
  h.pair_a = ctx->pair_a;
  h.pair_b = ctx->pair_b;
  build_sched(h.kind, h.order, P, h.sched, h.pair_a, h.pair_b);
  for (int i = 0; i < 8; ++i) h.kt_start[i] = ~0ull;
  CU(cudaMemcpy(ctx->st, &h, sizeof(h), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->preds_dev, pd.data(), sizeof(PredDev) * kMaxPred, cudaMemcpyHostToDevice));
  ctx->pd_host = pd;
  // workspace
  ctx->list_stride = (maxb + 7) & ~7ull;
  CU(cudaMalloc(&ctx->lists, sizeof(uint32_t) * ctx->list_stride * (P + 1)));
  CU(cudaMalloc(&ctx->counts, sizeof(uint32_t) * (kMaxPred + 2)));
  CU(cudaMemset(ctx->counts, 0, sizeof(uint32_t) * (kMaxPred + 2)));
  ctx->bits_stride = ((maxb + 31) / 32 + 3) & ~3ull;
  CU(cudaMalloc(&ctx->bits, sizeof(uint32_t) * ctx->bits_stride * std::max(P, 1)));
  CU(cudaMalloc(&ctx->warm_bits, sizeof(uint32_t) * ctx->bits_stride * std::max(P, 1)));
  const uint64_t max_segs = (maxb + kRouteTile - 1) / kRouteTile + 1;
  ctx->max_segs = (max_segs + 3) & ~3ull;  // warp counts follow, 16-byte aligned
  CU(cudaMalloc(&ctx->seg_counts, sizeof(uint32_t) * ctx->max_segs * 9));
  CU(cudaMemset(ctx->seg_counts, 0, sizeof(uint32_t) * ctx->max_segs * 9));
  CU(cudaMalloc(&ctx->fused_status, sizeof(unsigned long long) * (8 * ctx->max_segs + 1)));  // tiles >= 256 positions
  CU(cudaMalloc(&ctx->warm_and, sizeof(uint32_t) * ctx->bits_stride));
  if (ctx->cfg.balance == HYDRO_BALANCE_DATA_AWARE && ctx->has_area) {
    CU(cudaMalloc(&ctx->bal_chunks, sizeof(uint32_t) * ((maxb + 31) / 32 + 1)));
    CU(cudaMalloc(&ctx->bal_bounds, sizeof(uint32_t) * (ctx->num_sms + 1)));
  }
  ctx->slots.resize(ctx->cfg.max_inflight);
  for (Slot& s : ctx->slots) {
    CU(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&s.uploaded, cudaEventDisableTiming));
    CU(cudaMalloc(&s.out_ids, sizeof(uint64_t) * maxb));
    CU(cudaMalloc(&s.out_bbox, sizeof(uint64_t) * maxb));
    CU(cudaMalloc(&s.out_pos, sizeof(uint32_t) * maxb));
    CU(cudaMalloc(&s.rec, sizeof(BatchRec)));
  }
  ctx->frozen = true;
  return HYDRO_OK;
}

static hydro_status ensure_staging(hydro_ctx* ctx, Slot& s) {
  if (s.s_id) return HYDRO_OK;
  const uint64_t maxb = static_cast<uint64_t>(ctx->cfg.max_batch_tuples);
  CU(cudaMalloc(&s.s_id, sizeof(uint64_t) * maxb));
  CU(cudaMalloc(&s.s_frame, sizeof(uint32_t) * maxb));
  CU(cudaMalloc(&s.s_bbox, sizeof(uint64_t) * maxb));
  CU(cudaMalloc(&s.s_label, sizeof(uint16_t) * maxb + 16));
  return HYDRO_OK;
}

static RouteParams route_base(hydro_ctx* ctx, const uint64_t* id, const uint32_t* fr, const uint64_t* bb,
                              const uint16_t* lab) {
  RouteParams r{};
  r.lists = ctx->lists;
  r.list_stride = ctx->list_stride;
  r.counts = ctx->counts;
  r.bits = ctx->bits;
  r.bits_stride = ctx->bits_stride;
  r.seg_counts = ctx->seg_counts;
  r.warp_counts = ctx->seg_counts + ctx->max_segs;
  r.id = id;
  r.frame_id = fr;
  r.bbox = bb;
  r.label = lab;
  r.st = ctx->st;
  r.preds = ctx->preds_dev;
  r.collect_stats = 1;
  r.explicit_pred = -1;
  return r;
}

static CompactParams compact_base(hydro_ctx* ctx, const uint64_t* id, const uint64_t* bb, Slot& sl) {
  CompactParams c{};
  c.seg_counts = ctx->seg_counts;
  c.warp_counts = ctx->seg_counts + ctx->max_segs;
  c.lists = ctx->lists;
  c.list_stride = ctx->list_stride;
  c.counts = ctx->counts;
  c.bits = ctx->bits;
  c.bits_stride = ctx->bits_stride;
  c.out_ids = sl.out_ids;
  c.out_bbox = sl.out_bbox;
  c.out_pos = sl.out_pos;
  c.id = id;
  c.bbox = bb;
  c.st = ctx->st;
  return c;
}

static ClsParams cls_base(hydro_ctx* ctx, const uint32_t* fr, const uint64_t* bb) {
  ClsParams c{};
  c.lists = ctx->lists;
  c.list_stride = ctx->list_stride;
  c.counts = ctx->counts;
  c.bits = ctx->bits;
  c.bits_stride = ctx->bits_stride;
  c.frame_id = fr;
  c.bbox = bb;
  c.frames = ctx->cfg.frames;
  c.n_frames = ctx->cfg.n_frames;
  c.frame_h = ctx->cfg.frame_h;
  c.frame_w = ctx->cfg.frame_w;
  c.st = ctx->st;
  c.preds = ctx->preds_dev;
  c.seg_counts = ctx->seg_counts;
  c.warp_counts = ctx->seg_counts + ctx->max_segs;
  c.collect_stats = 1;
  c.explicit_pred = -1;
  if (ctx->pair_a >= 0) {
    c.pair_w_tiled = ctx->pair_w_tiled;
    c.pair_bias = ctx->pair_bias;
    c.pair_npa = ctx->pair_npa;
    c.pair_n_pad = ctx->pair_n_pad;
    c.pair_unscale_a = std::ldexp(1.0f, -ctx->preds[ctx->pair_a].w_scale_log2);
    c.pair_unscale_b = std::ldexp(1.0f, -ctx->preds[ctx->pair_b].w_scale_log2);
  }
  return c;
}

static int route_grid(hydro_ctx* ctx, uint64_t positions) {
  const uint64_t tiles = (positions + kRouteTile - 1) / kRouteTile;
#ifdef HYDRO_K1_ONE_TILE_PER_CTA
  const uint64_t cap = 1u << 20;
#else
  const uint64_t cap = static_cast<uint64_t>(ctx->num_sms) * ctx->k1_occ;
#endif
  return static_cast<int>(std::max<uint64_t>(1, std::min(tiles, cap)));
}

static hydro_status launch_route(hydro_ctx* ctx, const RouteParams& r, uint64_t max_positions) {
  const int grid = route_grid(ctx, max_positions);
  return timed_launch(ctx, 0, [&] { hydro_route_launch(r, grid, ctx->stream, ctx->k1_compact); });
}

// K1F applies to a chain without classifiers: 1..4 LABEL_EQ / uniform-units HASH predicates
// (units below the compacted-HASH threshold), no verdict cache, no selection input
static bool fused_chain_ok(const hydro_ctx* ctx, const hydro_tuples* t) {
  const int P = static_cast<int>(ctx->preds.size());
  if (P < 1 || P > kFusedMaxRun || t->sel || getenv_flag("HYDRO_NO_K1F")) return false;
  for (const PredHost& ph : ctx->preds) {
    const hydro_predicate_desc& d = ph.desc;
    if (ph.cache_known) return false;
    if (d.kind == HYDRO_PRED_LABEL_EQ) continue;
    if (d.kind != HYDRO_PRED_HASH || d.units_per_area > 0 || d.units >= kCompactUnits) return false;
  }
  return true;
}

static hydro_status launch_compact(hydro_ctx* ctx, const CompactParams& c, uint64_t max_positions) {
  const uint64_t segs = (max_positions + kRouteTile - 1) / kRouteTile;
  const int grid = static_cast<int>(std::max<uint64_t>(1, (segs + kCompactSegs - 1) / kCompactSegs));
  return timed_launch(ctx, 3, [&] { hydro_compact_kernel<<<grid, kRouteThreads, 0, ctx->stream>>>(c); });
}

// classifier kernel kinds: the linear head (K4), the MLP head (K4-MLP), the HSV heuristic (K4-HSV)
enum ClsKind { kClsLinear = 0, kClsMlp = 1, kClsHsv = 2 };
static ClsKind cls_kind_of(int32_t pred_kind) {
  return pred_kind == HYDRO_PRED_MLP ? kClsMlp : (pred_kind == HYDRO_PRED_HSV ? kClsHsv : kClsLinear);
}

static hydro_status launch_cls(hydro_ctx* ctx, const ClsParams& c0, uint64_t max_positions, ClsKind kind = kClsLinear) {
  const uint64_t tiles = (max_positions + kTileM - 1) / kTileM;
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(tiles, ctx->num_sms)));
  ClsParams c = c0;
  if (kind == kClsLinear && ctx->bal_bounds && !(c.dbg_crops || c.dbg_logits || c.dbg_verdict)) {
    // data-aware: K6 cuts an AREA hop's input into `grid` ranges of equal estimated cost (it exits
    // on other hops, and K4 then ignores the bounds)
    c.bal_chunks = ctx->bal_chunks;
    c.bal_bounds = ctx->bal_bounds;
    c.bal_ctas = grid;
    c.bounds = ctx->bal_bounds;
    ctx->bal_last_ctas = grid;
    hydro_status s = timed_launch(ctx, 6, [&] { hydro_balance_launch(c, max_positions, ctx->num_sms, ctx->stream); });
    if (s != HYDRO_OK) return s;
    ctx->launches += 1;  // two kernels per K6 launch
  }
  return timed_launch(ctx, kind == kClsMlp ? 4 : (kind == kClsHsv ? 5 : 1), [&] {
    const bool dbg = c.dbg_crops || c.dbg_logits || c.dbg_verdict;
    if (kind == kClsMlp) hydro_mlp_launch(c, grid, ctx->stream, dbg);
    else if (kind == kClsHsv) hydro_hsv_launch(c, max_positions, ctx->num_sms, ctx->stream);
    // kernel instantiation by context capability: nearest heads on K4-T, AREA heads on K4 (its
    // AREA instance); a context with both launches both per linear slot, each kernel exits on the
    // other's hops (the hop's head is known on the device only)
    else if (!ctx->has_area && !ctx->k4_legacy) hydro_classifier_tm_launch(c, grid, ctx->stream, dbg);
    else if (ctx->has_area && !ctx->k4_legacy) {
      if (ctx->has_nearest_linear) {
        hydro_classifier_tm_launch(c, grid, ctx->stream, dbg);
        ctx->launches += 1;
      }
      ClsParams ca = c;
      ca.area_only = 1;
      hydro_classifier_launch(ca, grid, ctx->stream, dbg, true);
    } else hydro_classifier_launch(c, grid, ctx->stream, dbg, ctx->has_area);
  });
}

static hydro_status launch_fold(hydro_ctx* ctx, BatchRec* rec, int mode, int snap_slot = 0, int apply_slot = 0) {
  return timed_launch(ctx, 2, [&] {
    hydro_fold_kernel<<<1, 32, 0, ctx->stream>>>(ctx->st, rec, mode, 0u, snap_slot, apply_slot);
  });
}

// Sums the window snapshot in xfer[slot] over the ranks, in place.  NCCL:
// an all-reduce on the side stream after the snapshot, completion recorded in xchg_done[slot]
// (the compute stream never waits for it until the window is folded, one sync point later).
// HOST: the caller's callback on a pinned copy (synchronous), written back in stream order.
static hydro_status exchange_slot(hydro_ctx* ctx, int slot) {
  void* buf = reinterpret_cast<char*>(ctx->st) + offsetof(DevState, xfer) + sizeof(uint64_t) * 4 * kMaxPred * slot;
  const size_t bytes = sizeof(uint64_t) * 4 * kMaxPred;
  if (ctx->comm) {
    CU(cudaEventRecord(ctx->xchg_ready[slot], ctx->stream));
    CU(cudaStreamWaitEvent(ctx->xchg_stream, ctx->xchg_ready[slot], 0));
    ncclResult_t r = ncclAllReduce(buf, buf, 4 * kMaxPred, ncclUint64, ncclSum, ctx->comm, ctx->xchg_stream);
    if (r != ncclSuccess) return ctx_fail(ctx, HYDRO_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
    CU(cudaEventRecord(ctx->xchg_done[slot], ctx->xchg_stream));
    return HYDRO_OK;
  }
  CU(cudaMemcpyAsync(ctx->host_xfer, buf, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  const int32_t rc = ctx->cfg.allreduce_fn(ctx->cfg.allreduce_user, ctx->host_xfer, 4 * kMaxPred);
  if (rc != 0) return ctx_fail(ctx, HYDRO_ENCCL, "HOST transport all-reduce callback failed (" + std::to_string(rc) + ")");
  CU(cudaMemcpyAsync(buf, ctx->host_xfer, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return HYDRO_OK;
}

// The compute stream may fold xfer[slot] once its exchange completed.
static hydro_status wait_exchange(hydro_ctx* ctx, int slot) {
  if (ctx->comm) CU(cudaStreamWaitEvent(ctx->stream, ctx->xchg_done[slot], 0));
  return HYDRO_OK;
}

// End-of-batch (record = 1) or warmup-slice (force = true) statistics step.  Single rank: the
// deltas are folded at once.  Multi-rank: the deltas join the local window; at a sync point
// (every sync_every batches) ONE launch records, snapshots the window into a slot and folds the
// window exchanged at the previous sync point, then the new slot's exchange is started.  force:
// the window is exchanged and folded immediately (the warmup slice, hydro_flush_stats).
static hydro_status fold_and_sync(hydro_ctx* ctx, BatchRec* rec, int record, bool force) {
  hydro_status s;
  const int rec_bits = rec ? (1 | (record ? 4 : 0)) : 0;
  if (!ctx->exchange) return launch_fold(ctx, rec, rec_bits | 2);
  ctx->since_sync += record ? 1 : 0;
  if (!force && ctx->since_sync < ctx->cfg.sync_every) return launch_fold(ctx, rec, rec_bits);
  const int snap = ctx->xchg_next;
  ctx->xchg_next ^= 1;
  const int prev = ctx->xchg_outstanding;
  if (prev >= 0 && (s = wait_exchange(ctx, prev)) != HYDRO_OK) return s;
  if ((s = launch_fold(ctx, rec, rec_bits | 16 | (prev >= 0 ? (2 | 32) : 0), snap, prev >= 0 ? prev : 0)) != HYDRO_OK)
    return s;
  if ((s = exchange_slot(ctx, snap)) != HYDRO_OK) return s;
  ctx->since_sync = 0;
  ctx->xchg_outstanding = snap;
  if (force) {
    if ((s = wait_exchange(ctx, snap)) != HYDRO_OK) return s;
    if ((s = launch_fold(ctx, nullptr, 2 | 32, 0, snap)) != HYDRO_OK) return s;
    ctx->xchg_outstanding = -1;
  }
  return HYDRO_OK;
}

static hydro_status validate_host_tuples(hydro_ctx* ctx, const hydro_tuples* t) {
  const bool frames = ctx->cfg.frames != nullptr;
  for (int64_t i = 0; i < t->n; ++i) {
    const uint16_t* b = t->bbox + 4 * i;
    if (!(b[0] < b[2] && b[1] < b[3])) return set_err(HYDRO_EINVAL, "bbox must satisfy x0 < x1 and y0 < y1");
    if (frames) {
      if (b[2] > ctx->cfg.frame_w || b[3] > ctx->cfg.frame_h) return set_err(HYDRO_EINVAL, "bbox outside the frame");
      if (t->frame_id[i] >= static_cast<uint32_t>(ctx->cfg.n_frames))
        return set_err(HYDRO_EINVAL, "frame_id >= n_frames");
    }
  }
  return HYDRO_OK;
}

hydro_status hydro_submit_batch(hydro_ctx* ctx, const hydro_tuples* t, int64_t* batch_id) {
  if (!ctx || !t) return set_err(HYDRO_EINVAL, "NULL argument");
  hydro_status s = check_sticky(ctx);
  if (s != HYDRO_OK) return s;
  if (t->n < 0 || t->n > ctx->cfg.max_batch_tuples) return set_err(HYDRO_EINVAL, "n must be in [0, max_batch_tuples]");
  if (t->n > 0 && (!t->id || !t->frame_id || !t->bbox || !t->label)) return set_err(HYDRO_EINVAL, "NULL column");
  const bool has_sel = t->sel != nullptr;
  if (has_sel && (!t->sel_count || !t->on_device))
    return set_err(HYDRO_EINVAL, "a selection needs sel_count and device columns");
  if (has_sel && ctx->cfg.policy == HYDRO_POLICY_REUSE) return set_err(HYDRO_EINVAL, "REUSE does not take selections");
  if ((s = freeze(ctx)) != HYDRO_OK) return s;
  int si = -1;
  for (int i = 0; i < static_cast<int>(ctx->slots.size()); ++i)
    if (!ctx->slots[i].busy) {
      si = i;
      break;
    }
  if (si < 0) return set_err(HYDRO_EBUSY, "all in-flight batch slots hold uncollected results");
  Slot& sl = ctx->slots[si];
  const uint64_t n = static_cast<uint64_t>(t->n);
  const uint64_t* id = t->id;
  const uint32_t* fr = t->frame_id;
  const uint64_t* bb = reinterpret_cast<const uint64_t*>(t->bbox);
  const uint16_t* lab = t->label;
  if (!t->on_device && n > 0) {
    if ((s = validate_host_tuples(ctx, t)) != HYDRO_OK) return s;
    if ((s = ensure_staging(ctx, sl)) != HYDRO_OK) return s;
    // upload on the copy stream (overlaps the previous batch's kernels); the compute stream waits
    CU(cudaMemcpyAsync(sl.s_id, t->id, 8 * n, cudaMemcpyHostToDevice, ctx->copy_stream));
    CU(cudaMemcpyAsync(sl.s_frame, t->frame_id, 4 * n, cudaMemcpyHostToDevice, ctx->copy_stream));
    CU(cudaMemcpyAsync(sl.s_bbox, t->bbox, 8 * n, cudaMemcpyHostToDevice, ctx->copy_stream));
    CU(cudaMemcpyAsync(sl.s_label, t->label, 2 * n, cudaMemcpyHostToDevice, ctx->copy_stream));
    CU(cudaEventRecord(sl.uploaded, ctx->copy_stream));
    CU(cudaStreamWaitEvent(ctx->stream, sl.uploaded, 0));
    id = sl.s_id;
    fr = sl.s_frame;
    bb = sl.s_bbox;
    lab = sl.s_label;
  }
  if (t->wait_event) CU(cudaStreamWaitEvent(ctx->stream, static_cast<cudaEvent_t>(t->wait_event), 0));
  if (ctx->user_stream) {  // a green-context worker: after the caller's stream's earlier work
    CU(cudaEventRecord(ctx->user_ev, ctx->user_stream));
    CU(cudaStreamWaitEvent(ctx->stream, ctx->user_ev, 0));
  }
  CU(cudaMemsetAsync(sl.rec, 0, sizeof(BatchRec), ctx->stream));
  const int P = static_cast<int>(ctx->preds.size());
  uint64_t warm = 0;
  if (ctx->warmup_pending && !has_sel) {  // a selection batch never runs the warmup slice
    // ---- warmup slice (R8): every predicate on the slice, no short-circuit
    warm = std::min<uint64_t>(n, static_cast<uint64_t>(ctx->cfg.warmup_tuples));
    for (int k = 0; k < P; ++k) {
      uint32_t* wb = ctx->warm_bits + static_cast<uint64_t>(k) * ctx->bits_stride;
      if (is_classifier(ctx->preds[k].desc.kind)) {
        ClsParams c = cls_base(ctx, fr, bb);
        c.dispatch = 0;
        c.explicit_pred = k;
        c.list_in = nullptr;
        c.range_base = 0;
        c.range_n = static_cast<uint32_t>(warm);
        c.bits_out = wb;
        if ((s = launch_cls(ctx, c, warm, cls_kind_of(ctx->preds[k].desc.kind))) != HYDRO_OK) return s;
      } else {
        RouteParams r = route_base(ctx, id, fr, bb, lab);
        r.dispatch = 0;
        r.explicit_pred = k;
        r.range_base = 0;
        r.range_n = static_cast<uint32_t>(warm);
        r.bitmap_out = wb;
        if ((s = launch_route(ctx, r, warm)) != HYDRO_OK) return s;
      }
    }
    // AND of the P verdict bitmaps -> K2 emits the slice's rows first in the batch output
    RouteParams r = route_base(ctx, id, fr, bb, lab);
    r.dispatch = 0;
    r.range_base = 0;
    r.range_n = static_cast<uint32_t>(warm);
    r.n_and = P;
    for (int k = 0; k < P; ++k) r.and_bits[k] = ctx->warm_bits + static_cast<uint64_t>(k) * ctx->bits_stride;
    r.bitmap_out = ctx->warm_and;
    r.collect_stats = 0;
    if ((s = launch_route(ctx, r, warm)) != HYDRO_OK) return s;
    CompactParams c = compact_base(ctx, id, bb, sl);
    c.dispatch = 0;
    c.range_base = 0;
    c.range_n = static_cast<uint32_t>(warm);
    c.bits_in = ctx->warm_and;
    c.emit = 1;
    c.emit_count = &sl.rec->warm_count;
    c.emit_offset = nullptr;
    if ((s = launch_compact(ctx, c, warm)) != HYDRO_OK) return s;
    if ((s = fold_and_sync(ctx, sl.rec, 0, true)) != HYDRO_OK) return s;
    ctx->warmup_pending = false;
  }
  // ---- the eddy chain on the rest of the batch: per hop, the evaluator (K1 for a run of cheap
  // predicates, or K4 for a classifier) then K2 compaction into the next hop's alive list / emit
  const uint32_t rest_base = static_cast<uint32_t>(warm);
  const uint32_t rest_n = static_cast<uint32_t>(n - warm);
  if (ctx->cfg.policy == HYDRO_POLICY_REUSE && rest_n > 0) {
    // reuse-aware routing: this batch's cache hit rates -> order by estimated cost
    const int pgrid = static_cast<int>(std::min<uint64_t>((rest_n + 2047) / 2048, static_cast<uint64_t>(ctx->num_sms) * 4));
    if ((s = timed_launch(ctx, 0, [&] {
           hydro_probe_kernel<<<pgrid, kRouteThreads, 0, ctx->stream>>>(ctx->st, ctx->preds_dev, id, rest_base, rest_n);
         })) != HYDRO_OK)
      return s;
    if ((s = timed_launch(ctx, 2, [&] {
           hydro_fold_kernel<<<1, 32, 0, ctx->stream>>>(ctx->st, sl.rec, 8, rest_n, 0, 0);
         })) != HYDRO_OK)
      return s;
  }
  // chain slots: any order has at most L classifier hops and min(C, L + 1) cheap runs
  int n_lin = 0;
  for (int k = 0; k < P; ++k) n_lin += is_classifier(ctx->preds[k].desc.kind) ? 1 : 0;
  const int n_cheap = P - n_lin;
  const int slots = (P == 0 || n_lin == 0) ? 1 : std::min(P, n_lin + std::min(n_cheap, n_lin + 1));
  // K1F when the batch's tiles fit one wave of co-resident CTAs: each CTA then runs one
  // load -> evaluate -> gather -> look-back -> write chain (measured faster than K1 + K2 there);
  // over several waves those chains serialize per CTA and K1 + K2 stream better
  static const int k1f_occ = hydro_route_emit_occupancy();
  const bool fused = n_lin == 0 && fused_chain_ok(ctx, t) &&
                     (static_cast<uint64_t>(rest_n) + hydro_route_emit_tile() - 1) / hydro_route_emit_tile() <=
                         static_cast<uint64_t>(k1f_occ) * ctx->num_sms;
  if (fused) {  // K1F: the whole cheap chain and the emit in one pass (decoupled look-back)
    FusedParams f{};
    f.r = route_base(ctx, id, fr, bb, lab);
    f.r.dispatch = 1;
    f.r.hop = 0;
    f.r.range_base = rest_base;
    f.r.range_n = rest_n;
    f.out_ids = sl.out_ids;
    f.out_bbox = sl.out_bbox;
    f.out_pos = sl.out_pos;
    f.emit_count = &sl.rec->total_count;
    f.emit_offset = &sl.rec->warm_count;
    f.tile_status = ctx->fused_status;
    f.tile_counter = reinterpret_cast<uint32_t*>(ctx->fused_status + 8 * ctx->max_segs);
    const uint64_t tiles = (static_cast<uint64_t>(rest_n) + hydro_route_emit_tile() - 1) / hydro_route_emit_tile();
    CU(cudaMemsetAsync(ctx->fused_status, 0, sizeof(unsigned long long) * (tiles + 1), ctx->stream));
    CU(cudaMemsetAsync(f.tile_counter, 0, sizeof(uint32_t), ctx->stream));
    const int grid = static_cast<int>(std::max<uint64_t>(1, tiles));  // one tile per CTA, all co-resident
    if ((s = timed_launch(ctx, 0, [&] { hydro_route_emit_launch(f, grid, ctx->stream); })) != HYDRO_OK) return s;
  }
  for (int h = 0; h < (fused ? 0 : slots); ++h) {
    RouteParams r = route_base(ctx, id, fr, bb, lab);
    r.dispatch = 1;
    r.hop = h;
    r.range_base = rest_base;
    r.range_n = rest_n;
    r.sel0 = t->sel;
    r.sel0_count = t->sel_count;
    if ((s = launch_route(ctx, r, rest_n)) != HYDRO_OK) return s;
    if (n_lin > 0) {  // the classifier kernel(s) the context needs; each exits unless its kind is the hop's
      ClsParams c = cls_base(ctx, fr, bb);
      c.dispatch = 1;
      c.hop = h;
      c.range_base = rest_base;
      c.range_n = rest_n;
      c.sel0 = t->sel;
      c.sel0_count = t->sel_count;
      c.id = id;
      if (ctx->cache_count) {  // K0c: cached verdicts of this hop (exits unless it is a cached classifier)
        c.cache_idx = ctx->cache_idx;
        c.cache_pos = ctx->cache_pos;
        c.cache_count = ctx->cache_count;
        CU(cudaMemsetAsync(ctx->cache_count, 0, sizeof(uint32_t), ctx->stream));
        if ((s = timed_launch(ctx, 7, [&] { hydro_cache_split_launch(c, rest_n, ctx->num_sms, ctx->stream); })) !=
            HYDRO_OK)
          return s;
      }
      if (ctx->has_linear && (s = launch_cls(ctx, c, rest_n, kClsLinear)) != HYDRO_OK) return s;
      if (ctx->has_mlp && (s = launch_cls(ctx, c, rest_n, kClsMlp)) != HYDRO_OK) return s;
      if (ctx->has_hsv && (s = launch_cls(ctx, c, rest_n, kClsHsv)) != HYDRO_OK) return s;
    }
    CompactParams k2 = compact_base(ctx, id, bb, sl);
    k2.dispatch = 1;
    k2.hop = h;
    k2.range_base = rest_base;
    k2.range_n = rest_n;
    k2.sel0 = t->sel;
    k2.sel0_count = t->sel_count;
    k2.emit_count = &sl.rec->total_count;
    k2.emit_offset = &sl.rec->warm_count;
    if ((s = launch_compact(ctx, k2, rest_n)) != HYDRO_OK) return s;
  }
  if ((s = fold_and_sync(ctx, sl.rec, 1, false)) != HYDRO_OK) return s;
  CU(cudaEventRecord(sl.done, ctx->stream));
  sl.busy = true;
  sl.batch_id = ctx->next_batch++;
  sl.n = static_cast<int64_t>(n);
  sl.warm_n = static_cast<int64_t>(warm);
  sl.rec_valid = false;
  if (batch_id) *batch_id = sl.batch_id;
  return HYDRO_OK;
}

static Slot* find_slot(hydro_ctx* ctx, int64_t batch_id) {
  for (Slot& s : ctx->slots)
    if (s.busy && s.batch_id == batch_id) return &s;
  return nullptr;
}

static hydro_status wait_slot(hydro_ctx* ctx, Slot* sl) {
  CU(cudaEventSynchronize(sl->done));
  hydro_status s = check_sticky(ctx);
  if (s != HYDRO_OK) return s;
  if (!sl->rec_valid) {
    CU(cudaMemcpy(&sl->rec_host, sl->rec, sizeof(BatchRec), cudaMemcpyDeviceToHost));
    sl->rec_valid = true;
  }
  return HYDRO_OK;
}

hydro_status hydro_batch_count(hydro_ctx* ctx, int64_t batch_id, int64_t* count) {
  if (!ctx || !count) return set_err(HYDRO_EINVAL, "NULL argument");
  Slot* sl = find_slot(ctx, batch_id);
  if (!sl) return set_err(HYDRO_EINVAL, "unknown or already collected batch id");
  hydro_status s = wait_slot(ctx, sl);
  if (s != HYDRO_OK) return s;
  *count = sl->rec_host.total_count;
  return HYDRO_OK;
}

hydro_status hydro_batch_output(hydro_ctx* ctx, int64_t batch_id, const uint32_t** positions,
                                const uint32_t** count, void** done_event) {
  if (!ctx || !positions || !count || !done_event) return set_err(HYDRO_EINVAL, "NULL argument");
  Slot* sl = find_slot(ctx, batch_id);
  if (!sl) return set_err(HYDRO_EINVAL, "unknown or already collected batch_id");
  *positions = sl->out_pos;
  *count = &sl->rec->total_count;
  *done_event = static_cast<void*>(sl->done);
  return HYDRO_OK;
}

hydro_status hydro_collect_results(hydro_ctx* ctx, int64_t batch_id, uint64_t* ids, uint16_t* bboxes,
                                   int64_t capacity, int64_t* count, int32_t out_on_device) {
  if (!ctx || !count) return set_err(HYDRO_EINVAL, "NULL argument");
  Slot* sl = find_slot(ctx, batch_id);
  if (!sl) return set_err(HYDRO_EINVAL, "unknown or already collected batch id");
  hydro_status s = wait_slot(ctx, sl);
  if (s != HYDRO_OK) return s;
  const int64_t c = sl->rec_host.total_count;
  *count = c;
  if (capacity < c) return set_err(HYDRO_ERANGE, "capacity < result count");
  if (c > 0) {
    if (!ids || !bboxes) return set_err(HYDRO_EINVAL, "NULL output buffer");
    // copy on the copy stream after this batch only (the compute stream may already run later batches)
    const cudaMemcpyKind k = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CU(cudaStreamWaitEvent(ctx->copy_stream, sl->done, 0));
    CU(cudaMemcpyAsync(ids, sl->out_ids, 8 * c, k, ctx->copy_stream));
    CU(cudaMemcpyAsync(bboxes, sl->out_bbox, 8 * c, k, ctx->copy_stream));
    CU(cudaStreamSynchronize(ctx->copy_stream));
  }
  sl->busy = false;
  return HYDRO_OK;
}

hydro_status hydro_release_batch(hydro_ctx* ctx, int64_t batch_id) {
  if (!ctx) return set_err(HYDRO_EINVAL, "NULL argument");
  Slot* sl = find_slot(ctx, batch_id);
  if (!sl) return set_err(HYDRO_EINVAL, "unknown or already collected batch id");
  CU(cudaEventSynchronize(sl->done));
  sl->busy = false;
  return HYDRO_OK;
}

hydro_status hydro_batch_info(hydro_ctx* ctx, int64_t batch_id, hydro_batch_report* out) {
  if (!ctx || !out) return set_err(HYDRO_EINVAL, "NULL argument");
  Slot* sl = find_slot(ctx, batch_id);
  if (!sl) return set_err(HYDRO_EINVAL, "unknown or already collected batch id (call before collect)");
  hydro_status s = wait_slot(ctx, sl);
  if (s != HYDRO_OK) return s;
  std::memset(out, 0, sizeof(*out));
  const BatchRec& r = sl->rec_host;
  out->n_tuples = sl->n;
  out->n_results = r.total_count;
  out->warmup_tuples = sl->warm_n;
  out->n_pred = static_cast<int32_t>(ctx->preds.size());
  for (int k = 0; k < kMaxPred; ++k) {
    out->order_used[k] = r.order_used[k];
    out->tuples_in[k] = static_cast<int64_t>(r.d_in[k]);
    out->tuples_passed[k] = static_cast<int64_t>(r.d_pass[k]);
    out->cost_raw[k] = static_cast<double>(r.d_cost[k]);
    out->tuples_computed[k] = static_cast<int64_t>(r.d_comp[k]);
  }
  return HYDRO_OK;
}

static hydro_status read_state(hydro_ctx* ctx, DevState* h) {
  if (!ctx->frozen) return set_err(HYDRO_ESTATE, "no batch submitted yet");
  CU(cudaStreamSynchronize(ctx->stream));
  hydro_status s = check_sticky(ctx);
  if (s != HYDRO_OK) return s;
  CU(cudaMemcpy(h, ctx->st, sizeof(DevState), cudaMemcpyDeviceToHost));
  return HYDRO_OK;
}

hydro_status hydro_get_stats(hydro_ctx* ctx, int32_t k, hydro_pred_stats* out) {
  if (!ctx || !out) return set_err(HYDRO_EINVAL, "NULL argument");
  if (k < 0 || k >= static_cast<int32_t>(ctx->preds.size())) return set_err(HYDRO_EINVAL, "bad pred id");
  DevState h;
  hydro_status s = read_state(ctx, &h);
  if (s != HYDRO_OK) return s;
  out->tuples_in = static_cast<int64_t>(h.tot_in[k]);
  out->tuples_passed = static_cast<int64_t>(h.tot_pass[k]);
  out->cost_per_tuple = h.cost[k];
  out->selectivity = h.sel[k];
  out->rank = h.key[k];
  out->position = h.position[k];
  out->s_in = h.s_in[k];
  out->s_pass = h.s_pass[k];
  out->s_cost = h.s_cost[k];
  out->cost_raw_total = h.tot_cost[k];
  out->tuples_computed = static_cast<int64_t>(h.tot_comp[k]);
  out->cache_hit_rate = h.hit[k];
  out->operand_fp16 = ctx->preds[k].a_fp16;
  out->operand_scale_log2 = ctx->preds[k].w_scale_log2;
  out->fused_pair = (k == ctx->pair_a || k == ctx->pair_b) ? 1 : 0;
  return HYDRO_OK;
}

hydro_status hydro_get_order(hydro_ctx* ctx, int32_t* order, int32_t* n) {
  if (!ctx || !order || !n) return set_err(HYDRO_EINVAL, "NULL argument");
  DevState h;
  hydro_status s = read_state(ctx, &h);
  if (s != HYDRO_OK) return s;
  *n = h.n_pred;
  for (int i = 0; i < h.n_pred; ++i) order[i] = h.order[i];
  return HYDRO_OK;
}

hydro_status hydro_route_workers(hydro_ctx* const* workers, int32_t n, int32_t policy, int32_t* order, double* cost,
                                 double* sel) {
  if (!workers || !order) return set_err(HYDRO_EINVAL, "NULL argument");
  if (n < 1 || n > kMaxPred) return set_err(HYDRO_EINVAL, "n must be in [1, 8]");
  if (policy != HYDRO_POLICY_COST && policy != HYDRO_POLICY_SCORE && policy != HYDRO_POLICY_SELECTIVITY)
    return set_err(HYDRO_EINVAL, "policy must be COST, SCORE or SELECTIVITY");
  WorkerRoute wr{};
  wr.n = n;
  wr.policy = policy;
  for (int i = 0; i < n; ++i) {
    hydro_ctx* w = workers[i];
    if (!w) return set_err(HYDRO_EINVAL, "NULL worker");
    if (w->preds.size() != 1 || !w->frozen) return set_err(HYDRO_EINVAL, "a worker holds one predicate and has run a batch");
    if (w->cfg.device != workers[0]->cfg.device) return set_err(HYDRO_EINVAL, "workers on different devices");
    hydro_status s = hydro_synchronize(w);
    if (s != HYDRO_OK) return s;
    wr.st[i] = w->st;
    wr.sms[i] = static_cast<double>(std::max(w->num_sms, 1));
  }
  hydro_ctx* ctx = workers[0];
  void* buf = nullptr;
  CU(cudaMalloc(&buf, 256));
  int32_t* d_order = static_cast<int32_t*>(buf);
  double* d_cost = reinterpret_cast<double*>(static_cast<char*>(buf) + 64);
  double* d_sel = reinterpret_cast<double*>(static_cast<char*>(buf) + 128);
  hydro_route_workers_kernel<<<1, 32, 0, ctx->stream>>>(wr, d_order, d_cost, d_sel);
  ctx->launches += 1;
  cudaError_t e = cudaGetLastError();
  double h_cost[kMaxPred], h_sel[kMaxPred];
  if (e == cudaSuccess) e = cudaMemcpyAsync(order, d_order, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_cost, d_cost, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_sel, d_sel, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(buf);
  if (e != cudaSuccess) return ctx_fail(ctx, HYDRO_ECUDA, std::string("hydro_route_workers: ") + cudaGetErrorString(e));
  for (int i = 0; i < n; ++i) {
    if (cost) cost[i] = h_cost[i];
    if (sel) sel[i] = h_sel[i];
  }
  return HYDRO_OK;
}

hydro_status hydro_flush_stats(hydro_ctx* ctx) {
  if (!ctx) return set_err(HYDRO_EINVAL, "NULL argument");
  hydro_status s = check_sticky(ctx);
  if (s != HYDRO_OK) return s;
  if (!ctx->exchange || !ctx->frozen) return HYDRO_OK;
  if ((s = fold_and_sync(ctx, nullptr, 0, true)) != HYDRO_OK) return s;
  CU(cudaStreamSynchronize(ctx->stream));
  return check_sticky(ctx);
}

hydro_status hydro_synchronize(hydro_ctx* ctx) {
  if (!ctx) return set_err(HYDRO_EINVAL, "NULL argument");
  CU(cudaStreamSynchronize(ctx->stream));
  return check_sticky(ctx);
}

hydro_status hydro_launch_count(hydro_ctx* ctx, int64_t* launches) {
  if (!ctx || !launches) return set_err(HYDRO_EINVAL, "NULL argument");
  *launches = ctx->launches;
  return HYDRO_OK;
}

hydro_status hydro_set_kernel_timing(hydro_ctx* ctx, int32_t enable) {
  if (!ctx) return set_err(HYDRO_EINVAL, "NULL argument");
  CU(cudaStreamSynchronize(ctx->stream));
  for (TimedLaunch& t : ctx->timed) {
    ctx->event_pool.push_back(t.a);
    ctx->event_pool.push_back(t.b);
  }
  ctx->timed.clear();
  ctx->timing = enable != 0;
  return HYDRO_OK;
}

hydro_status hydro_debug_balance_bounds(hydro_ctx* ctx, uint32_t* out, int32_t capacity, int32_t* n) {
  if (!ctx || !n) return set_err(HYDRO_EINVAL, "NULL argument");
  if (!ctx->bal_bounds || ctx->bal_last_ctas == 0) return set_err(HYDRO_ESTATE, "no data-aware AREA hop ran");
  *n = ctx->bal_last_ctas + 1;
  if (capacity < *n || !out) return set_err(HYDRO_ERANGE, "capacity < G + 1");
  CU(cudaStreamSynchronize(ctx->stream));
  hydro_status s = check_sticky(ctx);
  if (s != HYDRO_OK) return s;
  CU(cudaMemcpy(out, ctx->bal_bounds, sizeof(uint32_t) * (*n), cudaMemcpyDeviceToHost));
  return HYDRO_OK;
}

hydro_status hydro_device_time(hydro_ctx* ctx, int32_t kind, int32_t reset, double* total_ms, int64_t* launches) {
  if (!ctx || !total_ms || !launches) return set_err(HYDRO_EINVAL, "NULL argument");
  if (kind != 1 && kind != 4 && kind != 5) return set_err(HYDRO_EINVAL, "device timers exist for kinds 1, 4, 5");
  DevState h;
  hydro_status s = read_state(ctx, &h);
  if (s != HYDRO_OK) return s;
  *total_ms = static_cast<double>(h.kt_total[kind]) * 1e-6;
  *launches = static_cast<int64_t>(h.kt_count[kind]);
  if (reset) {
    const unsigned long long z[2] = {0ull, 0ull};
    CU(cudaMemcpy(reinterpret_cast<char*>(ctx->st) + offsetof(DevState, kt_total) + 8 * kind, z, 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(reinterpret_cast<char*>(ctx->st) + offsetof(DevState, kt_count) + 8 * kind, z, 8, cudaMemcpyHostToDevice));
  }
  return HYDRO_OK;
}

hydro_status hydro_device_items(hydro_ctx* ctx, int32_t kind, int32_t reset, int64_t* items) {
  if (!ctx || !items) return set_err(HYDRO_EINVAL, "NULL argument");
  if (kind != 1 && kind != 4 && kind != 5) return set_err(HYDRO_EINVAL, "device counters exist for kinds 1, 4, 5");
  DevState h;
  hydro_status s = read_state(ctx, &h);
  if (s != HYDRO_OK) return s;
  *items = static_cast<int64_t>(h.kt_items[kind]);
  if (reset) {
    const unsigned long long z = 0ull;
    CU(cudaMemcpy(reinterpret_cast<char*>(ctx->st) + offsetof(DevState, kt_items) + 8 * kind, &z, 8, cudaMemcpyHostToDevice));
  }
  return HYDRO_OK;
}

hydro_status hydro_kernel_time(hydro_ctx* ctx, int32_t kind, double* total_ms, int64_t* launches) {
  if (!ctx || !total_ms || !launches) return set_err(HYDRO_EINVAL, "NULL argument");
  CU(cudaStreamSynchronize(ctx->stream));
  double tot = 0.0;
  int64_t nl = 0;
  for (TimedLaunch& t : ctx->timed) {
    if (t.kind != kind) continue;
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, t.a, t.b));
    tot += ms;
    ++nl;
  }
  *total_ms = tot;
  *launches = nl;
  return HYDRO_OK;
}

hydro_status hydro_debug_linear(hydro_ctx* ctx, int32_t k, const hydro_tuples* t, float* logits_out,
                                uint16_t* crops_out, uint8_t* verdict_out) {
  if (!ctx || !t) return set_err(HYDRO_EINVAL, "NULL argument");
  if (k < 0 || k >= static_cast<int32_t>(ctx->preds.size()) || !is_classifier(ctx->preds[k].desc.kind))
    return set_err(HYDRO_EINVAL, "pred_id is not a classifier (LINEAR, MLP or HSV) predicate");
  if (!t->on_device) return set_err(HYDRO_EINVAL, "debug_linear needs device tuples");
  if (t->n < 0 || t->n > ctx->cfg.max_batch_tuples) return set_err(HYDRO_EINVAL, "bad n");
  hydro_status s = freeze(ctx);
  if (s != HYDRO_OK) return s;
  ClsParams c = cls_base(ctx, t->frame_id, reinterpret_cast<const uint64_t*>(t->bbox));
  c.dispatch = 0;
  c.explicit_pred = k;
  c.range_base = 0;
  c.range_n = static_cast<uint32_t>(t->n);
  c.bits_out = ctx->warm_bits;
  c.dbg_logits = logits_out;
  c.dbg_crops = crops_out;
  c.dbg_verdict = verdict_out;
  c.collect_stats = 0;
  if ((s = launch_cls(ctx, c, static_cast<uint64_t>(t->n), cls_kind_of(ctx->preds[k].desc.kind))) != HYDRO_OK)
    return s;
  CU(cudaStreamSynchronize(ctx->stream));
  return check_sticky(ctx);
}

hydro_status hydro_cache_fill(hydro_ctx* ctx, int32_t k, const hydro_tuples* t) {
  if (!ctx || !t) return set_err(HYDRO_EINVAL, "NULL argument");
  if (k < 0 || k >= static_cast<int32_t>(ctx->preds.size())) return set_err(HYDRO_EINVAL, "bad pred id");
  if (!ctx->preds[k].cache_known) return set_err(HYDRO_EINVAL, "no verdict cache on this predicate (hydro_cache_enable)");
  if (!t->on_device) return set_err(HYDRO_EINVAL, "cache_fill needs device tuples");
  if (t->n < 0 || t->n > ctx->cfg.max_batch_tuples) return set_err(HYDRO_EINVAL, "bad n");
  hydro_status s = freeze(ctx);
  if (s != HYDRO_OK) return s;
  if (t->n == 0) return HYDRO_OK;
  if (is_classifier(ctx->preds[k].desc.kind)) {  // the classifier alone over the batch, verdicts recorded
    ClsParams c = cls_base(ctx, t->frame_id, reinterpret_cast<const uint64_t*>(t->bbox));
    c.dispatch = 0;
    c.explicit_pred = k;
    c.list_in = nullptr;
    c.range_base = 0;
    c.range_n = static_cast<uint32_t>(t->n);
    c.bits_out = ctx->warm_bits;
    c.collect_stats = 0;
    c.id = t->id;
    c.force_fill = 1;
    if ((s = launch_cls(ctx, c, static_cast<uint64_t>(t->n), cls_kind_of(ctx->preds[k].desc.kind))) != HYDRO_OK)
      return s;
    CU(cudaStreamSynchronize(ctx->stream));
    return check_sticky(ctx);
  }
  RouteParams r = route_base(ctx, t->id, t->frame_id, reinterpret_cast<const uint64_t*>(t->bbox), t->label);
  r.dispatch = 0;
  r.explicit_pred = k;
  r.range_base = 0;
  r.range_n = static_cast<uint32_t>(t->n);
  r.bitmap_out = ctx->warm_bits;
  r.collect_stats = 0;
  r.force_fill = 1;
  if ((s = launch_route(ctx, r, static_cast<uint64_t>(t->n))) != HYDRO_OK) return s;
  CU(cudaStreamSynchronize(ctx->stream));
  return check_sticky(ctx);
}

hydro_status hydro_destroy(hydro_ctx* ctx) {
  if (!ctx) return HYDRO_OK;
  cudaSetDevice(ctx->cfg.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (Slot& s : ctx->slots) {
    if (s.done) cudaEventDestroy(s.done);
    if (s.uploaded) cudaEventDestroy(s.uploaded);
    cudaFree(s.out_ids);
    cudaFree(s.out_bbox);
    cudaFree(s.out_pos);
    cudaFree(s.rec);
    cudaFree(s.s_id);
    cudaFree(s.s_frame);
    cudaFree(s.s_bbox);
    cudaFree(s.s_label);
  }
  for (PredHost& p : ctx->preds) {
    cudaFree(p.w_tiled);
    cudaFree(p.w_tiled_tm);
    cudaFree(p.bias);
    cudaFree(p.w2_tiled);
    cudaFree(p.bias1);
    cudaFree(p.cache_known);
    cudaFree(p.cache_pass);
  }
  for (TimedLaunch& t : ctx->timed) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  cudaFree(ctx->st);
  cudaFree(ctx->preds_dev);
  cudaFree(ctx->lists);
  cudaFree(ctx->counts);
  cudaFree(ctx->bits);
  cudaFree(ctx->warm_bits);
  cudaFree(ctx->pair_w_tiled);
  cudaFree(ctx->pair_bias);
  cudaFree(ctx->cache_idx);
  cudaFree(ctx->cache_pos);
  cudaFree(ctx->cache_count);
  cudaFree(ctx->seg_counts);
  cudaFree(ctx->fused_status);
  cudaFree(ctx->warm_and);
  cudaFree(ctx->bal_chunks);
  cudaFree(ctx->bal_bounds);
  cudaFree(ctx->zero_word);
  if (ctx->xchg_stream) cudaStreamSynchronize(ctx->xchg_stream);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->xchg_stream) cudaStreamDestroy(ctx->xchg_stream);
  for (int i = 0; i < 2; ++i) {
    if (ctx->xchg_ready[i]) cudaEventDestroy(ctx->xchg_ready[i]);
    if (ctx->xchg_done[i]) cudaEventDestroy(ctx->xchg_done[i]);
  }
  if (ctx->host_xfer) cudaFreeHost(ctx->host_xfer);
  if (ctx->user_ev) cudaEventDestroy(ctx->user_ev);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->green) green_api().ctxDestroy(ctx->green);
  delete ctx;
  return HYDRO_OK;
}

}  // extern "C"
