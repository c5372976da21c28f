/*
 * hydro.h -- C ABI of the B200-native eddy hot path of Hydro (arXiv 2403.14902).
 *
 * The library evaluates a CONJUNCTION of (expensive) UDF predicates over a stream of
 * detection tuples, the way Hydro's Eddy does:
 *   SELECT id, bbox FROM video ... WHERE p_1 AND ... AND p_P
 * Per submitted routing batch it
 *   1. orders the predicates by cost / (1 - selectivity), lowest first,
 *   2. runs the next predicate only on the still-alive tuples and drops failures at once
 *      ("eager materialization"),
 *   3. folds per-predicate pass counts and measured costs into running statistics
 *      (PAPER.md:247-249, 416), which fix the order of the next batch.
 * A warmup slice is first evaluated on every predicate.
 *
 * Every step runs in CUDA kernels for sm_100a on the context's stream; the host never
 * synchronises inside a batch (the order lives in device memory).  Readings of points the
 * paper leaves open are numbered R1..R24 in DESIGN.md §2 and cited below.
 *
 * Conventions
 *  - Every function returns hydro_status: HYDRO_OK (0) or a negative error.  No C++
 *    exception crosses the ABI.  hydro_last_error() returns a thread-local message for the
 *    last failure on the calling thread.
 *  - CUDA / NCCL errors raised by asynchronous work are sticky per context and are reported
 *    (HYDRO_ECUDA / HYDRO_ENCCL) by the next call that synchronises (typically collect).
 *  - A context is bound to one device and one stream and is NOT thread-safe (like a cuBLAS
 *    handle); one rank per process, one context per thread.
 *  - Pointers are plain host or device addresses as stated per argument.  The caller owns
 *    every buffer it passes; the library owns its internal device buffers.
 */
#ifndef HYDRO_H
#define HYDRO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hydro_status;
enum {
  HYDRO_OK = 0,
  HYDRO_EINVAL = -1, /* invalid argument (value, size, pointer or layout)                */
  HYDRO_ENOMEM = -2, /* device or host allocation failed                                  */
  HYDRO_ECUDA = -3,  /* CUDA runtime error (sticky; message via hydro_last_error)         */
  HYDRO_ENCCL = -4,  /* NCCL error (sticky)                                               */
  HYDRO_ESTATE = -5, /* call out of lifecycle order (e.g. add_predicate after a submit)   */
  HYDRO_ERANGE = -6, /* caller's output buffer too small; *count holds the needed size    */
  HYDRO_EBUSY = -7   /* all in-flight batch slots hold uncollected results                */
};

/* Routing policy. */
enum {
  HYDRO_POLICY_SCORE = 0,       /* default: cost / (1 - selectivity), lowest first */
  HYDRO_POLICY_STATIC = 1,      /* "Best Reordering": declared cost / selectivity, never updated
                                   (PAPER.md:412-413); no warmup */
  HYDRO_POLICY_FIXED_ORDER = 2, /* "No Reordering" / test hook: the order set by
                                   hydro_set_fixed_order (default: add order) */
  HYDRO_POLICY_COST = 3,        /* cost only */
  HYDRO_POLICY_SELECTIVITY = 4, /* selectivity only */
  HYDRO_POLICY_REUSE = 5        /* reuse-aware: per batch, estimated cost
                                   (1 - cache hit rate of the batch) * cost of computing the UDF,
                                   lowest first; needs verdict caches (hydro_cache_enable) */
};

/* Work distribution of a classifier hop over the persistent K4 CTAs (the hop's "workers";
   SURVEY.md §8(f) f4). */
enum {
  HYDRO_BALANCE_ROUND_ROBIN = 0, /* tile i -> CTA i mod G, the paper's default     */
  HYDRO_BALANCE_DATA_AWARE = 1   /* AREA heads: contiguous position ranges of equal estimated cost,
                                    the input size w*h of each tuple being the cost proxy
                                    (PAPER.md:863-882); NEAREST heads keep round-robin (every
                                    tuple samples 64 rows: its cost does not follow w*h)       */
};

/* Where the per-tuple cost of a predicate comes from (R6). */
enum {
  HYDRO_COST_MEASURED = 0, /* SM-cycles per tuple measured in the kernels (clock64) */
  HYDRO_COST_DECLARED = 1  /* the declared_cost of the predicate; selectivity is still measured */
};

/* Predicate kinds (R5, R12-R14). */
enum {
  HYDRO_PRED_LABEL_EQ = 0, /* label == label_value                                          */
  HYDRO_PRED_HASH = 1,     /* synthetic predicate with set selectivity and per-tuple cost (R5) */
  HYDRO_PRED_LINEAR = 2,   /* argmax(W . Crop(frame, bbox) + b) == target (R10-R14, R19)     */
  HYDRO_PRED_MLP = 3,      /* argmax(W2 . bf16(relu(W1 . Crop + b1)) + b2) == target: the
                              "small MLP classifier" of the north star (
                              stand-in for the ViT breed model; R25)  */
  HYDRO_PRED_HSV = 4       /* DogColorClassifier as the paper implements it (
                              R27): the HSV colour class with most pixels of the 64x64 nearest
                              crop == target (0 red, 1 black, 2 gray, 3 yellow, 4 green, 5 blue,
                              6 purple, 7 pink, 8 white, 9 other); no weights                */
};

enum { HYDRO_CROP_NEAREST = 0, HYDRO_CROP_AREA = 1 }; /* R10 */

#define HYDRO_MAX_PREDICATES 8
#define HYDRO_CROP 64
#define HYDRO_FEATURES 12288 /* 64 * 64 * 3, feature k = (dy*64 + dx)*3 + ch (R10) */
#define HYDRO_MAX_CLASSES 128
#define HYDRO_MLP_HIDDEN_MAX 512 /* MLP hidden width: 256 or 512 */

typedef struct hydro_ctx hydro_ctx; /* opaque */

/* How the ranks of a data-parallel run exchange their statistics deltas. */
enum {
  HYDRO_TRANSPORT_NCCL = 0, /* ncclAllReduce(sum) on a library side stream (default)             */
  HYDRO_TRANSPORT_HOST = 1  /* the caller's host callback (e.g. a gloo all-reduce): synchronous   */
};
/* HOST transport: sums `count` u64 values in place over all ranks (every rank calls it with the
   same count at the same point); returns 0 on success, anything else is reported as HYDRO_ENCCL.
   Called on the thread that called hydro_submit_batch / hydro_flush_stats. */
typedef int32_t (*hydro_allreduce_fn)(void* user, uint64_t* data, int32_t count);

typedef struct {
  int32_t device;            /* CUDA device ordinal                                           */
  void* stream;              /* cudaStream_t to run on (e.g. torch.cuda.current_stream());
                                NULL = a library-owned non-blocking stream                    */
  int32_t policy;            /* HYDRO_POLICY_*                       (default SCORE)          */
  int32_t cost_source;       /* HYDRO_COST_*                         (default MEASURED)       */
  double decay_gamma;        /* S <- gamma*S + delta per fold, in (0,1] (default 0.5; 1 = plain
                                counts) (R4)                                   */
  double prior_selectivity;  /* selectivity with no observation (default 0.5) (R3)           */
  int64_t warmup_tuples;     /* warmup slice of the first batch: evaluated on every predicate
                                without short-circuit (default 65536; 0 disables) (R8)       */
  int64_t max_batch_tuples;  /* largest batch accepted (default 1<<20, max 1<<30)             */
  int32_t max_inflight;      /* uncollected batches held at once (default 4)                 */
  int32_t rank, world;       /* data-parallel rank / world size (default 0 / 1)              */
  int32_t sync_every;        /* world > 1: the statistics exchange (a11) every sync_every batches
                                (default 1).  At each sync point the window of the last
                                sync_every batches' deltas is snapshot and summed over the ranks
                                (NCCL on a side stream, or the HOST callback) and the window of
                                the PREVIOUS sync point is folded: every rank folds identical
                                integers at the same batch, so every rank holds the same order
                                (routing converges by construction), and the exchange is never
                                waited on by the batch that starts it.  The warmup slice's
                                statistics are exchanged and folded at once.  Every rank must
                                submit the same number of batches (empty batches are legal).  */
  const void* nccl_unique_id;/* world > 1: the 128-byte ncclUniqueId from
                                hydro_nccl_unique_id() on rank 0, broadcast by the caller.
                                Also accepted with world == 1 (a 1-rank communicator: the fold
                                then runs the same NCCL all-reduce path as a multi-GPU run)  */
  const uint8_t* frames;     /* DEVICE frame pool, HWC uint8 [n_frames][frame_h][frame_w][3],
                                BORROWED for the context's lifetime (R11); may be NULL when no
                                LINEAR predicate is used                                      */
  int32_t n_frames, frame_h, frame_w; /* frame_w % 16 == 0, frames 16-byte aligned, pool < 64 GiB */
  int32_t balance;           /* HYDRO_BALANCE_*: how a classifier hop's tiles are spread over the
                                SMs (default ROUND_ROBIN)                                     */
  int32_t max_sms;           /* SM budget of the context's persistent kernels (grids capped at
                                this many SMs; 0 = all).  Two contexts with budgets summing to
                                the SM count on two streams run side by side, but the
                                hardware may place their CTAs on any SM                       */
  int32_t sm_groups, sm_group; /* sm_groups >= 2: the context is a worker on its own SM
                                partition -- group sm_group of an even split of the device's
                                SMs into sm_groups CUDA green-context partitions; the context
                                then runs on a library-owned stream of that partition (stream
                                above is ignored) and its grids fit the partition.  Contexts
                                with distinct sm_group values run on disjoint SMs (SURVEY.md
                                §8(f) f3, R29).  0 or 1: the whole device.  The batch's kernels
                                still run after the work enqueued on `stream` (when non-NULL)
                                before the submit (the library stream waits on an event)       */
  int32_t transport;         /* HYDRO_TRANSPORT_* (world > 1, or world == 1 with a HOST callback) */
  hydro_allreduce_fn allreduce_fn; /* HOST transport callback (required for it)                 */
  void* allreduce_user;      /* passed to allreduce_fn                                         */
} hydro_config;

typedef struct {
  int32_t kind;               /* HYDRO_PRED_*                                                  */
  /* LABEL_EQ */
  int32_t label_value;        /* e.g. 16 = COCO 'dog' (R15)                                   */
  /* HASH (R5):  h = hi32(splitmix64(id ^ seed)); repeat units(t) times h = fmix32(h + r);
     pass iff h < T(t), T(t) = threshold[id >= drift_id], T in [0, 2^32]                      */
  uint64_t seed;
  uint64_t threshold[2];
  uint64_t drift_id;          /* UINT64_MAX: no drift                                         */
  int32_t units;              /* rounds per tuple (>= 0) when units_per_area == 0             */
  int32_t units_per_area;     /* > 0: units(t) = ceil(w*h / units_per_area) (cfg4)            */
  /* LINEAR (R12-R14): z = W x + b over the 64x64x3 crop x; pass iff argmax z == target
     (lowest index on ties).  Weights are COPIED at add time.                                 */
  const uint16_t* weight_bf16;/* bf16 bits, row-major [n_classes][HYDRO_FEATURES]             */
  const float* bias;          /* [n_classes]                                                   */
  int32_t weights_on_device;  /* 1: weight_bf16 / bias are device pointers, 0: host pointers  */
  int32_t n_classes;          /* 2 .. HYDRO_MAX_CLASSES                                        */
  int32_t target;             /* 0 .. n_classes-1                                              */
  int32_t crop_mode;          /* HYDRO_CROP_* (MLP: NEAREST only)                              */
  /* MLP (R25): h = bf16_rne(relu(W1 x + b1)) with fp32 accumulation; z = W2 h + b2.  For an MLP
     weight_bf16 / bias are W1 [hidden][HYDRO_FEATURES] / b1 [hidden]; the second layer is below
     (same residency flag, COPIED at add time).                                                */
  int32_t hidden;             /* 256 or 512                                                    */
  const uint16_t* weight2_bf16;/* bf16 bits, row-major [n_classes][hidden]                     */
  const float* bias2;         /* [n_classes]                                                   */
  /* statistics priors (STATIC policy values; DECLARED cost source; used before any fold)    */
  double declared_cost;       /* > 0, same unit as the measured cost for a mixed SCORE policy  */
  double declared_selectivity;/* in [0, 1]                                                     */
} hydro_predicate_desc;

/* One routing batch of detection tuples, SoA (D1).  bbox is [n][4]
   u16 (x0, y0, x1, y1), half-open, inside the frame, w, h >= 1 (R9).  frame_id < n_frames.  */
typedef struct {
  const uint64_t* id;
  const uint32_t* frame_id;
  const uint16_t* bbox;
  const uint16_t* label;
  int64_t n;
  int32_t on_device;          /* 1: DEVICE columns, BORROWED until the batch is collected
                                   (not validated: out-of-range values are clamped in-kernel);
                                 0: HOST columns (pinned memory recommended), validated on the
                                   host, then uploaded asynchronously on the context's copy
                                   stream so batch k+1's upload overlaps batch k's kernels:
                                   BORROWED until the batch is collected                       */
  const uint32_t* sel;        /* optional DEVICE selection (NULL: all n positions): the batch is
                                 the positions sel[0 .. *sel_count) of the columns, in that order
                                 (each < the columns' length, ascending for input-order output);
                                 n is then an upper bound of *sel_count.  Device columns only; no
                                 warmup slice runs on a selection batch; not with REUSE.  Used to
                                 chain workers (hydro_batch_output of another context)          */
  const uint32_t* sel_count;  /* DEVICE count of sel (read by the kernels, never by the host)   */
  void* wait_event;           /* optional cudaEvent_t the context stream waits on before the
                                 batch's kernels (e.g. the producer batch's done_event)         */
} hydro_tuples;

typedef struct {
  int64_t tuples_in;          /* cumulative tuples routed to the predicate (all batches)      */
  int64_t tuples_passed;      /* cumulative tuples it passed                                   */
  double cost_per_tuple;      /* current estimate c (SM-cycles per tuple, or declared)         */
  double selectivity;         /* current estimate s                                            */
  double rank;                /* policy key (c/(1-s) for SCORE)                                */
  int32_t position;           /* position in the current order (0 = first)                     */
  double s_in, s_pass, s_cost;/* decayed counters S (R4)                                       */
  double cost_raw_total;      /* cumulative measured raw cycles                                */
  int64_t tuples_computed;    /* cumulative tuples actually evaluated (not served by the verdict
                                 cache); == tuples_in without a cache                           */
  double cache_hit_rate;      /* REUSE policy: the last batch's cache hit rate (0 otherwise)   */
  int32_t operand_fp16;       /* LINEAR / MLP: 1 when the contraction runs on fp16 operands (every
                                 weight exactly representable in fp16, after the power-of-two
                                 rescale below: the same products as bf16), 0 on bf16 operands;
                                 0 for other kinds                                               */
  int32_t operand_scale_log2; /* LINEAR: k of the exact rescale W' = 2^k W that makes a general
                                 bf16 head fp16-exact (logits are multiplied by 2^-k, exactly,
                                 before the bias); 0 when none was needed or possible             */
  int32_t fused_pair;         /* 1: this LINEAR head is one of the context's fused pair (two nearest
                                 heads evaluated in one K4-T contraction whenever the order puts
                                 them next to each other; counters as if evaluated in turn)      */
} hydro_pred_stats;

/* Per-batch record, available after the batch completed (hydro_batch_info). */
typedef struct {
  int64_t n_tuples;
  int64_t n_results;
  int64_t warmup_tuples;      /* size of the warmup slice evaluated on every predicate (R8)   */
  int32_t order_used[HYDRO_MAX_PREDICATES]; /* order for the post-warmup part of the batch    */
  int64_t tuples_in[HYDRO_MAX_PREDICATES];  /* this batch's counters (warmup included)         */
  int64_t tuples_passed[HYDRO_MAX_PREDICATES];
  double cost_raw[HYDRO_MAX_PREDICATES];
  int64_t tuples_computed[HYDRO_MAX_PREDICATES]; /* evaluated, not served by the verdict cache  */
  int32_t n_pred;
} hydro_batch_report;

/* ---------------------------------------------------------------------------------------- */

const char* hydro_version(void);
const char* hydro_last_error(void);

/* Fills *cfg with the defaults listed above (device 0, NULL stream, SCORE, MEASURED ...). */
hydro_status hydro_config_default(hydro_config* cfg);

/* world > 1 only: writes a fresh 128-byte ncclUniqueId to out128 (host).  Call on rank 0 and
   broadcast it to the other ranks before hydro_create. */
hydro_status hydro_nccl_unique_id(void* out128);

/* Creates a context on cfg->device.  EINVAL on bad sizes; ENOMEM; ENCCL when the communicator
   cannot be formed (world > 1; collective over all ranks).  EINVAL: REUSE policy with world > 1
   (its order is per batch, from that batch's own cache hit rates, which differ between ranks),
   HOST transport without a callback. */
hydro_status hydro_create(const hydro_config* cfg, hydro_ctx** out);

/* Registers predicate number *pred_id = 0, 1, 2 ... (call order = the conjunction's textual
   order = the FIXED_ORDER default).  At most HYDRO_MAX_PREDICATES.  ESTATE after the first
   submit.  EINVAL: n_classes out of range, target outside [0, n_classes), threshold > 2^32,
   negative units, LINEAR / MLP without a frame pool, MLP with hidden not in {256, 512} or an
   AREA crop, declared values out of range. */
hydro_status hydro_add_predicate(hydro_ctx* ctx, const hydro_predicate_desc* desc, int32_t* pred_id);

/* Verdict cache for reuse-aware routing: predicate
   pred_id (any kind: LABEL_EQ, HASH, or a classifier -- LINEAR, MLP, HSV, the expensive UDFs
   UC2 reuses) keeps a device bitmap of known verdicts over tuple ids [0, id_capacity) (2 bits
   per id, library-owned).  A cached verdict is used instead of evaluating the predicate (the
   result is unchanged: the cache holds the predicate's verdicts): a cheap predicate looks its
   alive tuples up inside K1; a classifier hop is first split by K0c into cached verdicts and the
   uncached tuples, and only those go through the classifier kernel.  Cost statistics count only
   evaluated tuples (the cost of computing the UDF).  fill = 1 also records every verdict the
   predicate computes.  Any time no batch is in flight (ESTATE otherwise); EINVAL for
   id_capacity 0 or > 2^34, or a second call.  The first cache on a classifier allocates two
   u32 lists of max_batch_tuples (ENOMEM / ECUDA on failure). */
hydro_status hydro_cache_enable(hydro_ctx* ctx, int32_t pred_id, uint64_t id_capacity, int32_t fill);

/* Records verdicts[i] (0 / 1) of predicate pred_id for tuple ids[i], i < n (e.g. the results of
   an earlier query that evaluated the same UDF).  Ordered on the context stream; ids and
   verdicts are host arrays (copied before return) or device arrays (on_device = 1, borrowed
   until the next synchronising call).  ids >= id_capacity are ignored.  The caller vouches
   that the verdicts are the predicate's.  EINVAL without an enabled cache. */
hydro_status hydro_cache_put(hydro_ctx* ctx, int32_t pred_id, const uint64_t* ids, const uint8_t* verdicts,
                             int64_t n, int32_t on_device);

/* Evaluates predicate pred_id alone on every tuple of the DEVICE batch `tuples` (K1 for a cheap
   predicate, its classifier kernel for LINEAR / MLP / HSV) and records its verdicts in its cache
   -- the exploratory single-UDF queries whose results a later query reuses (Q1 / Q2 of
   PAPER.md:565-570).  Statistics untouched.  Synchronises.  EINVAL without an enabled cache or
   with host tuples. */
hydro_status hydro_cache_fill(hydro_ctx* ctx, int32_t pred_id, const hydro_tuples* tuples);

/* FIXED_ORDER policy: sets the order (a permutation of 0..P-1).  EINVAL if not a permutation. */
hydro_status hydro_set_fixed_order(hydro_ctx* ctx, const int32_t* order, int32_t n);

/* Enqueues one routing batch on the context's stream and returns its id (0, 1, 2 ...).
   Asynchronous: returns before the GPU work finishes.  n == 0 is legal (0 results).
   EINVAL: n > max_batch_tuples, NULL columns, invalid host tuples.  EBUSY: max_inflight
   batches are uncollected.  The results are the passing (id, bbox) rows in input order.
   The columns (host or device) must stay valid until the batch is collected or released. */
hydro_status hydro_submit_batch(hydro_ctx* ctx, const hydro_tuples* tuples, int64_t* batch_id);

/* Blocks until batch_id finished and returns its result count. */
hydro_status hydro_batch_count(hydro_ctx* ctx, int64_t batch_id, int64_t* count);

/* Blocks until batch_id finished, then copies its rows: ids[count] (u64) and bboxes[count][4]
   (u16), in input order, to HOST (out_on_device = 0) or DEVICE (1) buffers, and releases the
   batch slot.  capacity < count: ERANGE with *count set and the batch kept. */
/* The survivors of an uncollected batch as DEVICE data, for chaining a second context (worker)
   without a host round trip: *positions = their input positions (u32, input
   order), *count = device pointer to their number, *done_event = the cudaEvent_t recorded when
   the batch completes (pass it as the consumer's hydro_tuples.wait_event).  The pointers stay
   valid until the batch is collected or released.  Non-blocking.                                */
hydro_status hydro_batch_output(hydro_ctx* ctx, int64_t batch_id, const uint32_t** positions,
                                const uint32_t** count, void** done_event);

hydro_status hydro_collect_results(hydro_ctx* ctx, int64_t batch_id, uint64_t* ids, uint16_t* bboxes,
                                   int64_t capacity, int64_t* count, int32_t out_on_device);

/* Releases a batch slot without copying (results dropped). */
hydro_status hydro_release_batch(hydro_ctx* ctx, int64_t batch_id);

/* Per-batch counters and the order used (after the batch finished). */
hydro_status hydro_batch_info(hydro_ctx* ctx, int64_t batch_id, hydro_batch_report* out);

/* Snapshot of predicate pred_id's statistics after the last fold (synchronises the stream). */
hydro_status hydro_get_stats(hydro_ctx* ctx, int32_t pred_id, hydro_pred_stats* out);

/* Current order (synchronises): order[0..P-1]; *n = P. */
hydro_status hydro_get_order(hydro_ctx* ctx, int32_t* order, int32_t* n);

/* Router of concurrent workers ("cost-driven routing" when
   the predicates' workers run concurrently; R29).  workers[i] (i < n <= 8) is a context holding ONE
   predicate (worker i), normally on its own SM partition (sm_groups / sm_group), that has folded
   statistics (e.g. after a warmup batch every worker evaluated).  A device kernel
   takes, per worker, its time per tuple c_i = (SM-cycles per tuple, R6) / (the worker's SM count)
   and its selectivity s_i, and writes order[0..n) = the workers sorted by the policy key, lowest
   first, ties by index (R2): HYDRO_POLICY_COST c, HYDRO_POLICY_SCORE c / (1 - s)
   (R1), HYDRO_POLICY_SELECTIVITY s.  cost / sel (host, nullable) receive c_i and
   s_i.  Synchronises every worker's stream.  EINVAL: n outside [1, 8], a NULL worker, a worker
   with a predicate count != 1 or no batch yet, workers on different devices, other policies. */
hydro_status hydro_route_workers(hydro_ctx* const* workers, int32_t n, int32_t policy, int32_t* order, double* cost,
                                 double* sel);

/* Multi-rank only (a no-op otherwise): folds the outstanding exchanged window, then exchanges and
   folds the deltas of the batches since the last sync point, so every rank's statistics and order
   cover every batch.  Collective: every rank calls it at the same point.  Synchronises. */
hydro_status hydro_flush_stats(hydro_ctx* ctx);

/* Waits for all enqueued work of the context. */
hydro_status hydro_synchronize(hydro_ctx* ctx);

/* Number of kernels the library has launched so far (evidence for bench "gpu_launches"). */
hydro_status hydro_launch_count(hydro_ctx* ctx, int64_t* launches);

/* Kernel timing (CUDA events on the context stream around every launch of the kind):
   enable = 1 starts recording (and clears), 0 stops.  kind: 0 = route kernel (K1, cheap
   predicates), 1 = linear classifier kernel (K4), 2 = fold (K5), 3 = compaction / emit kernel
   (K2), 4 = MLP classifier kernel (K4-MLP), 5 = HSV classifier kernel (K4-HSV), 6 = data-aware
   balance kernels (K6, 2 kernels per launch).  hydro_kernel_time synchronises and returns the
   summed milliseconds and the number of launches recorded since the last enable. */
hydro_status hydro_set_kernel_timing(hydro_ctx* ctx, int32_t enable);

/* Debug (tests): the position bounds K6 computed for the most recent launch of a data-aware
   classifier hop (HYDRO_BALANCE_DATA_AWARE with an AREA head):
   out[c], c = 0..G, CTA c of that K4 launch owned hop-input positions [out[c], out[c+1]).  The
   bounds are only meaningful if that hop was an AREA hop (K6 exits on other hops).  Writes
   *n = G + 1; HYDRO_ERANGE (with *n set) when capacity < G + 1; HYDRO_ESTATE when the context
   has no data-aware AREA head or no hop ran yet.  Synchronises the context stream.           */
hydro_status hydro_debug_balance_bounds(hydro_ctx* ctx, uint32_t* out, int32_t capacity, int32_t* n);
hydro_status hydro_kernel_time(hydro_ctx* ctx, int32_t kind, double* total_ms, int64_t* launches);

/* Device launch timers of the classifier kernels (kind 1 = K4 linear, 4 = K4-MLP, 5 = K4-HSV),
   always on and free of host events: every launch that evaluates a hop adds (%globaltimer at its
   last CTA's end - at its first CTA's start) to the kind's total.  Returns the summed
   milliseconds and the launch count (synchronises the context stream); reset = 1 then zeroes them. */
hydro_status hydro_device_time(hydro_ctx* ctx, int32_t kind, int32_t reset, double* total_ms, int64_t* launches);

/* The classifier-input tuples (crops) the same kinds' launches evaluated, counted on the device
   (a fused linear pair's crops once); reset = 1 then zeroes the count.  Synchronises. */
hydro_status hydro_device_items(hydro_ctx* ctx, int32_t kind, int32_t reset, int64_t* items);

/* Destroys the context (synchronises first).  Safe on NULL. */
hydro_status hydro_destroy(hydro_ctx* ctx);

/* ---- debug hooks (tests) ---------------------------------------------------------------- */

/* Runs predicate pred_id's classifier kernel (LINEAR, MLP or HSV; for HSV the "logits" are the
   10 colour-class pixel counts) on every tuple of the DEVICE batch `tuples`
   (no short-circuit, statistics untouched) and writes, when non-NULL, the f32 logits
   logits_out[n][n_classes] (device) and the bf16 crop features crops_out[n][HYDRO_FEATURES]
   (device, bf16 bits) plus the verdicts verdict_out[n] (device, uint8 0/1).  Synchronises. */
hydro_status hydro_debug_linear(hydro_ctx* ctx, int32_t pred_id, const hydro_tuples* tuples,
                                float* logits_out, uint16_t* crops_out, uint8_t* verdict_out);

#ifdef __cplusplus
}
#endif
#endif /* HYDRO_H */
