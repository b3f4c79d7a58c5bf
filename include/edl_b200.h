/*
 * edl_b200.h — C ABI of the B200-native elastic data-parallel SGD hot path.
 *
 * Drop-in boundary for the reference EDL implementation (/root/reference/proj, C++20).
 * Every entry point names the reference interface it replaces (file:line, relative to
 * /root/reference/proj).  Conventions:
 *   - plain pointers and sizes only; no C++ or torch types cross this boundary;
 *   - no exceptions cross it: each reference exception class maps to an EDL_E* code and
 *     the message is kept in a thread-local string read by edl_last_error();
 *   - "_dev" pointers are caller-owned device buffers on the current CUDA device; the
 *     `stream` argument is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - worker ids are NUL-terminated strings, as in the reference (std::string).
 */
#ifndef EDL_B200_H
#define EDL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status codes
 * Union of ReduceStatus (include/edl/allreduce.hpp:39), PipeStatus
 * (include/edl/datapipeline.hpp:53), SendStatus (include/edl/transport.hpp:51) and the
 * exception classes thrown by trainer.cpp / dataset.cpp / bytes.hpp.                  */
enum {
  EDL_OK = 0,
  EDL_RETRY = 1,               /* a scaling operation is in flight          */
  EDL_EINVAL = 2,              /* std::invalid_argument (trainer.cpp:16-17,57-58), Invalid */
  EDL_PEER_GONE = 3,           /* ReduceStatus::PeerGone                                  */
  EDL_TIMEOUT = 4,             /* ReduceStatus::Timeout                                   */
  EDL_VERSION_MISMATCH = 5,    /* ReduceStatus::VersionMismatch                           */
  EDL_UNKNOWN_WORKER = 6,      /* PipeStatus::UnknownWorker                               */
  EDL_STALE_SHARD = 7,         /* PipeStatus::StaleShard                                  */
  EDL_SHAPE_MISMATCH = 8,      /* PipeStatus::ShapeMismatch                               */
  EDL_OUT_OF_RANGE = 9,        /* std::out_of_range (dataset.cpp:37)                      */
  EDL_ECUDA = 10,              /* CUDA runtime / driver failure                           */
  EDL_ENOMEM = 11,             /* allocation failure                                      */
  EDL_ALLOWANCE_EXCEEDED = 12, /* scale_in leaver missed its allowance      */
  EDL_EIO = 13,                /* std::runtime_error on file I/O (trainer.cpp:104)        */
  EDL_ETRUNCATED = 14,         /* std::runtime_error "truncated payload" (bytes.hpp:112)  */
  EDL_NO_CHECKPOINT = 15       /* consistent recovery without a checkpoint  */
};

const char* edl_last_error(void);
const char* edl_version(void);

/* ------------------------------------------------------------------ enums */
enum { EDL_MODEL_LEAST_SQUARES = 0, EDL_MODEL_LOGISTIC = 1, EDL_MODEL_MLP = 2 }; /* trainer.hpp:18 */
enum { EDL_REDUCE_SUM = 0, EDL_REDUCE_AVERAGE = 1 };                           /* allreduce.hpp:25 */
enum { EDL_DTYPE_F64 = 0, EDL_DTYPE_BF16 = 1, EDL_DTYPE_F32 = 2 };
enum { EDL_NEXT_SHARD = 0, EDL_NEXT_EPOCH_END = 1, EDL_NEXT_PENDING = 2 };    /* datapipeline.hpp:51 */

/* ================================================================== partition leasing
 * Replaces edl::ShardManager (include/edl/datapipeline.hpp:58-127, src/datapipeline.cpp).
 * Bit-compatible: same std::mt19937_64 + std::shuffle permutation stream, same
 * reclaimed-first hand-out order and the same snapshot byte layout.                     */
typedef struct EdlLeaseManager EdlLeaseManager;

typedef struct {
  uint32_t index;   /* PartitionMeta::index  */
  uint64_t offset;  /* PartitionMeta::offset (first global sample id) */
  uint64_t length;  /* PartitionMeta::length */
} EdlPartitionMeta;

typedef struct {
  int32_t kind;            /* EDL_NEXT_SHARD | EDL_NEXT_EPOCH_END | EDL_NEXT_PENDING */
  EdlPartitionMeta meta;   /* valid for EDL_NEXT_SHARD                              */
  uint64_t resume_offset;  /* Shard::resume_offset                                  */
  uint64_t epoch;          /* EpochEnd::epoch                                       */
} EdlNextShard;

/* default_partition_count, datapipeline.cpp:9-11 */
int32_t edl_default_partition_count(int32_t max_expected_workers);
/* ShardManager::ShardManager, datapipeline.cpp:13-17 */
int edl_lease_create(uint64_t dataset_size, int32_t partitions, uint64_t seed,
                     const char* locator, EdlLeaseManager** out);
void edl_lease_destroy(EdlLeaseManager* lm);
/* register_worker / unregister_worker / is_registered, datapipeline.cpp:26-32 */
int edl_lease_register(EdlLeaseManager* lm, const char* worker);
int edl_lease_unregister(EdlLeaseManager* lm, const char* worker);
int edl_lease_is_registered(const EdlLeaseManager* lm, const char* worker);
/* next_shard, datapipeline.cpp:43-62; returns EDL_UNKNOWN_WORKER like PipeStatus */
int edl_lease_next(EdlLeaseManager* lm, const char* worker, EdlNextShard* out);
/* report_progress, datapipeline.cpp:64-71 */
int edl_lease_report(EdlLeaseManager* lm, const char* worker, uint32_t partition,
                     uint64_t next_sample_offset);
/* reclaim / reclaim_at / reclaim_missing, datapipeline.cpp:73-104 */
int edl_lease_reclaim(EdlLeaseManager* lm, const char* worker);
int edl_lease_reclaim_at(EdlLeaseManager* lm, const char* worker, const uint32_t* partitions,
                         const uint64_t* offsets, size_t n);
int edl_lease_reclaim_missing(EdlLeaseManager* lm, const char* const* live, size_t n);
/* partition_meta, datapipeline.cpp:34-41 */
int edl_lease_partition_meta(const EdlLeaseManager* lm, uint32_t index, EdlPartitionMeta* out);
/* worker_shards, datapipeline.cpp:106-113; returns count, fills up to cap entries */
size_t edl_lease_worker_shards(const EdlLeaseManager* lm, const char* worker,
                               uint32_t* partitions, uint64_t* offsets, size_t cap);
/* snapshot / restore, datapipeline.cpp:115-178 (identical byte layout).
 * snapshot: writes up to cap bytes, stores the full size in *len.                      */
int edl_lease_snapshot(const EdlLeaseManager* lm, uint8_t* buf, size_t cap, size_t* len);
int edl_lease_restore(EdlLeaseManager* lm, const uint8_t* buf, size_t len);
/* accessors, datapipeline.hpp:86-95 */
uint64_t edl_lease_epoch(const EdlLeaseManager* lm);
uint64_t edl_lease_epochs_completed(const EdlLeaseManager* lm);
uint64_t edl_lease_cursor(const EdlLeaseManager* lm);
size_t edl_lease_permutation(const EdlLeaseManager* lm, uint32_t* out, size_t cap);
size_t edl_lease_reclaimed_count(const EdlLeaseManager* lm);
size_t edl_lease_in_flight_count(const EdlLeaseManager* lm);

/* ================================================================== batch splits
 * split_batch (absent in the reference): sizes floor/ceil(B/p), larger
 * shares to the lowest ranks.  Returns EDL_EINVAL when B < p or p < 1.                   */
int edl_split_batch(int64_t B, int32_t p, int64_t* out);
/* k = max(1, ceil(T_a / T_b)) */
int64_t edl_switch_delay(double t_a_ms, double t_b_ms);
/* eta_at, trainer.hpp:27-29 */
double edl_eta_at(double eta, double decay, uint64_t t);

/* ================================================================== synthetic dataset
 * Replaces edl::SyntheticDataset (dataset.hpp:25-50, dataset.cpp:11-58), materialised
 * once in HBM.  Features are bit-identical to SyntheticDataset::get; with dtype F64 the
 * labels are bit-identical too (sequential, FMA-free dot product as dataset.cpp:49).
 * dtype BF16 (the MLP workload) stores features rounded f64 -> f32 -> bf16 (RNE) and
 * int32 class labels  splitmix64(seed ^ ~(i*0xd1342543de82ef95+1)) % num_classes.        */
typedef struct EdlDataset EdlDataset;
typedef struct {
  uint64_t size;
  int32_t dim;
  uint64_t seed;
  double noise;
  int32_t sign_labels;
} EdlSyntheticSpec;

int edl_dataset_create_synthetic(const EdlSyntheticSpec* spec, int32_t dtype,
                                 int32_t num_classes, EdlDataset** out);
void edl_dataset_destroy(EdlDataset* ds);
uint64_t edl_dataset_size(const EdlDataset* ds);
int32_t edl_dataset_dim(const EdlDataset* ds);
/* device pointers: features [size][dim] (f64 or bf16), labels [size] (f64 or int32) */
const void* edl_dataset_features(const EdlDataset* ds);
const void* edl_dataset_labels(const EdlDataset* ds);
/* SyntheticDataset::true_weights (host copy, dim doubles) */
int edl_dataset_true_weights(const EdlDataset* ds, double* out);
/* SyntheticDataset::get (dataset.cpp:36-54): D2H copy of one sample; EDL_OUT_OF_RANGE
 * when index >= size.  features_out holds dim doubles (bf16 datasets are widened).      */
int edl_dataset_get(const EdlDataset* ds, uint64_t index, double* features_out,
                    double* label_out);

/* A contiguous run of sample ids [first, first+count) — what one shard lease yields. */
typedef struct {
  uint64_t first;
  uint64_t count;
} EdlRun;

/* Coalesced gather of leased runs into a contiguous batch: x_out [n][dim] in the
 * dataset's dtype, y_out [n] labels.  runs_dev may be a device or mapped-host pointer.  */
int edl_gather(const EdlDataset* ds, const EdlRun* runs_dev, int32_t n_runs, int64_t n_rows,
               void* x_out_dev, void* y_out_dev, void* stream);

/* ================================================================== linear trainer (f64)
 * Device versions of trainer.cpp.  All reproduce the reference's operation order
 * (sequential per-sample accumulation, no FMA contraction) and are bit-identical.       */
/* local_gradient, trainer.cpp:30-39: grad_out_dev[0..dim) = grad_sum, grad_out_dev[dim]
 * = count (the allreduce convention of trainer.cpp:244-254).                            */
int edl_local_gradient(int32_t kind, const double* w_dev, const double* x_dev,
                       const double* y_dev, int64_t n, int32_t dim, double* grad_out_dev,
                       void* stream);
/* batch_loss, trainer.cpp:41-54 */
int edl_batch_loss(int32_t kind, const double* w_dev, const double* x_dev, const double* y_dev,
                   int64_t n, int32_t dim, double* loss_out_dev, void* stream);
/* sgd_step, trainer.cpp:56-61: w -= (eta / count) * g.  count is read from
 * g_dev[dim] when count < 0 (device-side count), otherwise the given value.
 * EDL_EINVAL when count == 0.                                                           */
int edl_sgd_step(double* w_dev, const double* g_dev, int64_t count, double eta, int32_t dim,
                 void* stream);

/* ================================================================== collective
 * ring_allreduce (allreduce.cpp:60-130) executed as one kernel over n device buffers
 * (local workers, or peer buffers mapped over NVLink).  Chunk c = [c*len/n, (c+1)*len/n)
 * folds ranks c, c+1, ..., c+n-1 left to right (ring_order_reduce, allreduce.cpp:132-148)
 * so the f64 result is bit-identical to the reference collective.  `out_dev` receives
 * the reduced vector; inputs are untouched.                                             */
int edl_ring_allreduce_f64(const double* const* inputs_dev, int32_t n, size_t len,
                           int32_t op, double* out_dev, void* stream);

/* ================================================================== MLP step kernels  */
/* tcgen05/TMA GEMM: C[M][N] = sum_k A(m,k) B(n,k), bf16 in, fp32 accumulate.
 * a_mn = 0: A row-major [M][lda];  a_mn = 1: A row-major [K][lda] (A^T stored).
 * b_mn = 0: B row-major [N][ldb];  b_mn = 1: B row-major [K][ldb].
 * Epilogue: optional ReLU, optional mask (C = 0 where mask <= 0, mask [M][ldm] bf16),
 * bf16 or fp32 output.  bn = N tile (0 = auto).                                         */
int edl_gemm_bf16(const void* A, int32_t lda, int32_t a_mn, const void* B, int32_t ldb,
                  int32_t b_mn, void* C, int32_t ldc, int32_t M, int32_t N, int32_t K,
                  int32_t relu, int32_t out_f32, const void* mask, int32_t ldm, int32_t bn,
                  void* stream);

/* ================================================================== elastic job runtime
 * The reference runtime is absent (CMake lists src/runtime.cpp, which does not exist);
 * its API is specified in SPEC.md:272-392 / PAPER.md Table 1.  A job owns the partition
 * leases (leader role), the versioned ring (Topology, include/edl/topology.hpp:13-51),
 * the per-worker batch splits, the assignment log (trainer.hpp:59-90) and one model
 * replica per GPU.  Mini-batch protocol: see DESIGN.md §3 (identical to
 * oracle/job_driver.hpp).                                                              */
typedef struct EdlJob EdlJob;

typedef struct {
  int32_t model;             /* EDL_MODEL_LEAST_SQUARES | EDL_MODEL_LOGISTIC | EDL_MODEL_MLP */
  EdlSyntheticSpec data;     /* synthetic dataset (dataset.hpp:32-38)                      */
  int32_t num_classes;       /* MLP: classes of the softmax layer                          */
  int32_t layers;            /* MLP: number of Linear layers (ReLU between them)           */
  int32_t hidden;            /* MLP: width of hidden layers                                */
  double eta;                /* HyperParams::eta   (trainer.hpp:20)                        */
  double decay;              /* HyperParams::decay                                         */
  double momentum;           /* 0 = plain sgd_step (reference)                             */
  int64_t batch;             /* aggregate batch B, constant across scaling   */
  int64_t per_worker_batch;  /* > 0: fixed per-worker batch (static throughput sweeps)     */
  uint64_t lease_seed;       /* ShardManager seed                                          */
  int32_t partitions;        /* 0 = default_partition_count(max_workers)                   */
  int32_t max_workers;       /* expected maximum parallelism                               */
  uint64_t init_seed;        /* MLP weight init seed                                       */
  double t_a_ms;             /* switch allowance T_a, default 500             */
  int32_t keep_log;          /* record the assignment log                                  */
  int32_t dry_run;           /* host protocol only (leases, ring, log): no device work      */
  int32_t appx_recovery;     /* keep the mini-batch boundary state for approximate recovery
                                (USE_APPX_RECOVERY; default from that env var) */
} EdlJobConfig;

typedef struct {
  uint64_t t;         /* mini-batch index described                                         */
  uint64_t version;   /* topology version in effect for this mini-batch                     */
  int32_t ring_size;  /* workers in the ring                                                */
  int32_t switched;   /* 1 when a topology switch was installed right before this batch     */
  uint64_t count;     /* samples in the global mini-batch                                   */
  double loss;        /* mean loss over the global mini-batch, before the update (NaN if
                         not yet known)                                                     */
  double step_ms;     /* device time of the mini-batch (CUDA events)                        */
  double stall_ms;    /* device idle time between the previous mini-batch and this one     */
} EdlStepReport;

void edl_job_config_default(EdlJobConfig* cfg);
/* ring: worker ids in rank order; devices: CUDA device hosting each worker */
int edl_job_create(const EdlJobConfig* cfg, const char* const* ring, const int32_t* devices,
                   int32_t n, EdlJob** out);
/* One process per GPU, scale-out: a newcomer process's job.  ring: the
 * job's current ring (all hosted by other processes); newcomers: every worker joining at
 * switch_t (one process each); self_id (one of them) is built now on `device` while the ring
 * keeps stepping.  The ring's processes schedule the same event with device -1
 * (edl_job_schedule) and copy the model into the newcomers over NVLink at the switch.  rank
 * orders this replica after the existing ones.  Handles are exchanged (edl_job_export /
 * edl_job_import) before the switch; until then edl_job_step replays the lease protocol
 * without device work.                                                                   */
int edl_job_create_joining(const EdlJobConfig* cfg, const char* const* ring, int32_t n,
                           const char* const* newcomers, int32_t n_new, const char* self_id,
                           int32_t device, int32_t rank, int64_t switch_t, EdlJob** out);
void edl_job_destroy(EdlJob* job);
/* One mini-batch on every ring member with notify_batch_end folded in:
 * due topology switches are installed first.  Asynchronous: fills t/version/ring/count
 * and returns once the device work is enqueued.                                        */
int edl_job_step(EdlJob* job, EdlStepReport* rep);
/* Waits for the last launched mini-batch and fills its full report.                   */
int edl_job_sync(EdlJob* job, EdlStepReport* rep);
/* scale_out: newcomers are prepared on a side thread while the job keeps
 * stepping; they join at switch_t = t + max(1, ceil(T_a / T_b)).  EDL_RETRY while another
 * scaling operation is pending.                                           */
int edl_job_scale_out(EdlJob* job, const char* const* ids, const int32_t* devices, int32_t n,
                      int64_t* switch_t);
/* scale_in: leavers train until switch_t, then their leases are
 * reclaimed (datapipeline.cpp:73-84) and they leave; no restart.                        */
int edl_job_scale_in(EdlJob* job, const char* const* ids, int32_t n, double allowance_ms,
                     int64_t* switch_t);
/* Scripted topology event at an explicit switch step (test and benchmark protocols).    */
int edl_job_schedule(EdlJob* job, int64_t switch_t, int32_t out, const char* const* ids,
                     const int32_t* devices, int32_t n);
/* Parameters of a worker's replica: linear f64[dim]; MLP fp32 master [param_count].    */
int edl_job_params(EdlJob* job, const char* worker, void* host_out, size_t bytes);
/* Checkpoint restore into every replica (same layout as edl_job_params).                */
int edl_job_set_params(EdlJob* job, const void* host, size_t bytes);
size_t edl_job_param_count(const EdlJob* job);
uint64_t edl_job_t(const EdlJob* job);
double edl_job_median_step_ms(const EdlJob* job);
/* Assignment log in the reference text format (trainer.cpp:79-100).                    */
int edl_job_log(const EdlJob* job, char* buf, size_t cap, size_t* len);
int edl_job_ring(const EdlJob* job, char* buf, size_t cap, size_t* len);
int edl_job_lease_snapshot(const EdlJob* job, uint8_t* buf, size_t cap, size_t* len);
/* Instrumentation (bench.py): the CUDA stream the job's kernels run on (cudaStream_t);
 * per-phase device time from CUDA events recorded on that stream while profiling is on
 * (phase_ms[6] = gather, forward GEMMs, loss, backward GEMMs, allreduce+update, and the
 * weight-gradient GEMMs alone — a sub-phase of the backward), the steps
 * profiled and the number of library kernels launched since the last reset.            */
void* edl_job_stream(const EdlJob* job);
/* How the N>1 gradient exchange of this job runs (valid after the first step): 0 one fused
 * reduce-scatter + SGD + all-gather kernel after the backward, 1 per-layer side-stream
 * collectives, 2 per-layer copy-engine transfers, 3 reduce-scatter routed from the
 * weight-gradient GEMM epilogues + push all-gather, 4 the whole exchange inside the
 * weight-gradient GEMMs, 5 reduce-scatter as per-layer copy-engine peer copies under the
 * backward + push all-gather (the default with one member per GPU on two GPUs), 6 the
 * reduce-scatter split between the GEMM epilogues (nearest peers) and the copy engines
 * (the default from three GPUs).                                                          */
int edl_job_exchange_mode(const EdlJob* job);
/* Orders the job stream (edl_job_stream) after all device work of the launched mini-batches,
 * including the push collective that exchange mode 3 defers onto a side stream to overlap
 * the next mini-batch's forward.  No host synchronisation: record a CUDA event on the job
 * stream after this call to time a sequence of edl_job_step calls. */
int edl_job_join(EdlJob* job);
/* Multi-process data parallelism (one process per GPU, e.g. torchrun): every process
 * creates the job with the full ring, device = its GPU for its own worker and -1 for
 * workers hosted elsewhere; exports a blob of CUDA IPC handles (gradients, weights, flags,
 * losses), ships it to the others by any side channel and imports every peer's blob.
 * The per-step allreduce + update then runs as one kernel per GPU over NVLink peer memory. */
int edl_job_export(const EdlJob* job, uint8_t* buf, size_t cap, size_t* len);
int edl_job_import(EdlJob* job, const uint8_t* blob, size_t len);
/* Scheduler-facing scale-out across processes (the newcomer receives the
 * pending topology): the leader exports its host protocol state (t_cur, version, ring,
 * ShardManager snapshot, shard cursors) at the boundary where it fixes switch_t
 * (EDL_RETRY while another scaling operation is pending); a newcomer process created with
 * edl_job_create_joining adopts it before its first step and replays only from there.   */
int edl_job_export_state(const EdlJob* job, uint8_t* buf, size_t cap, size_t* len);
int edl_job_adopt_state(EdlJob* job, const uint8_t* blob, size_t len, int64_t switch_t);
/* Collective: all-gather the sharded fp32 master so every replica holds all of it
 * (before edl_job_params / checkpoints in multi-process jobs).                          */
int edl_job_gather_master(EdlJob* job);
void edl_job_set_profile(EdlJob* job, int32_t on);
/* phase_ms[7]: device ms per phase accumulated while profiling is on -- gather, forward,
 * loss, backward, update, and inside the backward: weight-gradient GEMMs, backward pair
 * launches (dgrad l-1 + wgrad/SGD l) -- plus mini-batches and library kernels launched.  */
void edl_job_counters(const EdlJob* job, double* phase_ms, uint64_t* steps, uint64_t* launches);
void edl_job_reset_counters(EdlJob* job);

/* Failure recovery (§4.2).  A checkpoint file holds the
 * JobCheckpoint fields: fp32 master (or f64 w), momentum, t_cur, topology
 * version, B and the lease state in the reference snapshot layout (datapipeline.cpp:115);
 * saving waits for the device.  Loading resumes at its t_cur with the job's current
 * workers: the checkpointed members' in-flight shards are reclaimed at their offsets,
 * leavers unregistered, newcomers registered, `restore <t-1>` + `topo` are logged.
 * edl_job_fail(ids) reports that `ids` failed during the last launched mini-batch:
 * approximate != 0 (needs cfg.appx_recovery) rolls the model, leases and log back to that
 * mini-batch's start and redoes it without them; approximate == 0 restores the latest
 * checkpoint saved by this job with the survivors, or (EDL_NO_CHECKPOINT) restarts them
 * from the initial state.                                                                 */
typedef struct {
  int32_t mode;      /* 1 approximate (redo the mini-batch), 0 consistent (checkpoint)  */
  int32_t status;    /* EDL_OK, or EDL_NO_CHECKPOINT (restarted from the initial state)  */
  uint64_t t_resume; /* next mini-batch index                                           */
  uint64_t version;  /* topology version after recovery                                 */
} EdlRecovery;
int edl_job_save_checkpoint(EdlJob* job, const char* path);
int edl_job_load_checkpoint(EdlJob* job, const char* path);
int edl_job_fail(EdlJob* job, const char* const* ids, int32_t n, int32_t approximate,
                 EdlRecovery* out);

/* Straggler detection ("longer than 1.2 times of the median
 * for 10 mini-batches"): durations[n_batches][n_workers] (NaN = worker absent); *worker =
 * the lowest index whose duration exceeds factor x the per-batch median (strict) in each
 * of the last `window` batches, else -1.                                                */
int edl_detect_straggler(const double* durations, int32_t n_batches, int32_t n_workers,
                         int32_t window, double factor, int32_t* worker);
/* The job's own statistics: device time of each worker's share of a mini-batch (gather to
 * end of backward), the last 64 completed steps.  edl_job_straggler writes the straggler's
 * id ("" if none) into buf.  edl_job_set_worker_delay injects a slowdown of `us`
 * microseconds per mini-batch into one worker (PAPER.md:529's straggler experiment).     */
int edl_job_worker_ms(const EdlJob* job, const char* worker, double* out, size_t cap,
                      size_t* n);
int edl_job_straggler(const EdlJob* job, int32_t window, double factor, char* buf, size_t cap,
                      size_t* len);
int edl_job_set_worker_delay(EdlJob* job, const char* worker, double us);

/* Weight-gradient GEMM with sgd_step (trainer.cpp:56-61) fused into its epilogue, for a job
 * with a single replica: dW[M][N] = dy^T x (dy row-major [K][ld_dy], x row-major [K][ld_x]),
 * then master -= scale * bf16(dW) and W (bf16) <- master.  No gradient buffer is written. */
int edl_gemm_wgrad_sgd(const void* dy, int32_t ld_dy, const void* x, int32_t ld_x,
                       float* master, void* W, int32_t ldw, int32_t M, int32_t N, int32_t K,
                       float scale, void* stream);

/* The same over the split master a single-replica job keeps: the fp32
 * master m is stored as its bf16 rounding W (the weights the GEMMs read) plus lo, the low 16
 * bits of m, so the update moves 8 B per parameter instead of 10.  mode 1: (W, lo) in and
 * out; 2: (W, lo) in, the fp32 master + W out; 3: the fp32 master in, (W, lo) out (master
 * may be NULL for mode 1).  edl_master_split writes W = RNE(m) and lo; edl_master_join
 * rebuilds m.  The one lossy case: an m that RNE rounds up
 * from an exact tie (low half 0x8000, odd high half) comes back one fp32 ulp larger.        */
int edl_gemm_wgrad_sgd_split(const void* dy, int32_t ld_dy, const void* x, int32_t ld_x,
                             uint16_t* lo, void* W, float* master, int32_t mode, int32_t ldw,
                             int32_t M, int32_t N, int32_t K, float scale, void* stream);
int edl_master_split(const float* master, uint16_t* lo, void* W, size_t n, void* stream);
int edl_master_join(const void* W, const uint16_t* lo, float* master, size_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EDL_B200_H */
