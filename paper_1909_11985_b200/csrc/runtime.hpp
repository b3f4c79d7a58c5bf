// Elastic data-parallel job runtime (the reference's absent runtime layer).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "collective.hpp"
#include "edl_internal.hpp"
#include "kernels.hpp"
#include "lease.hpp"

namespace edl {

constexpr int kSlots = 4;  // steps in flight on the host side (pinned staging ring)

struct LogRec {  // LogRecord, include/edl/trainer.hpp:59-70
  enum Kind { Batch = 0, Topo = 1, Restore = 2 } kind = Batch;
  uint64_t t = 0;
  std::string worker;
  std::vector<std::pair<uint64_t, uint64_t>> samples;  // (epoch, id) in draw order
  uint64_t version = 0;
  std::vector<std::string> ring;
};

struct Cursor {  // a worker's current shard lease
  bool has = false;
  uint32_t part = 0;
  uint64_t off = 0, len = 0, first = 0, epoch = 0;
};

// Model state + scratch on one GPU.  Workers on the same device share it: their replicas
// would be bit-identical at every mini-batch boundary (SPEC.md trainer invariants).
struct Replica {
  int device = 0;
  cudaStream_t stream = nullptr;
  Dataset* ds = nullptr;
  // MLP
  float* master = nullptr;
  __nv_bfloat16* W = nullptr;
  // split master (single-replica fused update): the low 16 bits of the fp32 master; while
  // lo_live the master is (W, mlo) and `master` is stale (Job::master_sync rebuilds it)
  uint16_t* mlo = nullptr;
  bool lo_live = false;
  // scale-out source: the newcomers' model copies still run on side3 (the next mini-batch's
  // stream waits for them before anything else)
  bool copies_pending = false;
  bool loss_on_side = false;  // the loss of recent mini-batches was read on `side`
  float* mom = nullptr;
  uint32_t* flags = nullptr;
  int64_t rows_cap = 0;
  std::vector<__nv_bfloat16*> act;  // act[l]: input of layer l, [rows][in_l]
  float* logits = nullptr;
  __nv_bfloat16* dlog = nullptr;
  // dgrad outputs, rotated by layer (dgrad l writes dx[l % 3]): the backward pair launch
  // runs dgrad l-1 (writing dx[(l-1) % 3]) next to wgrad l (reading dx[(l+1) % 3])
  __nv_bfloat16* dx[3] = {nullptr, nullptr, nullptr};
  float* row_loss = nullptr;
  unsigned* xent_done = nullptr;  // CTA counter of the fused softmax + loss-sum kernel
  int32_t* labels = nullptr;
  int64_t plan_rows = -1;
  std::vector<GemmPlan> fwd, dgrad;
  // linear
  double* w = nullptr;
  double* xb = nullptr;
  double* yb = nullptr;
  double* ws = nullptr;
  double* total = nullptr;
  double* loss_sum = nullptr;
  // approximate recovery: parameters at the start of the last launched mini-batch
  float* shadow_master = nullptr;
  float* shadow_mom = nullptr;
  double* shadow_w = nullptr;
  // per-step events
  cudaEvent_t ev_begin[kSlots] = {};
  cudaEvent_t ev_end[kSlots] = {};
  cudaEvent_t ev_done[kSlots] = {};  // end of this replica's share of a mini-batch
  cudaEvent_t ev_sync = nullptr;     // cross-stream ordering (model broadcast)
  // overlapped update: per-layer update / collective on `side` while the backward continues
  // on `stream`; ev_grad[l] = layer l's gradients final, ev_side = side work of the step done
  cudaStream_t side = nullptr;
  // copy-engine mode: side2 = reduce-scatter pushes, side = shard updates, side3 =
  // all-gather pushes; ev_rs[l] / ev_upd[l] order them per layer
  cudaStream_t side2 = nullptr, side3 = nullptr;
  std::vector<cudaEvent_t> ev_rs, ev_upd;
  __nv_bfloat16* recv = nullptr;  // [P]: peers' gradient slices of the shard this replica owns
  std::vector<cudaEvent_t> ev_grad;
  cudaEvent_t ev_side = nullptr;
  int layer_colls = 0;  // layer collectives launched this step
  // deferred all-gather (exchange mode 3 with EDL_AG_DEFER != 0): the push collective of
  // mini-batch t runs on `side` after ev_bwd (end of t's backward) while t+1's forward runs
  // on `stream`; t+1's forward GEMM of layer l waits for the layer's flags (ag_wait_epoch),
  // its first routed weight-gradient GEMM waits for ev_push (the peers' recv reads are done)
  cudaEvent_t ev_bwd = nullptr, ev_push = nullptr;
  uint32_t ag_wait_epoch = 0;  // 0: the weights are final (no deferred push in flight)
  bool side_pending = false;   // a deferred push on `side` not yet joined into `stream`
  double* host_loss = nullptr;  // pinned [kSlots]
};

struct Worker {
  std::string id;
  bool remote = false;    // hosted by another process; buffers below are IPC-mapped
  bool imported = false;  // remote worker whose handles have been imported
  int host_rank = -1;     // remote worker: PeerRep::rank of the process hosting it
  // device time of this worker's share of each in-flight mini-batch (gather .. backward)
  cudaEvent_t ev_w0[kSlots] = {}, ev_w1[kSlots] = {};
  double delay_us = 0.0;  // injected slowdown (straggler experiments)
  Replica* rep = nullptr;
  __nv_bfloat16* grad = nullptr;  // MLP gradient sum [P]
  double* g = nullptr;            // linear [grad_sum, count] (dim + 1)
  double* loss = nullptr;         // device scalar (sum over this worker's batch)
  EdlRun* runs_dev = nullptr;
  EdlRun* runs_host = nullptr;  // pinned [kSlots][runs_cap]
  int64_t runs_cap = 0;
  std::vector<GemmPlan> wgrad;
  std::vector<GemmPlan> wgrad_sgd;  // fused weight-gradient + SGD (single-member ring)
  std::vector<GemmPlan> wgrad_rs;   // weight gradient + reduce-scatter into the owners' recv
  std::vector<GemmPlan> wgrad_x;    // fused exchange: RS + sharded SGD + weight all-gather
  int64_t x_plan_rows = -1;
  uint64_t x_plan_version = 0;
  int64_t rs_plan_rows = -1;
  uint64_t rs_plan_version = 0;
  int rs_plan_mode = 0;
  int64_t plan_rows = -1;
  int64_t sgd_plan_rows = -1;
  Cursor cur;
  // current step
  std::vector<std::pair<uint64_t, uint64_t>> plan;
  int n_runs = 0;
};

// Straggler rule of SPEC.md:348-356 over a [n_batches][n_workers] duration matrix (NaN =
// worker absent); returns the worker index or -1 (runtime.cpp).
int detect_straggler(const double* dur, int n_batches, int n_workers, int window, double factor);

struct Event {
  // scheduler-facing scale_out: switch_t is fixed only once the newcomers report Ready
  // (preparation done), as t_cur + max(1, ceil(T_a / T_b))
  bool await_ready = false;
  std::atomic<bool> ready{false};
  int64_t switch_t;
  bool out;
  std::vector<std::string> ids;
  std::vector<int> devices;
  std::vector<std::unique_ptr<Worker>> prepared;  // scale-out newcomers built off-thread
  std::unique_ptr<std::thread> prep;
  int prep_rc = EDL_OK;
  double requested_ms = 0;
  std::vector<std::unique_ptr<Replica>> new_reps;  // GPUs joining the job (built off-thread)
};

// A replica as seen by every process: pointers valid in this process (local allocations
// or CUDA IPC mappings of a peer process's allocations over NVLink).
struct PeerRep {
  int rank = 0;  // replica order (smallest initial ring index of its workers)
  int device = -1;
  bool local = false;
  __nv_bfloat16* W = nullptr;
  float* master = nullptr;
  uint32_t* flags = nullptr;
  __nv_bfloat16* recv = nullptr;
  float* mom = nullptr;  // momentum (momentum != 0 only)
  uint16_t* mlo = nullptr;  // split-master low halves (single-replica fused update)
  Replica* rep = nullptr;  // local replicas
};

class Job {
 public:
  static int create(const EdlJobConfig& cfg, const std::vector<std::string>& ring,
                    const std::vector<int>& devices, Job** out);
  // One process per GPU, scale-out: a newcomer process's job.  `ring` is the job's current
  // ring (every member hosted by another process); worker `self_id` on `device` is built now
  // (context, dataset, buffers -- while the ring keeps stepping) and joins at `switch_t`;
  // `rank` orders its replica after the existing ones.  Until the switch step() replays the
  // lease protocol only (no device work).
  static int create_joining(const EdlJobConfig& cfg, const std::vector<std::string>& ring,
                            const std::vector<std::string>& newcomers, const std::string& self_id,
                            int device, int rank, int64_t switch_t, Job** out);
  ~Job();

  int step(EdlStepReport* rep);
  int sync(EdlStepReport* rep);
  int scale(bool out, const std::vector<std::string>& ids, const std::vector<int>& devices,
            int64_t explicit_switch, int64_t* switch_t);
  int params(const std::string& worker, void* host, size_t bytes);
  int set_params(const void* host, size_t bytes);
  std::string log_text() const;
  std::string ring_csv() const;
  uint64_t t() const { return t_; }
  size_t param_count() const { return P_; }
  double median_step_ms() const;
  int lease_snapshot(std::vector<uint8_t>* out) const {
    *out = lm_->snapshot();
    return EDL_OK;
  }
  void* stream() const {
    Replica* r = primary();
    return r ? r->stream : nullptr;
  }
  // multi-process data parallelism (one process per GPU): CUDA IPC handle exchange
  int export_handles(std::vector<uint8_t>* out) const;
  int import_handles(const uint8_t* blob, size_t len);
  // scheduler-facing scale-out across processes: the leader's host state at a boundary and
  // its adoption by a newcomer process (created with create_joining) before its first step
  int export_host_state(std::vector<uint8_t>* out) const;
  int adopt_host_state(const uint8_t* blob, size_t len, int64_t switch_t);
  bool peers_ready() const;
  // all-gather of the sharded fp32 master across replicas (collective: every process calls)
  int gather_master();
  void set_profile(bool on) { profile_ = on; }
  // how the N>1 gradient exchange runs (fixed at the first step after the peers are known):
  // 0 one fused collective after the backward, 1 per-layer side-stream collectives,
  // 2 per-layer copy-engine transfers, 3 reduce-scatter routed from the wgrad GEMM epilogues
  int exchange_mode() const { return overlap_mode_; }
  // accumulated device ms per phase (gather, forward, loss, backward, update) + launches
  void phase_totals(double* ms, uint64_t* steps, uint64_t* launches) const {
    for (int k = 0; k < kPhases; ++k) ms[k] = phase_ms_[k];
    *steps = phase_steps_;
    *launches = launches_;
  }
  void reset_counters() {
    for (double& v : phase_ms_) v = 0;
    phase_steps_ = 0;
    launches_ = 0;
  }
  // + 5: weight-gradient GEMMs, 6: backward pair launches (both inside the backward)
  static constexpr int kPhases = 7;
  static constexpr int kMaxMarks = 64;

 private:
  Job() = default;
  int init(const EdlJobConfig& cfg, const std::vector<std::string>& ring,
           const std::vector<int>& devices);
  Replica* replica_for(int device, int* rc);
  int build_replica(Replica* r);
  int build_worker(Worker* w, Replica* r);
  void free_worker(Worker* w);
  void free_replica(Replica* r);
  int ensure_plans(Worker* w, int64_t rows);
  int install_due(bool* switched);
  void arm_ready_events();  // Ready -> switch_t for scale-outs whose preparation finished
  int64_t switch_delay_steps() const;
  void resplit();
  std::vector<std::pair<uint64_t, uint64_t>> draw(Worker* w, int64_t need);
  int run_worker_mlp(Worker* w, int slot, bool last);
  int run_worker_linear(Worker* w, int slot);
  // *loss_src: device double holding the mini-batch's loss sum for the D2H read
  int reduce_and_update(uint64_t count, uint64_t t, int slot, const double** loss_src);
  int step_dry(EdlStepReport* out);
  void collect_completed();

  EdlJobConfig cfg_{};
  bool mlp_ = false;
  bool dry_ = false;  // host protocol only (EdlJobConfig::dry_run)
  // Single ring member + plain SGD: the update is fused into the weight-gradient GEMMs
  // (there is nothing to all-reduce); set per step.
  bool fused_update_ = false;
  // split master this mini-batch (fused update, no per-layer overlap), and whether its fused
  // launches leave the master split (false: a switch is due next, write the fp32 master)
  bool split_step_ = false;
  bool sgd_out_split_ = true;
  float step_scale_ = 0.f;
  // Overlapped update (EDL_OVERLAP, default on): layer l's update (and, with several
  // replicas, its NVLink reduce-scatter / all-gather) runs on the replica's side stream as
  // soon as layer l's weight gradients exist, under the rest of the backward pass.
  bool overlap_ = false;
  int overlap_mode_ = 0;  // 1: side-stream collective kernels, 2: copy-engine transfers,
                          // 3: reduce-scatter fused into the wgrad GEMM epilogues
  bool exited_ = false;    // one process per GPU: this process's members left the ring
  bool ag_ce_ = false;     // EDL_AG_DEFER=2: the deferred all-gather on the copy engines
  bool ag_defer_ = false;  // mode 3 + the push collective overlapped with the next forward
  bool rs_eligible() const;
  bool xchg_eligible() const;  // exchange mode 4 (fused into the weight-gradient GEMMs)
  bool push_eligible() const;
  uint32_t ce_epoch_ = 0;
  int host_index(const std::string& id) const;  // peers_ index of the replica hosting id
  size_t shard8(int l, int p, size_t* lo) const;  // replica p's slice of layer l (units of 8)
  size_t shard_total8(int p) const;
  size_t seg_off8(int p, int l) const;
  int recv_slot(int p, size_t k) const;  // k-th ring member's slot in replica p's recv
  bool ce_fits() const;
  int launch_layer_ce(Replica* r, int l);
  int launch_layer_rs_ce(Replica* r, int l);
  bool rs_via_ce(int peer_offset, int n_rep) const;  // mode 6: this owner via the copy engines
  int rs_tma_every() const;  // exchange mode 5: reduce-scatter on the copy engines
  // per-worker mini-batch durations of the last kTimeWindow completed steps (straggler
  // detection)
  static constexpr size_t kTimeWindow = 64;
  std::deque<std::vector<std::pair<std::string, double>>> wtimes_;

  // approximate recovery: host state at the start of the last launched mini-batch
  struct HostSnap {
    bool valid = false;
    uint64_t t = 0, version = 0;
    std::vector<std::string> ring;
    std::vector<uint8_t> lease;
    std::map<std::string, Cursor> cur;
    size_t log_len = 0;
  };
  HostSnap pre_;
  int lm_parts_ = 0;
  std::string lm_loc_;
  std::string last_ckpt_;  // latest checkpoint written by this job (consistent recovery)
  int take_pre_snapshot();
  int remove_members(const std::vector<std::string>& ids);  // immediate scale-in

 public:
  int save_checkpoint(const std::string& path);
  int load_checkpoint(const std::string& path);
  int recover(const std::vector<std::string>& failed, bool approximate, EdlRecovery* out);
  int set_worker_delay(const std::string& id, double us);
  int worker_ms(const std::string& id, std::vector<double>* out) const;
  // worker over factor x the per-step median in each of the last `window` steps ("" if none)
  std::string straggler(int window, double factor) const;

 private:
  // EDL_CE_TRACE=1: timing events of one step's overlapped transfers, printed by sync()
  bool ce_trace_ = false;
  std::vector<std::string> ce_marks_;
  unsigned long long* ce_stamps_ = nullptr;  // mapped pinned [256]
  void ce_mark(const std::string& what, cudaStream_t s);
  uint64_t step_count_ = 0;
  uint32_t layer_epoch0_ = 0;  // epoch of the first layer collective of the step
  int launch_layer_coll(Replica* r, int l);
  // replica `me` owns slice me/n_rep of every layer (all MLP collectives, checkpoints)
  void own_segments(int me, int n_rep, CollArgs* a) const;
  int finish_layer_colls(Replica* r);
  int L_ = 0;
  std::vector<int> in_, out_;
  std::vector<size_t> off_;
  size_t P_ = 0;
  std::unique_ptr<LeaseManager> lm_;
  std::vector<PeerRep> peers_;  // sorted by rank; includes the local replica
  // multi-process: every replica known (local + imported), members or not; peers_ is the
  // subset hosting ring members
  std::vector<PeerRep> known_peers_;
  bool joining_ = false;  // newcomer process whose worker has not switched in yet
  int step_host_only(bool switched, EdlStepReport* out);
  int install_out_mp(Event* ev);
  int reshard_in_mp(const Event* ev);
  int add_copy(MultiCopyArgs* cp, void* dst, const void* src, size_t bytes, cudaStream_t s);
  // scale-out across processes from one replica holding the split master: ship the low
  // master halves (2 B/param of each new shard) instead of the fp32 master (4 B)
  bool lo_reshard(const Event& ev) const;
  // newcomer process: the join words it still has to read (finish_join) once its first
  // mini-batch's forward is enqueued
  struct JoinWait {
    bool pending = false;
    uint64_t version = 0;
    int n_src = 0, me_new = 0, n_new = 0;
  } join_;
  bool join_pipeline_enabled(int n_src) const;
  int finish_join();
  double reshard_piece_bytes(const std::vector<PeerRep>& old, int i,
                             const std::vector<PeerRep>& after, bool mom, bool lo) const;
  int add_reshard_copies(MultiCopyArgs* cp, const std::vector<PeerRep>& old, int i,
                         const std::vector<PeerRep>& after, const std::vector<PeerRep>& fresh,
                         Replica* r, bool lo, bool skip_w);
  int join_own_shard(Replica* r, int me, int n);  // fp32 master of shard me/n from (W, lo)
  int reshard_local(const std::vector<PeerRep>& old, const std::vector<Replica*>& fresh);
  Worker* find_worker(const std::string& id) const;
  int my_rank_ = 0;
  std::vector<void*> ipc_mapped_;
  int rep_index() const;
  int rep_index(const Replica* r) const;
  Replica* primary() const;  // replica of the lowest-ranked local ring member
  int enable_peers(Replica* a, const std::vector<Replica*>& also = {});
  // peer access between GPU `dev` and every GPU in `devs`, both ways (idempotent)
  int enable_peer_devices(int dev, const std::vector<int>& devs);
  void rebuild_peers();
  int consolidate_master();  // async all-gather of the sharded fp32 master (local replicas)
  // rebuild the fp32 master of every replica that holds it split (stream-ordered)
  int master_sync();
  // join_side + master_sync: before anything reads or writes the master / weights outside
  // the fused step pipeline
  int master_current();
  // the fused wgrad + SGD launch of one layer in this mini-batch's split-master mode
  int run_sgd_plan(const GemmPlan& p, Replica* r);
 public:
  // orders every local replica's stream after its deferred push collective (no host sync):
  // before anything that reads the master / weights / loss outside the step pipeline
  int join_side();
  int launch_ag_ce(Replica* r, int me, uint32_t epoch);  // EDL_AG_DEFER=2 copies + flags
 private:
  int broadcast_model(Replica* src, Replica* dst);
  cudaEvent_t slot_end_[kSlots] = {};
  std::map<int, std::unique_ptr<Replica>> reps_;
  std::map<std::string, std::unique_ptr<Worker>> workers_;
  std::vector<std::string> ring_;
  std::vector<int64_t> splits_;
  std::deque<std::unique_ptr<Event>> events_;
  std::vector<LogRec> log_;
  uint64_t t_ = 0, version_ = 1;
  uint64_t launched_ = 0;  // steps launched
  uint32_t coll_epoch_ = 0;
  // completed-step bookkeeping
  struct Pending {
    Replica* rep;  // primary replica whose events time this mini-batch
    uint64_t t;
    int slot;
    uint64_t count;
    uint64_t version;
    int ring_size;
    int switched;
    bool have_prev;
    cudaEvent_t prev_end;
    std::vector<std::pair<std::string, Worker*>> timed;  // local workers of this step
  };
  std::deque<Pending> inflight_;
  std::vector<double> step_ms_;
  EdlStepReport last_{};
  std::vector<std::pair<cudaEvent_t, std::unique_ptr<Worker>>> graveyard_;
  cudaEvent_t last_end_ = nullptr;
  // profiling: events at phase boundaries of each in-flight slot
  bool profile_ = false;
  struct Mark {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<Mark> marks_[kSlots];
  std::vector<cudaEvent_t> ev_pool_;
  double phase_ms_[kPhases] = {};
  uint64_t phase_steps_ = 0;
  uint64_t launches_ = 0;  // kernels of this library launched
  cudaEvent_t mark_event();
  // Records a phase boundary on s; returns the event that starts the next phase (or null
  // when profiling is off).
  cudaEvent_t mark(int slot, int phase, cudaEvent_t start, cudaStream_t s);
  cudaEvent_t mark_begin(cudaStream_t s);
};

}  // namespace edl
