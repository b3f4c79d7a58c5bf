// Elastic data-parallel job runtime.
//
// The reference's runtime layer is absent: JobState, scale_out/scale_in,
// notify_batch_end and split_batch exist only in SPEC.md:272-392.  This is the B200-native
// realisation.  Host C++ owns the control plane (leases, ring, splits, log, switch
// scheduling); per mini-batch the device work is
//   H2D lease runs -> gather -> model fwd/bwd (tcgen05 GEMMs or f64 linear kernels)
//   -> fused allreduce + SGD update -> D2H loss
// all enqueued asynchronously on the replica's stream.
//
// Mini-batch protocol (shared verbatim with the CPU oracle, oracle/job_driver.hpp):
//   1. install topology events with switch_t == t (notify_batch_end of step t-1):
//      scale-out appends newcomers in ascending id order and enrolls them; scale-in
//      reclaims each leaver's shards in ring order and retires it; version += 1;
//      logged as `topo <t-1> <version> <ring...>`;
//   2. workers draw split[rank] samples in ring order from their shard lease (next_shard
//      when exhausted; EpochEnd -> ask again; ShardPending -> fewer samples this step);
//      progress is reported after each worker's draw;
//   3. per-worker [grad_sum, count] vectors are summed in ring order and applied with
//      sgd_step(eta_at(t)) — reference-exact f64 for the linear models, bf16 gradients +
//      fp32 master for the MLP.
#include "runtime.hpp"

#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <limits>
#include <set>
#include <sstream>

namespace edl {

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

template <class T>
int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return EDL_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * count);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  return EDL_OK;
}

#define EDL_TRY(expr)          \
  do {                         \
    int _rc = (expr);          \
    if (_rc != EDL_OK) return _rc; \
  } while (0)

// EDL_SPLIT_MASTER=0 keeps the fp32 master in the fused update (10 B per parameter)
bool split_master_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EDL_SPLIT_MASTER");
    on = e ? atoi(e) != 0 : 1;
  }
  return on != 0;
}

std::vector<int64_t> split_batch_vec(int64_t B, int p) {
  std::vector<int64_t> out(static_cast<size_t>(p), B / p);
  for (int64_t r = 0; r < B % p; ++r) out[static_cast<size_t>(r)] += 1;
  return out;
}

}  // namespace

int Job::create(const EdlJobConfig& cfg, const std::vector<std::string>& ring,
                const std::vector<int>& devices, Job** out) {
  auto* j = new Job;
  int rc = j->init(cfg, ring, devices);
  if (rc != EDL_OK) {
    delete j;
    return rc;
  }
  *out = j;
  return EDL_OK;
}

int Job::create_joining(const EdlJobConfig& cfg, const std::vector<std::string>& ring,
                        const std::vector<std::string>& newcomers, const std::string& self_id,
                        int device, int rank, int64_t switch_t, Job** out) {
  if (std::find(newcomers.begin(), newcomers.end(), self_id) == newcomers.end())
    return fail(EDL_EINVAL, "create_joining: self_id is not one of the newcomers");
  if (cfg.dry_run) return fail(EDL_EINVAL, "create_joining: not for dry-run jobs");
  if (device < 0) return fail(EDL_EINVAL, "create_joining: the newcomer needs a local GPU");
  for (const auto& id : ring)
    if (id == self_id) return fail(EDL_EINVAL, "create_joining: already a ring member");
  auto* j = new Job;
  j->joining_ = true;
  int rc = j->init(cfg, ring, std::vector<int>(ring.size(), -1));
  Replica* r = nullptr;
  if (rc == EDL_OK) r = j->replica_for(device, &rc);
  auto ev = std::make_unique<Event>();
  for (const auto& id : newcomers) {  // the other newcomers are hosted by their own processes
    if (rc != EDL_OK) break;
    auto w = std::make_unique<Worker>();
    w->id = id;
    if (id == self_id)
      rc = j->build_worker(w.get(), r);
    else
      w->remote = true;
    ev->prepared.push_back(std::move(w));
  }
  if (rc != EDL_OK) {
    delete j;
    return rc;
  }
  j->my_rank_ = rank;
  PeerRep me;
  me.rank = rank;
  me.device = device;
  me.local = true;
  me.W = r->W;
  me.master = r->master;
  me.flags = r->flags;
  me.recv = r->recv;
  me.mom = r->mom;
  me.mlo = r->mlo;
  me.rep = r;
  j->known_peers_.push_back(me);
  j->peers_.clear();
  ev->out = true;
  ev->ids = newcomers;
  for (const auto& id : newcomers) ev->devices.push_back(id == self_id ? device : -1);
  ev->switch_t = switch_t;
  j->events_.push_back(std::move(ev));
  *out = j;
  return EDL_OK;
}

Worker* Job::find_worker(const std::string& id) const {
  auto it = workers_.find(id);
  if (it != workers_.end()) return it->second.get();
  for (const auto& ev : events_)
    if (ev->out)
      for (const auto& w : ev->prepared)
        if (w && w->id == id) return w.get();
  return nullptr;
}

int Job::init(const EdlJobConfig& cfg, const std::vector<std::string>& ring,
              const std::vector<int>& devices) {
  cfg_ = cfg;
  if (ring.empty() || ring.size() != devices.size()) return fail(EDL_EINVAL, "job: empty ring");
  if (cfg.model != EDL_MODEL_LEAST_SQUARES && cfg.model != EDL_MODEL_LOGISTIC &&
      cfg.model != EDL_MODEL_MLP)
    return fail(EDL_EINVAL, "job: unknown model");
  if (cfg.per_worker_batch <= 0 && cfg.batch < static_cast<int64_t>(ring.size()))
    return fail(EDL_EINVAL, "split_batch: B < p");
  mlp_ = cfg.model == EDL_MODEL_MLP;
  dry_ = cfg.dry_run != 0;
  if (mlp_) {
    L_ = cfg.layers;
    if (L_ < 1 || cfg.hidden <= 0 || cfg.num_classes <= 0) return fail(EDL_EINVAL, "job: MLP shape");
    if (L_ > kCollMaxSegs) return fail(EDL_EINVAL, "job: too many MLP layers");
    if (cfg.data.dim % 8 || cfg.hidden % 8 || cfg.num_classes % 8)
      return fail(EDL_EINVAL, "job: MLP widths must be multiples of 8 (16-byte TMA rows)");
    if (cfg.num_classes > 16384) return fail(EDL_EINVAL, "job: num_classes > 16384");
    for (int l = 0; l < L_; ++l) {
      in_.push_back(l == 0 ? cfg.data.dim : cfg.hidden);
      out_.push_back(l == L_ - 1 ? cfg.num_classes : cfg.hidden);
      off_.push_back(P_);
      P_ += static_cast<size_t>(in_.back()) * out_.back();
    }
  } else {
    P_ = static_cast<size_t>(cfg.data.dim);
  }
  const int parts = cfg.partitions > 0 ? cfg.partitions
                                       : default_partitions(std::max<int>(cfg.max_workers,
                                                                          static_cast<int>(ring.size())));
  std::ostringstream loc;
  loc << "synthetic:" << cfg.data.seed << ":" << cfg.data.size;  // dataset.cpp:56-58
  lm_ = std::make_unique<LeaseManager>(cfg.data.size, parts, cfg.lease_seed, loc.str());
  lm_parts_ = parts;
  lm_loc_ = loc.str();
  int first_local = -1;
  for (size_t i = 0; i < ring.size(); ++i) {
    if (workers_.count(ring[i])) return fail(EDL_EINVAL, "job: duplicate worker id");
    auto w = std::make_unique<Worker>();
    w->id = ring[i];
    if (devices[i] < 0) {
      w->remote = true;  // hosted by a peer process; buffers arrive via import_handles
    } else {
      int rc = EDL_OK;
      Replica* r = replica_for(devices[i], &rc);
      if (!r) return rc;
      EDL_TRY(build_worker(w.get(), r));
      if (first_local < 0) first_local = static_cast<int>(i);
    }
    lm_->enroll(ring[i]);
    workers_[ring[i]] = std::move(w);
  }
  if (joining_) {  // create_joining adds the newcomer's replica and worker
    ring_ = ring;
    version_ = 1;
    resplit();
    if (cfg_.keep_log) {
      LogRec r;
      r.kind = LogRec::Topo;
      r.t = 0;
      r.version = version_;
      r.ring = ring_;
      log_.push_back(r);
    }
    return EDL_OK;
  }
  if (first_local < 0) return fail(EDL_EINVAL, "job: no local worker (device >= 0) in the ring");
  my_rank_ = first_local;
  {
    Replica* r = reps_.begin()->second.get();
    PeerRep me;
    me.rank = my_rank_;
    me.device = r->device;
    me.local = true;
    me.W = r->W;
    me.master = r->master;
    me.flags = r->flags;
    me.recv = r->recv;
    me.mom = r->mom;
    me.mlo = r->mlo;
    me.rep = r;
    peers_.push_back(me);
    known_peers_.push_back(me);
  }
  ring_ = ring;
  version_ = 1;
  rebuild_peers();
  resplit();
  if (cfg_.keep_log) {
    LogRec r;
    r.kind = LogRec::Topo;
    r.t = 0;
    r.version = version_;
    r.ring = ring_;
    log_.push_back(r);
  }
  return EDL_OK;
}

Replica* Job::replica_for(int device, int* rc) {
  auto it = reps_.find(device);
  if (it != reps_.end()) return it->second.get();
  auto r = std::make_unique<Replica>();
  r->device = device;
  *rc = build_replica(r.get());
  if (*rc == EDL_OK) *rc = enable_peers(r.get());
  if (*rc != EDL_OK) return nullptr;
  Replica* raw = r.get();
  reps_[device] = std::move(r);
  return raw;
}

// NVLink peer access between a new replica's GPU and every other replica's, both ways.
int Job::enable_peers(Replica* a, const std::vector<Replica*>& also) {
  std::vector<int> devs;
  for (auto& [dev, r] : reps_) devs.push_back(dev);
  for (Replica* o : also) devs.push_back(o->device);
  return enable_peer_devices(a->device, devs);
}

int Job::enable_peer_devices(int a_dev, const std::vector<int>& devs) {
  if (dry_) return EDL_OK;
  for (int dev : devs) {
    if (dev == a_dev) continue;
    for (int pass = 0; pass < 2; ++pass) {
      const int from = pass ? dev : a_dev, to = pass ? a_dev : dev;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, from, to);
      if (!can) return fail(EDL_ECUDA, "GPUs " + std::to_string(from) + " and " +
                                           std::to_string(to) + " have no peer access");
      DeviceGuard g(from);
      const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      cudaGetLastError();  // clear "already enabled"
    }
  }
  return EDL_OK;
}

Replica* Job::primary() const {
  for (const auto& id : ring_) {
    auto it = workers_.find(id);
    if (it != workers_.end() && !it->second->remote && it->second->rep) return it->second->rep;
  }
  return reps_.empty() ? nullptr : reps_.begin()->second.get();
}

// Single-process jobs: replicas ordered by their first ring member; replicas without
// members (all their workers left) drop out of the collective.  Multi-process jobs keep the
// static order fixed at import time.
void Job::rebuild_peers() {
  bool multi = false;
  for (const auto& p : known_peers_) multi = multi || !p.local;
  if (multi) {
    // one process per GPU: the replicas (local or imported) that host a ring member, in
    // rank order; their indices (shards, recv slots) follow from it
    std::vector<PeerRep> v;
    for (const auto& p : known_peers_) {
      bool hosts = false;
      for (const auto& id : ring_) {
        const Worker* w = workers_.at(id).get();
        hosts = hosts || (p.local ? !w->remote && w->rep == p.rep
                                  : w->remote && w->host_rank == p.rank);
      }
      if (hosts) v.push_back(p);
    }
    peers_ = v;
    return;
  }
  std::vector<PeerRep> v;
  for (auto& [dev, r] : reps_) {
    int first = -1;
    for (size_t i = 0; i < ring_.size() && first < 0; ++i) {
      auto it = workers_.find(ring_[i]);
      if (it != workers_.end() && it->second->rep == r.get()) first = static_cast<int>(i);
    }
    if (first < 0) continue;
    PeerRep p;
    p.rank = first;
    p.device = dev;
    p.local = true;
    p.W = r->W;
    p.master = r->master;
    p.flags = r->flags;
    p.recv = r->recv;
    p.mom = r->mom;
    p.mlo = r->mlo;
    p.rep = r.get();
    v.push_back(p);
  }
  std::sort(v.begin(), v.end(), [](const PeerRep& a, const PeerRep& b) { return a.rank < b.rank; });
  if (!v.empty()) peers_ = v;
}

int Job::build_replica(Replica* r) {
  r->rows_cap = cfg_.per_worker_batch > 0 ? cfg_.per_worker_batch : cfg_.batch;
  if (dry_) return EDL_OK;
  DeviceGuard g(r->device);
  EDL_CUDA_TRY(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
  for (int s = 0; s < kSlots; ++s) {
    EDL_CUDA_TRY(cudaEventCreate(&r->ev_begin[s]));
    EDL_CUDA_TRY(cudaEventCreate(&r->ev_end[s]));
    EDL_CUDA_TRY(cudaEventCreateWithFlags(&r->ev_done[s], cudaEventDisableTiming));
  }
  EDL_CUDA_TRY(cudaEventCreateWithFlags(&r->ev_sync, cudaEventDisableTiming));
  if (mlp_) {
    EDL_CUDA_TRY(cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking));
    EDL_CUDA_TRY(cudaStreamCreateWithFlags(&r->side2, cudaStreamNonBlocking));
    EDL_CUDA_TRY(cudaStreamCreateWithFlags(&r->side3, cudaStreamNonBlocking));
    r->ev_rs.assign(static_cast<size_t>(L_), nullptr);
    for (auto& e : r->ev_rs) EDL_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    r->ev_upd.assign(static_cast<size_t>(L_), nullptr);
    for (auto& e : r->ev_upd) EDL_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    EDL_CUDA_TRY(cudaEventCreateWithFlags(&r->ev_side, cudaEventDisableTiming));
    EDL_CUDA_TRY(cudaEventCreateWithFlags(&r->ev_bwd, cudaEventDisableTiming));
    EDL_CUDA_TRY(cudaEventCreateWithFlags(&r->ev_push, cudaEventDisableTiming));
    r->ev_grad.assign(static_cast<size_t>(L_), nullptr);
    for (auto& e : r->ev_grad) EDL_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  EDL_CUDA_TRY(cudaMallocHost(&r->host_loss, sizeof(double) * kSlots));
  // newcomers run this on their preparation thread: kernel loading stays off the switch step
  EDL_TRY(coll_prepare_device());
  EDL_TRY(dataset_prepare_device());
  if (mlp_) {
    EDL_TRY(gemm_prepare_device());
    EDL_TRY(mlp_prepare_device());
  }
  EDL_TRY(dataset_create(cfg_.data, mlp_ ? EDL_DTYPE_BF16 : EDL_DTYPE_F64,
                         mlp_ ? cfg_.num_classes : 0, &r->ds));
  const int64_t rows = cfg_.per_worker_batch > 0 ? cfg_.per_worker_batch : cfg_.batch;
  r->rows_cap = rows;
  EDL_TRY(dalloc(&r->flags, kCollFlagBytes / 4));
  EDL_CUDA_TRY(cudaMemset(r->flags, 0, kCollFlagBytes));
  if (mlp_) {
    EDL_TRY(dalloc(&r->master, P_));
    EDL_TRY(dalloc(&r->W, P_));
    // split master for the single-replica fused update (not with approximate recovery,
    // which snapshots the fp32 master before every mini-batch)
    if (split_master_enabled() && cfg_.momentum == 0.0 && !cfg_.appx_recovery)
      EDL_TRY(dalloc(&r->mlo, P_));
    EDL_TRY(dalloc(&r->recv, P_));
    // exchange mode 4 reads "0xFFFF = not arrived yet" from the receive slots
    EDL_CUDA_TRY(cudaMemset(r->recv, 0xFF, sizeof(__nv_bfloat16) * P_));
    if (cfg_.momentum != 0.0) {
      EDL_TRY(dalloc(&r->mom, P_));
      EDL_CUDA_TRY(cudaMemset(r->mom, 0, sizeof(float) * P_));
    }
    for (int l = 0; l < L_; ++l) {
      const double bound = std::sqrt(6.0 / static_cast<double>(in_[l]));  // Kaiming-uniform
      EDL_TRY(mlp_init_weights(r->master + off_[l], r->W + off_[l],
                               static_cast<size_t>(in_[l]) * out_[l], cfg_.init_seed, off_[l],
                               bound, r->stream));
    }
    r->act.resize(static_cast<size_t>(L_));
    for (int l = 0; l < L_; ++l) EDL_TRY(dalloc(&r->act[l], static_cast<size_t>(rows) * in_[l]));
    EDL_TRY(dalloc(&r->logits, static_cast<size_t>(rows) * cfg_.num_classes));
    EDL_TRY(dalloc(&r->dlog, static_cast<size_t>(rows) * cfg_.num_classes));
    int widest = cfg_.data.dim > cfg_.hidden ? cfg_.data.dim : cfg_.hidden;
    EDL_TRY(dalloc(&r->dx[0], static_cast<size_t>(rows) * widest));
    EDL_TRY(dalloc(&r->dx[1], static_cast<size_t>(rows) * widest));
    EDL_TRY(dalloc(&r->dx[2], static_cast<size_t>(rows) * widest));
    EDL_TRY(dalloc(&r->row_loss, static_cast<size_t>(rows)));
    EDL_CUDA_TRY(cudaMalloc(&r->xent_done, sizeof(unsigned)));
    EDL_CUDA_TRY(cudaMemset(r->xent_done, 0, sizeof(unsigned)));
    EDL_TRY(dalloc(&r->labels, static_cast<size_t>(rows)));
  } else {
    const int dim = cfg_.data.dim;
    EDL_TRY(dalloc(&r->w, static_cast<size_t>(dim)));
    EDL_CUDA_TRY(cudaMemset(r->w, 0, sizeof(double) * dim));  // w0 = 0
    EDL_TRY(dalloc(&r->xb, static_cast<size_t>(rows) * dim));
    EDL_TRY(dalloc(&r->yb, static_cast<size_t>(rows)));
    EDL_TRY(dalloc(&r->ws, 2 * static_cast<size_t>(rows) + 1));  // scales, then z
    EDL_TRY(dalloc(&r->total, static_cast<size_t>(dim) + 1));
  }
  EDL_TRY(dalloc(&r->loss_sum, 1));
  // the cudaMemset calls above run on the legacy default stream, which does not order the
  // replica's non-blocking streams (nor peers reading the flags): wait for all of them here.
  // (A first mini-batch racing the xent counter's memset summed row losses too early.)
  EDL_CUDA_TRY(cudaDeviceSynchronize());
  return EDL_OK;
}

int Job::build_worker(Worker* w, Replica* r) {
  w->rep = r;
  if (dry_) return EDL_OK;
  DeviceGuard g(r->device);
  w->runs_cap = r->rows_cap + 2;
  EDL_TRY(dalloc(&w->runs_dev, static_cast<size_t>(w->runs_cap)));
  EDL_CUDA_TRY(cudaMallocHost(&w->runs_host, sizeof(EdlRun) * w->runs_cap * kSlots));
  // MLP: two slots by mini-batch parity (the deferred push collective of t reads slot t&1
  // while t+1's gather / softmax already write the other)
  EDL_TRY(dalloc(&w->loss, 2));
  if (mlp_)
    EDL_TRY(dalloc(&w->grad, P_));
  else
    EDL_TRY(dalloc(&w->g, static_cast<size_t>(cfg_.data.dim) + 1));
  for (int s = 0; s < kSlots; ++s) {
    EDL_CUDA_TRY(cudaEventCreate(&w->ev_w0[s]));
    EDL_CUDA_TRY(cudaEventCreate(&w->ev_w1[s]));
  }
  return EDL_OK;
}

void Job::free_worker(Worker* w) {
  if (!w || !w->rep || w->remote || dry_) return;
  DeviceGuard g(w->rep->device);
  cudaFree(w->runs_dev);
  cudaFreeHost(w->runs_host);
  cudaFree(w->loss);
  cudaFree(w->grad);
  cudaFree(w->g);
  for (int s = 0; s < kSlots; ++s) {
    if (w->ev_w0[s]) cudaEventDestroy(w->ev_w0[s]);
    if (w->ev_w1[s]) cudaEventDestroy(w->ev_w1[s]);
    w->ev_w0[s] = w->ev_w1[s] = nullptr;
  }
  w->rep = nullptr;
}

void Job::free_replica(Replica* r) {
  if (!r || dry_) return;
  DeviceGuard g(r->device);
  if (r->stream) cudaStreamSynchronize(r->stream);
  dataset_destroy(r->ds);
  cudaFree(r->master);
  cudaFree(r->mlo);
  cudaFree(r->W);
  cudaFree(r->recv);
  cudaFree(r->mom);
  cudaFree(r->flags);
  for (auto* a : r->act) cudaFree(a);
  cudaFree(r->logits);
  cudaFree(r->dlog);
  cudaFree(r->dx[0]);
  cudaFree(r->dx[1]);
  cudaFree(r->dx[2]);
  cudaFree(r->row_loss);
  cudaFree(r->xent_done);
  cudaFree(r->labels);
  cudaFree(r->w);
  cudaFree(r->xb);
  cudaFree(r->yb);
  cudaFree(r->ws);
  cudaFree(r->total);
  cudaFree(r->loss_sum);
  cudaFree(r->shadow_master);
  cudaFree(r->shadow_mom);
  cudaFree(r->shadow_w);
  r->shadow_master = r->shadow_mom = nullptr;
  r->shadow_w = nullptr;
  cudaFreeHost(r->host_loss);
  for (int s = 0; s < kSlots; ++s) {
    cudaEventDestroy(r->ev_begin[s]);
    cudaEventDestroy(r->ev_end[s]);
    cudaEventDestroy(r->ev_done[s]);
  }
  cudaEventDestroy(r->ev_sync);
  for (auto e : r->ev_grad) cudaEventDestroy(e);
  r->ev_grad.clear();
  for (auto e : r->ev_rs) cudaEventDestroy(e);
  r->ev_rs.clear();
  for (auto e : r->ev_upd) cudaEventDestroy(e);
  r->ev_upd.clear();
  for (cudaStream_t* st : {&r->side2, &r->side3}) {
    if (*st) {
      cudaStreamSynchronize(*st);
      cudaStreamDestroy(*st);
    }
    *st = nullptr;
  }
  if (r->ev_side) cudaEventDestroy(r->ev_side);
  if (r->ev_bwd) cudaEventDestroy(r->ev_bwd);
  if (r->ev_push) cudaEventDestroy(r->ev_push);
  r->ev_bwd = r->ev_push = nullptr;
  if (r->side) {
    cudaStreamSynchronize(r->side);
    cudaStreamDestroy(r->side);
  }
  r->side = nullptr;
  r->ev_side = nullptr;
  cudaStreamDestroy(r->stream);
  r->ds = nullptr;
  r->stream = nullptr;
}

Job::~Job() {
  for (auto& e : events_)
    if (e->prep && e->prep->joinable()) e->prep->join();
  if (dry_) return;
  for (void* p : ipc_mapped_) cudaIpcCloseMemHandle(p);
  for (auto& [dev, r] : reps_) {
    DeviceGuard g(dev);
    if (r->stream) cudaStreamSynchronize(r->stream);
  }
  for (auto& [ev, w] : graveyard_) {
    free_worker(w.get());
    cudaEventDestroy(ev);
  }
  for (auto& e : events_) {
    for (auto& w : e->prepared) free_worker(w.get());
    for (auto& r : e->new_reps) free_replica(r.get());
  }
  for (auto& [id, w] : workers_) free_worker(w.get());
  for (auto& [dev, r] : reps_) free_replica(r.get());
}

void Job::resplit() {
  const int p = static_cast<int>(ring_.size());
  if (cfg_.per_worker_batch > 0)
    splits_.assign(static_cast<size_t>(p), cfg_.per_worker_batch);
  else
    splits_ = split_batch_vec(cfg_.batch, p);
}

// Draw `need` samples for one worker (protocol step 2).
std::vector<std::pair<uint64_t, uint64_t>> Job::draw(Worker* w, int64_t need) {
  std::vector<std::pair<uint64_t, uint64_t>> out;
  out.reserve(static_cast<size_t>(need));
  Cursor& c = w->cur;
  while (need > 0) {
    if (!c.has) {
      const Lease n = lm_->next(w->id);
      if (n.kind == LeaseKind::EpochEnd) continue;
      if (n.kind == LeaseKind::Pending || n.status != LeaseStatus::Ok) break;
      c.has = true;
      c.part = n.meta.index;
      c.off = n.resume;
      c.len = n.meta.length;
      c.first = n.meta.offset;
      c.epoch = lm_->epoch();
    }
    const uint64_t k = std::min<uint64_t>(static_cast<uint64_t>(need), c.len - c.off);
    for (uint64_t j = 0; j < k; ++j) out.emplace_back(c.epoch, c.first + c.off + j);
    c.off += k;
    need -= static_cast<int64_t>(k);
    if (c.off >= c.len) {
      lm_->progress(w->id, c.part, c.len);
      c.has = false;
    }
  }
  if (c.has) lm_->progress(w->id, c.part, c.off);
  return out;
}

// Protocol step 1: topology switches due at this mini-batch.
int64_t Job::switch_delay_steps() const {
  const double tb = median_step_ms();
  if (!(tb > 0)) return 1;
  return std::max<int64_t>(1, static_cast<int64_t>(std::ceil(cfg_.t_a_ms / tb)));
}

void Job::arm_ready_events() {
  bool armed = false;
  for (auto& e : events_) {
    if (!e->await_ready || !e->ready.load(std::memory_order_acquire)) continue;
    e->await_ready = false;
    e->switch_t = static_cast<int64_t>(t_) + switch_delay_steps();
    armed = true;
  }
  if (armed)
    std::stable_sort(events_.begin(), events_.end(),
                     [](const std::unique_ptr<Event>& a, const std::unique_ptr<Event>& b) {
                       return a->switch_t < b->switch_t;
                     });
}

int Job::install_due(bool* switched) {
  arm_ready_events();
  *switched = false;
  bool changed = false;
  while (!events_.empty() && events_.front()->switch_t <= static_cast<int64_t>(t_)) {
    // re-sharding, broadcasts and copies below read the fp32 master (a scale-out across
    // processes from a split-master replica ships the low halves instead: lo_reshard)
    if (!lo_reshard(*events_.front())) EDL_TRY(master_sync());
    std::unique_ptr<Event> ev = std::move(events_.front());
    events_.pop_front();
    // newcomers hosted by their own processes (scale-out across processes)
    bool multi = !dry_ && ev->out && joining_;
    for (const auto& w : ev->prepared) multi = multi || (!dry_ && w && w->remote);
    // the fp32 master is sharded across GPUs; make every replica whole before the
    // membership (and with it the sharding) changes -- except for a scale-out across
    // processes, which re-shards with targeted copies (install_out_mp)
    bool all_local = true;
    for (const auto& p : peers_) all_local = all_local && p.local;
    // one process driving every replica: re-shard with targeted copies after the switch
    // (reshard_local); EDL_RESHARD=0 falls back to consolidating the whole model
    static int reshard_env = -1;
    if (reshard_env < 0) {
      const char* e = getenv("EDL_RESHARD");
      reshard_env = e ? atoi(e) : 1;
    }
    const bool local_targeted = reshard_env && !multi && mlp_ && !dry_ && all_local &&
                                !peers_.empty();
    const std::vector<PeerRep> old_peers = peers_;
    std::vector<Replica*> fresh;  // replicas that join the collective at this switch
    if (ev->out && multi) {
      // the deferred push collective; the split master is joined above or shipped as is
      // (install_out_mp, lo_reshard)
      EDL_TRY(join_side());
    } else if (!ev->out && !all_local && mlp_ && !dry_ && peers_.size() > 1) {
      EDL_TRY(join_side());
      EDL_TRY(reshard_in_mp(ev.get()));  // targeted: each survivor gets its new shard only
    } else if (local_targeted) {
      EDL_TRY(join_side());
    } else {
      EDL_TRY(consolidate_master());
    }
    if (ev->out && multi) {
      EDL_TRY(install_out_mp(ev.get()));
    } else if (ev->out) {
      if (ev->prep && ev->prep->joinable()) ev->prep->join();  // stall only if prep is late
      if (ev->prep_rc != EDL_OK) return ev->prep_rc;
      Replica* src = primary();  // lowest existing ring member's replica
      std::set<Replica*> live;     // replicas currently in the collective (model is current)
      for (const auto& p : peers_)
        if (p.local) live.insert(p.rep);
      for (auto& nr : ev->new_reps) {
        Replica* dst = nr.get();
        auto have = reps_.find(dst->device);
        if (have != reps_.end()) {
          // an earlier event already brought this GPU in: join its replica instead
          for (auto& w : ev->prepared)
            if (w && w->rep == dst) w->rep = have->second.get();
          free_replica(dst);
          continue;
        }
        reps_[dst->device] = std::move(nr);
        // GPUs that joined since this event was prepared (its preparation ran concurrently)
        std::vector<int> all;
        for (auto& [d, r] : reps_) all.push_back(d);
        EDL_TRY(enable_peer_devices(dst->device, all));
      }
      // model broadcast to every replica that is not in the collective yet (new GPUs, or
      // GPUs whose members all left earlier and whose model is stale)
      // After consolidate_master every live replica holds the identical full model, so the
      // newcomers pull from the live replicas in turn (SPEC.md:376 names the lowest rank; the
      // bytes are bit-identical and no single GPU's NVLink egress carries every copy)
      // (sources: replicas hosting a current ring member, in ring order)
      std::vector<Replica*> srcs;
      for (const auto& id : ring_) {
        const Worker* wk = workers_[id].get();
        if (wk->remote || !wk->rep || !live.count(wk->rep)) continue;
        if (std::find(srcs.begin(), srcs.end(), wk->rep) == srcs.end()) srcs.push_back(wk->rep);
      }
      static int spread = -1;
      if (spread < 0) {
        const char* e = getenv("EDL_BCAST_SPREAD");
        spread = e ? atoi(e) : 1;
      }
      if (!spread) srcs.clear();
      if (srcs.empty()) srcs.push_back(src);
      std::set<Replica*> sent;
      for (auto& w : ev->prepared) {
        if (!w || live.count(w->rep) || sent.count(w->rep)) continue;
        if (local_targeted)
          fresh.push_back(w->rep);  // filled by reshard_local once the ring is re-formed
        else
          EDL_TRY(broadcast_model(srcs[sent.size() % srcs.size()], w->rep));
        sent.insert(w->rep);
      }
      std::vector<size_t> order(ev->ids.size());
      for (size_t i = 0; i < order.size(); ++i) order[i] = i;
      std::sort(order.begin(), order.end(),
                [&](size_t a, size_t b) { return ev->ids[a] < ev->ids[b]; });
      for (size_t i : order) {
        const std::string& id = ev->ids[i];
        if (std::find(ring_.begin(), ring_.end(), id) != ring_.end()) {
          free_worker(ev->prepared[i].get());  // already a member: nothing to join
          continue;
        }
        ring_.push_back(id);
        lm_->enroll(id);
        workers_[id] = std::move(ev->prepared[i]);
      }
    } else {
      std::vector<std::string> keep;
      for (const auto& id : ring_) {
        if (std::find(ev->ids.begin(), ev->ids.end(), id) == ev->ids.end()) {
          keep.push_back(id);
          continue;
        }
        lm_->reclaim(id);  // graceful exit: shard back at its last reported offset
        lm_->retire(id);
        auto it = workers_.find(id);
        if (dry_ || it->second->remote) {
          workers_.erase(it);
          continue;
        }
        cudaEvent_t done;
        DeviceGuard g(it->second->rep->device);
        cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
        cudaEventRecord(done, it->second->rep->stream);
        graveyard_.emplace_back(done, std::move(it->second));
        workers_.erase(it);
      }
      ring_ = keep;
    }
    ++version_;
    changed = true;
    if (cfg_.keep_log) {
      LogRec r;
      r.kind = LogRec::Topo;
      r.t = t_ == 0 ? 0 : t_ - 1;
      r.version = version_;
      r.ring = ring_;
      log_.push_back(r);
    }
    rebuild_peers();
    if (local_targeted) EDL_TRY(reshard_local(old_peers, fresh));
  }
  if (changed) {
    resplit();
    *switched = true;
  }
  return EDL_OK;
}

int Job::ensure_plans(Worker* w, int64_t rows) {
  Replica* r = w->rep;
  if (r->plan_rows != rows) {
    r->fwd.assign(static_cast<size_t>(L_), GemmPlan{});
    r->dgrad.assign(static_cast<size_t>(L_), GemmPlan{});
    for (int l = 0; l < L_; ++l) {
      const bool last = l == L_ - 1;
      void* outp = last ? static_cast<void*>(r->logits) : static_cast<void*>(r->act[l + 1]);
      EDL_TRY(gemm_plan_init(&r->fwd[l], r->act[l], in_[l], 0, r->W + off_[l], in_[l], 0, outp,
                             out_[l], static_cast<int>(rows), out_[l], in_[l], last ? 0 : 1,
                             last ? 1 : 0, nullptr, 0, 0));
      if (l > 0) {
        const __nv_bfloat16* dy = last ? r->dlog : r->dx[(l + 1) % 3];
        EDL_TRY(gemm_plan_init(&r->dgrad[l], dy, out_[l], 0, r->W + off_[l], in_[l], 1,
                               r->dx[l % 3], in_[l], static_cast<int>(rows), in_[l], out_[l], 0,
                               0, r->act[l], in_[l], 0));
        // while dgrad l runs (tensor-bound, HBM mostly idle) pull layer l's fp32 master into
        // L2 for the fused wgrad + SGD kernel that follows.  Opt-in (EDL_DGRAD_L2PF=1):
        // measured on B200 the wgrad kernel gains ~2 us but each dgrad loses ~8 us to the
        // extra HBM / L2 traffic (0.697 vs 0.661 ms per mini-batch)
        static int l2pf = -1;
        if (l2pf < 0) {
          const char* e = getenv("EDL_DGRAD_L2PF");
          l2pf = e ? atoi(e) : 0;
        }
        if (l2pf && r->mlo) {
          r->dgrad[l].ep.l2pf = r->mlo + off_[l];
          r->dgrad[l].ep.l2pf_bytes = sizeof(uint16_t) * static_cast<size_t>(in_[l]) * out_[l];
        } else if (l2pf) {
          r->dgrad[l].ep.l2pf = r->master + off_[l];
          r->dgrad[l].ep.l2pf_bytes = sizeof(float) * static_cast<size_t>(in_[l]) * out_[l];
        }
      }
    }
    r->plan_rows = rows;
  }
  if (w->plan_rows != rows) {
    w->wgrad.assign(static_cast<size_t>(L_), GemmPlan{});
    for (int l = 0; l < L_; ++l) {
      const bool last = l == L_ - 1;
      const __nv_bfloat16* dy = last ? r->dlog : r->dx[(l + 1) % 3];
      EDL_TRY(gemm_plan_init(&w->wgrad[l], dy, out_[l], 1, r->act[l], in_[l], 1,
                             w->grad + off_[l], in_[l], out_[l], in_[l], static_cast<int>(rows),
                             0, 0, nullptr, 0, 0));
    }
    w->plan_rows = rows;
  }
  if ((overlap_mode_ == 3 || overlap_mode_ == 6 || (overlap_mode_ == 5 && rs_tma_every() > 0)) &&
      (w->rs_plan_rows != rows || w->rs_plan_version != version_ ||
       w->rs_plan_mode != overlap_mode_)) {
    const int n = static_cast<int>(peers_.size());
    const int me = rep_index(r);
    w->wgrad_rs.assign(static_cast<size_t>(L_), GemmPlan{});
    for (int l = 0; l < L_; ++l) {
      const bool last = l == L_ - 1;
      const __nv_bfloat16* dy = last ? r->dlog : r->dx[(l + 1) % 3];
      EDL_TRY(gemm_plan_init(&w->wgrad_rs[l], dy, out_[l], 1, r->act[l], in_[l], 1,
                             w->grad + off_[l], in_[l], out_[l], in_[l], static_cast<int>(rows),
                             0, 0, nullptr, 0, 1000 + 128));
      const size_t prow = static_cast<size_t>(out_[l]) / n;
      void* dst[kMaxPeerMaps] = {};
      for (int o = 0; o < n; ++o) {  // the push collective's recv layout (collective.cu)
        if (o == me) continue;
        if (overlap_mode_ == 6 && rs_via_ce((o - me + n) % n, n)) {
          // mode 6: this owner's rows stay local; the copy engines move them (rs_ce)
          dst[o] = w->grad + off_[l] + static_cast<size_t>(o) * prow * in_[l];
          continue;
        }
        const size_t slot = static_cast<size_t>(me < o ? me : me - 1);
        dst[o] = peers_[o].recv + (slot * shard_total8(o) + seg_off8(o, l)) * 8;
      }
      EDL_TRY(gemm_plan_route(&w->wgrad_rs[l], static_cast<int>(prow), me, dst, n));
    }
    w->rs_plan_rows = rows;
    w->rs_plan_version = version_;
    w->rs_plan_mode = overlap_mode_;
  }
  if (overlap_mode_ == 4 && (w->x_plan_rows != rows || w->x_plan_version != version_)) {
    const int n = static_cast<int>(peers_.size());
    const int me = rep_index(r);
    w->wgrad_x.assign(static_cast<size_t>(L_), GemmPlan{});
    int order[kMaxPeerMaps] = {};
    for (size_t k = 0; k < ring_.size(); ++k) order[k] = host_index(ring_[k]);
    for (int l = 0; l < L_; ++l) {
      const bool last = l == L_ - 1;
      const __nv_bfloat16* dy = last ? r->dlog : r->dx[(l + 1) % 3];
      EDL_TRY(gemm_plan_init_sgd(&w->wgrad_x[l], dy, out_[l], 1, r->act[l], in_[l], 1,
                                 r->master + off_[l], r->W + off_[l], in_[l], out_[l], in_[l],
                                 static_cast<int>(rows)));
      const int prow = out_[l] / n;
      void* dst[kMaxPeerMaps] = {};
      __nv_bfloat16* wd[kMaxPeerMaps] = {};
      const __nv_bfloat16* src[kMaxPeerMaps] = {};
      for (int o = 0; o < n; ++o) {
        wd[o] = peers_[o].W + off_[l];
        if (o == me) continue;
        const size_t slot = static_cast<size_t>(me < o ? me : me - 1);  // mine in o's recv
        dst[o] = peers_[o].recv + (slot * shard_total8(o) + seg_off8(o, l)) * 8;
        const size_t from = static_cast<size_t>(o < me ? o : o - 1);  // o's in my recv
        src[o] = r->recv + (from * shard_total8(me) + seg_off8(me, l)) * 8;
      }
      EDL_TRY(gemm_plan_exchange(&w->wgrad_x[l], prow, me, n, dst, wd, src, in_[l], order));
    }
    w->x_plan_rows = rows;
    w->x_plan_version = version_;
  }
  if (fused_update_ && w->sgd_plan_rows != rows) {
    w->wgrad_sgd.assign(static_cast<size_t>(L_), GemmPlan{});
    for (int l = 0; l < L_; ++l) {
      const bool last = l == L_ - 1;
      const __nv_bfloat16* dy = last ? r->dlog : r->dx[(l + 1) % 3];
      if (r->mlo)  // split master: 8 B per parameter per update instead of 10
        EDL_TRY(gemm_plan_init_sgd_lo(&w->wgrad_sgd[l], dy, out_[l], r->act[l], in_[l],
                                      r->mlo + off_[l], r->W + off_[l], r->master + off_[l],
                                      in_[l], out_[l], in_[l], static_cast<int>(rows)));
      else
        EDL_TRY(gemm_plan_init_sgd(&w->wgrad_sgd[l], dy, out_[l], 1, r->act[l], in_[l], 1,
                                   r->master + off_[l], r->W + off_[l], in_[l], out_[l],
                                   in_[l], static_cast<int>(rows)));
    }
    w->sgd_plan_rows = rows;
  }
  return EDL_OK;
}

cudaEvent_t Job::mark_event() {
  if (!ev_pool_.empty()) {
    cudaEvent_t e = ev_pool_.back();
    ev_pool_.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

cudaEvent_t Job::mark_begin(cudaStream_t s) {
  if (!profile_) return nullptr;
  cudaEvent_t e = mark_event();
  cudaEventRecord(e, s);
  return e;
}

cudaEvent_t Job::mark(int slot, int phase, cudaEvent_t start, cudaStream_t s) {
  if (!profile_ || !start) return nullptr;
  cudaEvent_t e = mark_event();
  cudaEventRecord(e, s);
  marks_[slot].push_back(Mark{phase, start, e});
  return e;
}

int Job::run_worker_mlp(Worker* w, int slot, bool last) {
  Replica* r = w->rep;
  DeviceGuard dg(r->device);
  const bool prof = profile_ && r == primary();
  const int64_t rows = static_cast<int64_t>(w->plan.size());
  double* wloss = w->loss + (t_ & 1);
  EDL_CUDA_TRY(cudaEventRecord(w->ev_w0[slot], r->stream));
  if (rows == 0) {  // ShardPending for the whole step: contributes a zero gradient
    EDL_CUDA_TRY(cudaMemsetAsync(wloss, 0, sizeof(double), r->stream));
    EDL_CUDA_TRY(cudaMemsetAsync(w->grad, 0, sizeof(__nv_bfloat16) * P_, r->stream));
    if (overlap_ && last) EDL_TRY(finish_layer_colls(r));  // mode 3 needs rows > 0
    EDL_CUDA_TRY(cudaEventRecord(w->ev_w1[slot], r->stream));
    return EDL_OK;
  }
  EDL_TRY(ensure_plans(w, rows));
  cudaEvent_t m = prof ? mark_begin(r->stream) : nullptr;
  EdlRun* host = w->runs_host + static_cast<size_t>(slot) * w->runs_cap;
  if (w->n_runs <= kInlineRuns) {  // runs ride in the launch parameters; loss zeroed there
    EDL_TRY(gather_inline(r->ds, host, w->n_runs, rows, r->act[0], r->labels, wloss,
                          r->stream));
  } else {
    EDL_CUDA_TRY(cudaMemsetAsync(wloss, 0, sizeof(double), r->stream));
    EDL_CUDA_TRY(cudaMemcpyAsync(w->runs_dev, host, sizeof(EdlRun) * w->n_runs,
                                 cudaMemcpyHostToDevice, r->stream));
    EDL_TRY(gather(r->ds, w->runs_dev, w->n_runs, rows, r->act[0], r->labels, r->stream));
  }
  m = mark(slot, 0, m, r->stream);
  if (r->ag_wait_epoch) {
    // layer l's weights may still be arriving from the previous mini-batch's push collective
    // (side stream, every replica): the GEMM's producer waits for the layer's flags
    const int n_rep = static_cast<int>(peers_.size());
    for (int l = 0; l < L_; ++l)
      EDL_TRY(gemm_plan_run_wait(r->fwd[l], r->stream, ag_layer_flags(r->flags, l), n_rep,
                                 r->ag_wait_epoch));
  } else if (join_.pending) {
    // a newcomer's first mini-batch: layer l's weights are still arriving from the source,
    // which writes the layer's flag word after them (install_out_mp)
    for (int l = 0; l < L_; ++l)
      EDL_TRY(gemm_plan_run_wait(r->fwd[l], r->stream, ag_layer_flags(r->flags, l),
                                 join_.n_src, static_cast<uint32_t>(join_.version)));
  } else {
    for (int l = 0; l < L_; ++l) EDL_TRY(gemm_plan_run(r->fwd[l], r->stream));
  }
  m = mark(slot, 1, m, r->stream);
  // softmax cross-entropy + the worker's ordered loss sum in one kernel
  EDL_TRY(softmax_xent(r->logits, r->labels, static_cast<int>(rows), cfg_.num_classes, r->dlog,
                       r->row_loss, wloss, r->xent_done, r->stream));
  m = mark(slot, 2, m, r->stream);
  // N = 1 fused update: dgrad of layer l-1 and wgrad + SGD of layer l share one launch
  // (bwd_pair.cu) -- the tensor-bound and the HBM-bound halves of the backward overlap
  bool pair = fused_update_ && !overlap_ && L_ >= 3 && gemm_pair_enabled();
  for (int l = 2; pair && l < L_; ++l)
    pair = gemm_pair_eligible(r->dgrad[l - 1], w->wgrad_sgd[l]);
  if (pair) {
    EDL_TRY(gemm_plan_run(r->dgrad[L_ - 1], r->stream));
    for (int l = L_ - 1; l >= 2; --l) {
      cudaEvent_t mp = prof ? mark_begin(r->stream) : nullptr;
      EDL_TRY(gemm_pair_run(r->dgrad[l - 1], w->wgrad_sgd[l], r->stream, step_scale_));
      if (mp) mark(slot, 6, mp, r->stream);
    }
    for (int l = 1; l >= 0; --l) {
      cudaEvent_t mw = prof ? mark_begin(r->stream) : nullptr;
      EDL_TRY(gemm_plan_run(w->wgrad_sgd[l], r->stream, step_scale_));
      if (mw) mark(slot, 5, mw, r->stream);
    }
  }
  for (int l = pair ? -1 : L_ - 1; l >= 0; --l) {
    if (l > 0 && (fused_update_ || !r->dgrad[l].ep.l2pf_bytes)) {
      EDL_TRY(gemm_plan_run(r->dgrad[l], r->stream));
    } else if (l > 0) {  // the master prefetch only serves the fused update
      GemmPlan q = r->dgrad[l];
      q.ep.l2pf_bytes = 0;
      EDL_TRY(gemm_plan_run(q, r->stream));
    }
    const bool fused_here = fused_update_ && (!overlap_ || l == 0);
    if (!fused_here && (overlap_mode_ == 3 || overlap_mode_ == 5) && r->side_pending) {
      // the previous push collective reads every replica's recv until its final barrier
      // (waited on before the wgrad sub-phase mark so the wait is not timed as GEMM work)
      EDL_CUDA_TRY(cudaStreamWaitEvent(r->stream, r->ev_push, 0));
      r->side_pending = false;
    }
    cudaEvent_t mw = prof ? mark_begin(r->stream) : nullptr;  // wgrad sub-phase
    if (fused_here) {
      // dW + sgd_step in one kernel (layer 0 ends the backward: nothing left to overlap)
      EDL_TRY(run_sgd_plan(w->wgrad_sgd[l], r));
      if (mw) mark(slot, 5, mw, r->stream);
    } else if (overlap_mode_ == 4) {
      // dW + reduce-scatter + sharded SGD + weight all-gather in one kernel per layer
      EDL_TRY(gemm_plan_run(w->wgrad_x[l], r->stream, step_scale_));
      if (mw) mark(slot, 5, mw, r->stream);
    } else if (overlap_mode_ == 3 || overlap_mode_ == 6 ||
               (overlap_mode_ == 5 && rs_tma_every() > 0 && l % rs_tma_every() == 0)) {
      // dW with the reduce-scatter in its epilogue: rows owned elsewhere are stored into the
      // owner's recv over NVLink while the backward continues; the shard update + all-gather
      // run once, after the backward (the push collective with its phase A skipped)
      EDL_TRY(gemm_plan_run(w->wgrad_rs[l], r->stream));
      if (mw) mark(slot, 5, mw, r->stream);
      // mode 6: the far owners' rows were written locally; the copy engines move them
      if (overlap_mode_ == 6 && last) EDL_TRY(launch_layer_rs_ce(r, l));
      if (overlap_mode_ == 5 && last) ++r->layer_colls;  // this layer went out from the GEMM
    } else {
      EDL_TRY(gemm_plan_run(w->wgrad[l], r->stream));
      if (mw) mark(slot, 5, mw, r->stream);
      if (overlap_ && last) EDL_TRY(launch_layer_coll(r, l));
    }
  }
  // the fused launches above left the master split or, before a switch, in fp32
  if (fused_update_ && r->mlo) r->lo_live = split_step_ && sgd_out_split_;
  if (w->delay_us > 0) {
    EDL_TRY(spin(static_cast<uint64_t>(w->delay_us * 1e3), r->stream));
    launches_ += 1;
  }
  EDL_CUDA_TRY(cudaEventRecord(w->ev_w1[slot], r->stream));
  if (overlap_ && last && overlap_mode_ != 3 && overlap_mode_ != 4) EDL_TRY(finish_layer_colls(r));
  m = mark(slot, 3, m, r->stream);
  (void)m;
  // gather + L fwd + softmax-CE + backward (2L - 1 GEMMs, or L - 2 of them paired)
  launches_ += 1 + static_cast<uint64_t>(L_) + 1 +
               static_cast<uint64_t>(pair ? L_ + 1 : 2 * L_ - 1);
  return EDL_OK;
}

// Layer l's update on the replica's side stream, after the main stream's layer-l weight
// gradients (of every local worker: they run in stream order before this point).  With
// several replicas it is the fused NVLink collective restricted to layer l's parameters;
// the shard boundaries, epochs and launch order are the same on every replica.
// Exchange mode 5: layer l's reduce-scatter on the copy engines as soon as its weight
// gradients exist (plain wgrad GEMM, local gradient), under the rest of the backward; the
// push collective after the backward then sums, updates and all-gathers as in mode 3.
int Job::launch_layer_rs_ce(Replica* r, int l) {
  EDL_CUDA_TRY(cudaEventRecord(r->ev_grad[l], r->stream));
  const int n_rep = static_cast<int>(peers_.size());
  const int me = rep_index(r);
  const size_t base = off_[l];
  // one stream per peer offset (up to three), so several copy engines run at once
  cudaStream_t cs[3] = {r->side2, r->side3, r->side};
  for (int j = 1; j < n_rep && j <= 3; ++j)
    EDL_CUDA_TRY(cudaStreamWaitEvent(cs[j - 1], r->ev_grad[l], 0));
  for (int j = 1; j < n_rep; ++j) {
    if (overlap_mode_ == 6 && !rs_via_ce(j, n_rep)) continue;  // stored by the wgrad GEMM
    const int p = (me + j) % n_rep;  // rotated: every GPU copies to a different owner first
    cudaStream_t st = cs[(j - 1) % 3];
    size_t lo;
    const size_t n8 = shard8(l, p, &lo);
    if (n8 == 0) continue;
    const size_t slot8 = shard_total8(p);
    for (size_t k = 0; k < ring_.size(); ++k) {
      if (host_index(ring_[k]) != me) continue;
      __nv_bfloat16* dst =
          peers_[p].recv + (static_cast<size_t>(recv_slot(p, k)) * slot8 + seg_off8(p, l)) * 8;
      const __nv_bfloat16* src = workers_[ring_[k]]->grad + base + lo * 8;
      EDL_CUDA_TRY(cudaMemcpyAsync(dst, src, n8 * 16, cudaMemcpyDeviceToDevice, st));
    }
  }
  ++r->layer_colls;
  return EDL_OK;
}

// Mode 6 (three or more GPUs): the reduce-scatter to the nearest EDL_RS_TMA_PEERS peer
// offsets (default (N-1)/2, at least 1) is stored from the wgrad GEMM epilogues (mode 3), to the others by the
// copy engines (mode 5), so SM stores and copy engines share the NVLink egress.
// Mode 5 variant (EDL_RS_TMA_EVERY=k): every k-th layer's reduce-scatter is stored from the
// wgrad GEMM epilogue (mode 3) instead of the copy engines
int Job::rs_tma_every() const {
  static int k = -1;
  if (k < 0) {
    const char* e = getenv("EDL_RS_TMA_EVERY");
    k = e ? atoi(e) : 0;
  }
  return k;
}

bool Job::rs_via_ce(int j, int n_rep) const {
  // default: half of the peers (rounded down, at least one) through the SM stores; measured
  // at N=4: 1 peer 2.013M, 2 peers 2.019M samples/s
  static int tma_env = -2;
  if (tma_env == -2) {
    const char* e = getenv("EDL_RS_TMA_PEERS");
    tma_env = e ? atoi(e) : -1;
  }
  const int tma_peers = tma_env >= 0 ? tma_env : ((n_rep - 1) / 2 > 1 ? (n_rep - 1) / 2 : 1);
  return j > tma_peers && j < n_rep;
}

int Job::launch_layer_coll(Replica* r, int l) {
  if (overlap_mode_ == 2) return launch_layer_ce(r, l);
  if (overlap_mode_ == 5 || overlap_mode_ == 6) return launch_layer_rs_ce(r, l);
  EDL_CUDA_TRY(cudaEventRecord(r->ev_grad[l], r->stream));
  EDL_CUDA_TRY(cudaStreamWaitEvent(r->side, r->ev_grad[l], 0));
  const int n_rep = static_cast<int>(peers_.size());
  const int me = rep_index(r);
  CollArgs a;
  for (const auto& id : ring_) a.grads[a.n_src++] = workers_[id]->grad;
  for (const auto& p : peers_) {
    a.flags[a.n_dst] = p.flags;
    a.w_dst[a.n_dst++] = p.W;
  }
  a.me = me;
  a.n_rep = n_rep;
  a.epoch = layer_epoch0_ + static_cast<uint32_t>(r->layer_colls);
  const size_t len8 = static_cast<size_t>(in_[l]) * out_[l] / 8, base8 = off_[l] / 8;
  shard_range(len8, n_rep, me, &a.lo8, &a.hi8);  // = own_segments()'s segment of layer l
  a.lo8 += base8;
  a.hi8 += base8;
  a.master = r->master;
  a.mom = r->mom;
  const double eta_t = cfg_.eta / (1.0 + cfg_.decay * static_cast<double>(t_));
  a.scale = static_cast<float>(eta_t / static_cast<double>(step_count_));
  a.inv_count = static_cast<float>(1.0 / static_cast<double>(step_count_));
  a.eta = static_cast<float>(eta_t);
  a.mu = static_cast<float>(cfg_.momentum);
  a.update = 1;
  static int blocks = -1;  // one CTA per SM: co-resides with the backward GEMMs
  if (blocks < 0) {
    const char* e = getenv("EDL_OVERLAP_BLOCKS");
    blocks = e ? atoi(e) : 148;
  }
  a.blocks = blocks;
  EDL_TRY(allreduce_sgd(a, r->side));
  ++r->layer_colls;
  launches_ += 1;
  return EDL_OK;
}

int Job::host_index(const std::string& id) const {
  const Worker* w = workers_.at(id).get();
  for (size_t i = 0; i < peers_.size(); ++i) {
    if (!w->remote && peers_[i].local && peers_[i].rep == w->rep) return static_cast<int>(i);
    if (w->remote && peers_[i].rank == w->host_rank) return static_cast<int>(i);
  }
  return -1;
}

size_t Job::shard8(int l, int p, size_t* lo) const {
  size_t a, b;
  shard_range(static_cast<size_t>(in_[l]) * out_[l] / 8, static_cast<int>(peers_.size()), p, &a,
              &b);
  if (lo) *lo = a;
  return b - a;
}

size_t Job::shard_total8(int p) const {
  size_t t = 0;
  for (int l = 0; l < L_; ++l) t += shard8(l, p, nullptr);
  return t;
}

size_t Job::seg_off8(int p, int l) const {
  size_t t = 0;
  for (int k = 0; k < l; ++k) t += shard8(k, p, nullptr);
  return t;
}

// Replica p's recv buffer holds one slot (its whole shard) per ring member hosted elsewhere,
// in ring order.
int Job::recv_slot(int p, size_t k) const {
  int j = 0;
  for (size_t i = 0; i < k; ++i)
    if (host_index(ring_[i]) != p) ++j;
  return j;
}

// Mode 3 needs one ring member per replica (its gradient is the replica's), every member
// with a non-empty batch this step, and layer widths that split into 32-row owner blocks.
bool Job::rs_eligible() const {
  const int n = static_cast<int>(peers_.size());
  if (!mlp_ || n < 2 || n > kMaxPeerMaps || ring_.size() != peers_.size()) return false;
  std::vector<int> seen(static_cast<size_t>(n), 0);
  for (const auto& id : ring_) {
    const int h = host_index(id);
    if (h < 0 || seen[static_cast<size_t>(h)]++) return false;
    const Worker* w = workers_.at(id).get();
    if (w->plan.empty() || (w->remote && !w->imported)) return false;
  }
  for (const auto& p : peers_)
    if (!p.recv || !p.W || !p.flags) return false;
  for (int l = 0; l < L_; ++l)
    if (out_[l] % (32 * n) != 0 || out_[l] < 256) return false;
  return true;
}

// Push collective: one ring member per replica, every replica's recv mapped here.
// Mode 4 keeps whole 256-row tiles inside one owner block, plain SGD (the epilogue applies
// the update), and a topology that has not changed since the job started (every receive slot
// must hold the "not arrived" sentinel at the start of a mini-batch, which mode 4 restores
// after consuming; other modes leave gradients there).
bool Job::xchg_eligible() const {
  if (!rs_eligible() || cfg_.momentum != 0.0 || version_ != 1) return false;
  const int n = static_cast<int>(peers_.size());
  for (int l = 0; l < L_; ++l)
    if (out_[l] % (256 * n) != 0 || in_[l] % 128 != 0) return false;
  return true;
}

bool Job::push_eligible() const {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("EDL_COLL_PUSH");
    env = e && *e ? atoi(e) : 1;
  }
  const int n = static_cast<int>(peers_.size());
  if (!env || !mlp_ || n < 2 || ring_.size() != peers_.size()) return false;
  std::vector<int> seen(static_cast<size_t>(n), 0);
  for (const auto& id : ring_) {
    const int h = host_index(id);
    if (h < 0 || seen[static_cast<size_t>(h)]++) return false;
  }
  for (const auto& p : peers_)
    if (!p.recv || !p.W || !p.flags) return false;
  return true;
}

bool Job::ce_fits() const {
  for (size_t p = 0; p < peers_.size(); ++p) {
    if (!peers_[p].recv || !peers_[p].W) return false;
    size_t remote = 0;
    for (const auto& id : ring_) {
      const int h = host_index(id);
      if (h < 0) return false;
      if (h != static_cast<int>(p)) ++remote;
    }
    if (remote * shard_total8(static_cast<int>(p)) * 8 > P_) return false;
  }
  return ring_.size() <= static_cast<size_t>(kCollMaxSources);
}

// Layer l with copy-engine transfers, on the replica's side stream:
//   push my members' gradient slices of layer l owned by each peer into that peer's recv
//   (cudaMemcpyAsync over NVLink), signal; wait for every peer's slices of my shard; apply
//   the ring-order sum + SGD to my shard (shard_update); push my updated bf16 weights of the
//   shard into every peer's W, signal.  The NVLink bytes are the reduce-scatter +
//   all-gather lower bound, moved by the copy engines while the SMs run the backward.
// ------------------------------------------------------------------ failure recovery
// SPEC.md:321-329 / PAPER.md §4.2; the oracle (oracle/job_driver.hpp restore /
// fail_approximate) applies the same lease / ring / log transitions.

int Job::take_pre_snapshot() {
  pre_.valid = true;
  pre_.t = t_;
  pre_.version = version_;
  pre_.ring = ring_;
  pre_.lease = lm_->snapshot();
  pre_.cur.clear();
  for (const auto& id : ring_) pre_.cur[id] = workers_[id]->cur;
  pre_.log_len = log_.size();
  if (dry_) return EDL_OK;
  for (auto& [dev, r] : reps_) {  // device copy in stream order: the state before this step
    DeviceGuard g(dev);
    if (mlp_) {
      if (!r->shadow_master) EDL_TRY(dalloc(&r->shadow_master, P_));
      EDL_CUDA_TRY(cudaMemcpyAsync(r->shadow_master, r->master, sizeof(float) * P_,
                                   cudaMemcpyDeviceToDevice, r->stream));
      if (r->mom) {
        if (!r->shadow_mom) EDL_TRY(dalloc(&r->shadow_mom, P_));
        EDL_CUDA_TRY(cudaMemcpyAsync(r->shadow_mom, r->mom, sizeof(float) * P_,
                                     cudaMemcpyDeviceToDevice, r->stream));
      }
    } else {
      if (!r->shadow_w) EDL_TRY(dalloc(&r->shadow_w, P_));
      EDL_CUDA_TRY(cudaMemcpyAsync(r->shadow_w, r->w, sizeof(double) * P_,
                                   cudaMemcpyDeviceToDevice, r->stream));
    }
  }
  return EDL_OK;
}

// Immediate scale-in of `ids` (failed workers): shards back at their reported offsets.
int Job::remove_members(const std::vector<std::string>& ids) {
  EDL_TRY(master_current());  // the deferred push collective / split master
  std::vector<std::string> keep;
  for (const auto& id : ring_) {
    if (std::find(ids.begin(), ids.end(), id) == ids.end()) {
      keep.push_back(id);
      continue;
    }
    lm_->reclaim(id);
    lm_->retire(id);
    auto it = workers_.find(id);
    if (!dry_ && !it->second->remote) free_worker(it->second.get());
    workers_.erase(it);
  }
  ring_ = keep;
  rebuild_peers();
  return EDL_OK;
}

namespace {
constexpr char kCkptMagic[8] = {'E', 'D', 'L', 'C', 'K', 'P', 'T', '1'};
template <class T>
void put(std::string* b, const T& v) {
  b->append(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <class T>
bool get(const std::string& b, size_t* o, T* v) {
  if (*o + sizeof(T) > b.size()) return false;
  std::memcpy(v, b.data() + *o, sizeof(T));
  *o += sizeof(T);
  return true;
}
}  // namespace

int Job::save_checkpoint(const std::string& path) {
  EDL_TRY(master_current());  // the deferred push collective / split master
  if (path.empty()) return fail(EDL_EINVAL, "checkpoint: empty path");
  // one process per GPU: a collective -- every ring process saves at the same boundary (the
  // fp32 master / momentum shards are all-gathered, then each process writes the identical
  // checkpoint from its own replica; the host state is the same everywhere by construction)
  bool all_local = true;
  for (const auto& p : peers_) all_local = all_local && p.local;
  EDL_TRY(sync(nullptr));
  std::string b(kCkptMagic, 8);
  put<uint32_t>(&b, 1);  // format version
  put<int32_t>(&b, cfg_.model);
  put<uint64_t>(&b, t_);
  put<uint64_t>(&b, version_);
  put<int64_t>(&b, cfg_.batch);
  put<uint64_t>(&b, static_cast<uint64_t>(P_));
  put<uint32_t>(&b, static_cast<uint32_t>(ring_.size()));
  for (const auto& id : ring_) {
    put<uint32_t>(&b, static_cast<uint32_t>(id.size()));
    b += id;
  }
  const std::vector<uint8_t> lease = lm_->snapshot();  // PipelineCheckpoint + RNG state
  put<uint64_t>(&b, lease.size());
  b.append(reinterpret_cast<const char*>(lease.data()), lease.size());
  const size_t esz = mlp_ ? sizeof(float) : sizeof(double);
  std::vector<char> params(dry_ ? 0 : esz * P_), mom;
  if (!dry_) {
    Replica* r = primary();
    if (all_local)
      EDL_TRY(consolidate_master());
    else
      EDL_TRY(gather_master());
    DeviceGuard g(r->device);
    EDL_CUDA_TRY(cudaStreamSynchronize(r->stream));
    EDL_CUDA_TRY(cudaMemcpy(params.data(), mlp_ ? static_cast<void*>(r->master)
                                                : static_cast<void*>(r->w),
                            params.size(), cudaMemcpyDeviceToHost));
    if (mlp_ && r->mom) {
      mom.resize(sizeof(float) * P_);
      EDL_CUDA_TRY(cudaMemcpy(mom.data(), r->mom, mom.size(), cudaMemcpyDeviceToHost));
    }
  }
  put<uint64_t>(&b, params.size());
  b.append(params.data(), params.size());
  put<uint64_t>(&b, mom.size());
  b.append(mom.data(), mom.size());
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return fail(EDL_EIO, "checkpoint: cannot open " + path);
  const bool ok = std::fwrite(b.data(), 1, b.size(), f) == b.size();
  if (std::fclose(f) != 0 || !ok) return fail(EDL_EIO, "checkpoint: write failed " + path);
  last_ckpt_ = path;
  return EDL_OK;
}

int Job::load_checkpoint(const std::string& path) {
  EDL_TRY(master_current());  // the deferred push collective / split master
  // one process per GPU: every ring process loads the same checkpoint (each replica then
  // holds the whole model, which the sharded update keeps consistent from here)
  if (!events_.empty()) return fail(EDL_RETRY, "checkpoint: a scaling operation is pending");
  std::string b;
  {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return fail(EDL_EIO, "checkpoint: cannot open " + path);
    char buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) b.append(buf, n);
    std::fclose(f);
  }
  size_t o = 8;
  if (b.size() < 8 || std::memcmp(b.data(), kCkptMagic, 8) != 0)
    return fail(EDL_EINVAL, "checkpoint: not an edl checkpoint");
  uint32_t fmt = 0, nring = 0;
  int32_t model = 0;
  uint64_t t = 0, version = 0, P = 0, llen = 0, plen = 0, mlen = 0;
  int64_t B = 0;
  bool ok = get(b, &o, &fmt) && get(b, &o, &model) && get(b, &o, &t) && get(b, &o, &version) &&
            get(b, &o, &B) && get(b, &o, &P) && get(b, &o, &nring);
  std::vector<std::string> ring;
  for (uint32_t i = 0; ok && i < nring; ++i) {
    uint32_t len = 0;
    ok = get(b, &o, &len) && o + len <= b.size();
    if (ok) ring.emplace_back(b.data() + o, len);
    o += len;
  }
  ok = ok && get(b, &o, &llen) && o + llen <= b.size();
  const size_t lease_at = o;
  o += ok ? llen : 0;
  ok = ok && get(b, &o, &plen) && o + plen <= b.size();
  const size_t params_at = o;
  o += ok ? plen : 0;
  ok = ok && get(b, &o, &mlen) && o + mlen <= b.size();
  const size_t mom_at = o;
  if (!ok || fmt != 1) return fail(EDL_ETRUNCATED, "checkpoint: truncated payload");
  if (model != cfg_.model || P != P_ || B != cfg_.batch)
    return fail(EDL_SHAPE_MISMATCH, "checkpoint: model / size / batch differ from the job");
  const size_t esz = mlp_ ? sizeof(float) : sizeof(double);
  if (!dry_ && plen != esz * P_) return fail(EDL_SHAPE_MISMATCH, "checkpoint: parameter bytes");
  if (mlen != 0 && mlen != sizeof(float) * P_)
    return fail(EDL_SHAPE_MISMATCH, "checkpoint: momentum bytes");
  // pipeline: lease state as checkpointed, parsed into a copy first so a rejected or
  // truncated payload leaves the job untouched; the checkpointed members' in-flight shards go
  // back to the reclaimed queue at their offsets (their cursors are gone), leavers retire
  auto lm = std::make_unique<LeaseManager>(*lm_);
  LeaseStatus ls;
  try {
    ls = lm->restore(reinterpret_cast<const uint8_t*>(b.data()) + lease_at, llen);
  } catch (const std::exception&) {
    return fail(EDL_ETRUNCATED, "checkpoint: truncated lease state");
  }
  if (ls != LeaseStatus::Ok) return fail(EDL_SHAPE_MISMATCH, "checkpoint: lease state rejected");
  for (const auto& id : ring) {
    lm->reclaim(id);
    if (std::find(ring_.begin(), ring_.end(), id) == ring_.end()) lm->retire(id);
  }
  for (const auto& id : ring_)
    if (std::find(ring.begin(), ring.end(), id) == ring.end()) lm->enroll(id);
  // everything validated: parameters (every replica; MLP bf16 weights re-derived from the
  // master), momentum, lease state and t_cur change together
  EDL_TRY(sync(nullptr));
  if (!dry_) {
    EDL_TRY(set_params(b.data() + params_at, plen));
    for (auto& [dev, r] : reps_) {
      if (!r->mom) continue;
      DeviceGuard g(dev);
      if (mlen == sizeof(float) * P_)
        EDL_CUDA_TRY(cudaMemcpy(r->mom, b.data() + mom_at, mlen, cudaMemcpyHostToDevice));
      else
        EDL_CUDA_TRY(cudaMemsetAsync(r->mom, 0, sizeof(float) * P_, r->stream));
    }
  }
  lm_ = std::move(lm);
  for (auto& [id, w] : workers_) w->cur = Cursor{};
  t_ = t;
  version_ = std::max(version_, version) + 1;
  pre_.valid = false;
  if (cfg_.keep_log) {
    if (t_ > 0) {
      LogRec r;
      r.kind = LogRec::Restore;
      r.t = t_ - 1;
      log_.push_back(r);
    }
    LogRec r;
    r.kind = LogRec::Topo;
    r.t = t_ == 0 ? 0 : t_ - 1;
    r.version = version_;
    r.ring = ring_;
    log_.push_back(r);
  }
  resplit();
  return EDL_OK;
}

int Job::recover(const std::vector<std::string>& failed, bool approximate, EdlRecovery* out) {
  EDL_TRY(master_current());  // the deferred push collective / split master
  bool all_local = true;
  for (const auto& p : peers_) all_local = all_local && p.local;
  // one process per GPU: consistent recovery only -- each survivor drops the failed
  // processes' replicas (never touching their memory again) and reloads its checkpoint.
  // Approximate recovery would need the failed GPU's fp32 master shard, which died with it.
  if (!all_local && approximate)
    return fail(EDL_EINVAL, "recover: approximate recovery needs every master shard "
                            "(single process); use consistent recovery across processes");
  size_t hit = 0;
  for (const auto& id : failed) hit += std::count(ring_.begin(), ring_.end(), id);
  if (hit == 0 || hit != failed.size()) return fail(EDL_UNKNOWN_WORKER, "recover: not ring members");
  if (hit >= ring_.size()) return fail(EDL_EINVAL, "recover: no surviving worker");
  if (!events_.empty()) return fail(EDL_RETRY, "recover: a scaling operation is pending");
  EDL_TRY(sync(nullptr));
  *out = EdlRecovery{};
  out->mode = approximate ? 1 : 0;
  out->status = EDL_OK;
  if (approximate) {
    if (!cfg_.appx_recovery || !pre_.valid)
      return fail(EDL_EINVAL, "recover: approximate recovery needs cfg.appx_recovery");
    // model: back to the boundary state (every replica restores its own copy; the sharded
    // master is made whole before the membership change re-shards it)
    if (!dry_) {
      for (auto& [dev, r] : reps_) {
        DeviceGuard g(dev);
        if (mlp_) {
          EDL_CUDA_TRY(cudaMemcpyAsync(r->master, r->shadow_master, sizeof(float) * P_,
                                       cudaMemcpyDeviceToDevice, r->stream));
          if (r->mom)
            EDL_CUDA_TRY(cudaMemcpyAsync(r->mom, r->shadow_mom, sizeof(float) * P_,
                                         cudaMemcpyDeviceToDevice, r->stream));
        } else {
          EDL_CUDA_TRY(cudaMemcpyAsync(r->w, r->shadow_w, sizeof(double) * P_,
                                       cudaMemcpyDeviceToDevice, r->stream));
        }
      }
      EDL_TRY(consolidate_master());
      if (mlp_)
        for (auto& [dev, r] : reps_) {
          DeviceGuard g(dev);
          EDL_TRY(master_to_bf16(r->master, r->W, P_, r->stream));
        }
    }
    // pipeline and protocol state: back to the start of the failed mini-batch
    if (lm_->restore(pre_.lease.data(), pre_.lease.size()) != LeaseStatus::Ok)
      return fail(EDL_EINVAL, "recover: lease rollback failed");
    for (const auto& id : ring_) {
      auto it = pre_.cur.find(id);
      workers_[id]->cur = it == pre_.cur.end() ? Cursor{} : it->second;
    }
    if (log_.size() > pre_.log_len) log_.resize(pre_.log_len);
    t_ = pre_.t;
    version_ = pre_.version;
    pre_.valid = false;
    EDL_TRY(remove_members(failed));
  } else {
    EDL_TRY(remove_members(failed));
    if (!last_ckpt_.empty()) {
      EDL_TRY(load_checkpoint(last_ckpt_));
      out->t_resume = t_;
      out->version = version_;
      return EDL_OK;
    }
    // no checkpoint: the survivors restart from the initial state
    out->status = EDL_NO_CHECKPOINT;
    lm_ = std::make_unique<LeaseManager>(cfg_.data.size, lm_parts_, cfg_.lease_seed, lm_loc_);
    for (const auto& id : ring_) {
      lm_->enroll(id);
      workers_[id]->cur = Cursor{};
    }
    if (!dry_) {
      for (auto& [dev, r] : reps_) {
        DeviceGuard g(dev);
        if (mlp_) {
          for (int l = 0; l < L_; ++l) {
            const double bound = std::sqrt(6.0 / static_cast<double>(in_[l]));
            EDL_TRY(mlp_init_weights(r->master + off_[l], r->W + off_[l],
                                     static_cast<size_t>(in_[l]) * out_[l], cfg_.init_seed,
                                     off_[l], bound, r->stream));
          }
          if (r->mom) EDL_CUDA_TRY(cudaMemsetAsync(r->mom, 0, sizeof(float) * P_, r->stream));
        } else {
          EDL_CUDA_TRY(cudaMemsetAsync(r->w, 0, sizeof(double) * P_, r->stream));
        }
      }
    }
    t_ = 0;
    if (cfg_.keep_log) log_.clear();
  }
  ++version_;
  if (cfg_.keep_log) {
    LogRec r;
    r.kind = LogRec::Topo;
    r.t = t_ == 0 ? 0 : t_ - 1;
    r.version = version_;
    r.ring = ring_;
    log_.push_back(r);
  }
  resplit();
  out->t_resume = t_;
  out->version = version_;
  return EDL_OK;
}

int Job::set_worker_delay(const std::string& id, double us) {
  auto it = workers_.find(id);
  if (it == workers_.end()) return fail(EDL_UNKNOWN_WORKER, "set_worker_delay: unknown worker " + id);
  if (!(us >= 0.0)) return fail(EDL_EINVAL, "set_worker_delay: negative delay");
  it->second->delay_us = us;
  return EDL_OK;
}

int Job::worker_ms(const std::string& id, std::vector<double>* out) const {
  out->clear();
  for (const auto& step : wtimes_)
    for (const auto& [wid, ms] : step)
      if (wid == id) out->push_back(ms);
  return EDL_OK;
}

std::string Job::straggler(int window, double factor) const {
  if (window < 1 || wtimes_.size() < static_cast<size_t>(window)) return "";
  std::vector<std::string> ids;
  std::vector<double> dur;  // [window][ids.size()], NaN = absent
  const size_t first = wtimes_.size() - static_cast<size_t>(window);
  for (size_t b = first; b < wtimes_.size(); ++b)
    for (const auto& [id, ms] : wtimes_[b])
      if (std::find(ids.begin(), ids.end(), id) == ids.end()) ids.push_back(id);
  dur.assign(static_cast<size_t>(window) * ids.size(), std::nan(""));
  for (size_t b = first; b < wtimes_.size(); ++b)
    for (const auto& [id, ms] : wtimes_[b]) {
      const size_t k = static_cast<size_t>(std::find(ids.begin(), ids.end(), id) - ids.begin());
      dur[(b - first) * ids.size() + k] = ms;
    }
  const int k = detect_straggler(dur.data(), window, static_cast<int>(ids.size()), window, factor);
  return k >= 0 ? ids[static_cast<size_t>(k)] : "";
}

// worker k is a straggler if in each of the last `window`
// mini-batches its duration exceeds factor x that mini-batch's median over the workers
// present (strict inequality; median of an even count = mean of the middle two).  Returns
// the lowest such index, or -1.  durations: [n_batches][n_workers], NaN = absent.
int detect_straggler(const double* dur, int n_batches, int n_workers, int window, double factor) {
  if (window < 1 || n_batches < window || n_workers < 1) return -1;
  std::vector<int> hits(static_cast<size_t>(n_workers), 0);
  for (int b = n_batches - window; b < n_batches; ++b) {
    std::vector<double> v;
    for (int k = 0; k < n_workers; ++k) {
      const double d = dur[static_cast<size_t>(b) * n_workers + k];
      if (!std::isnan(d)) v.push_back(d);
    }
    if (v.empty()) return -1;
    std::sort(v.begin(), v.end());
    const size_t m = v.size();
    const double med = (m % 2) ? v[m / 2] : 0.5 * (v[m / 2 - 1] + v[m / 2]);
    for (int k = 0; k < n_workers; ++k) {
      const double d = dur[static_cast<size_t>(b) * n_workers + k];
      if (!std::isnan(d) && d > factor * med) ++hits[static_cast<size_t>(k)];
    }
  }
  for (int k = 0; k < n_workers; ++k)
    if (hits[static_cast<size_t>(k)] == window) return k;
  return -1;
}

void Job::ce_mark(const std::string& what, cudaStream_t s) {
  if (!ce_trace_ || ce_marks_.size() >= 256) return;
  if (!ce_stamps_ && cudaHostAlloc(&ce_stamps_, 256 * sizeof(unsigned long long),
                                   cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
    return;
  stamp(ce_stamps_ + ce_marks_.size(), s);
  ce_marks_.push_back(what);
}

int Job::launch_layer_ce(Replica* r, int l) {
  // side2: reduce-scatter pushes of layer l (as soon as its gradients exist); side: the
  // update + all-gather of layer l, pipelined against layer l-1's pushes
  EDL_CUDA_TRY(cudaEventRecord(r->ev_grad[l], r->stream));
  ce_mark("L" + std::to_string(l) + " wgrad done (main)", r->stream);
  EDL_CUDA_TRY(cudaStreamWaitEvent(r->side2, r->ev_grad[l], 0));
  const int n_rep = static_cast<int>(peers_.size());
  const int me = rep_index(r);
  const size_t base = off_[l];
  for (int p = 0; p < n_rep; ++p) {
    if (p == me) continue;
    size_t lo;
    const size_t n8 = shard8(l, p, &lo);
    if (n8 == 0) continue;
    const size_t slot8 = shard_total8(p);
    for (size_t k = 0; k < ring_.size(); ++k) {
      if (host_index(ring_[k]) != me) continue;
      __nv_bfloat16* dst =
          peers_[p].recv + (static_cast<size_t>(recv_slot(p, k)) * slot8 + seg_off8(p, l)) * 8;
      const __nv_bfloat16* src = workers_[ring_[k]]->grad + base + lo * 8;
      EDL_CUDA_TRY(cudaMemcpyAsync(dst, src, n8 * 16, cudaMemcpyDeviceToDevice, r->side2));
    }
  }
  CeSignal sg;
  for (int p = 0; p < n_rep; ++p) sg.flags[p] = peers_[p].flags;
  sg.n_rep = n_rep;
  sg.me = me;
  sg.kind = 0;
  sg.layer = l;
  sg.epoch = ce_epoch_;
  EDL_TRY(ce_signal(sg, r->side2));
  ce_mark("L" + std::to_string(l) + " RS pushed (side2)", r->side2);
  EDL_CUDA_TRY(cudaEventRecord(r->ev_rs[l], r->side2));
  EDL_CUDA_TRY(cudaStreamWaitEvent(r->side, r->ev_rs[l], 0));
  CeWait cw;
  cw.flags = r->flags;
  cw.n_rep = n_rep;
  cw.me = me;
  cw.kind = 0;
  cw.l_lo = l;
  cw.l_hi = l + 1;
  cw.epoch = ce_epoch_;
  EDL_TRY(ce_wait(cw, r->side));
  ce_mark("L" + std::to_string(l) + " peers' RS in (side)", r->side);

  size_t lo;
  const size_t n8 = shard8(l, me, &lo);
  ShardUpdateArgs u;
  const size_t slot8 = shard_total8(me), seg8 = seg_off8(me, l);
  for (size_t k = 0; k < ring_.size(); ++k) {
    if (host_index(ring_[k]) == me)
      u.src[u.n_src++] = workers_[ring_[k]]->grad + base + lo * 8;
    else
      u.src[u.n_src++] = r->recv + (static_cast<size_t>(recv_slot(me, k)) * slot8 + seg8) * 8;
  }
  u.master = r->master + base + lo * 8;
  u.mom = r->mom ? r->mom + base + lo * 8 : nullptr;
  u.W = r->W + base + lo * 8;
  u.n8 = n8;
  const double eta_t = cfg_.eta / (1.0 + cfg_.decay * static_cast<double>(t_));
  u.scale = static_cast<float>(eta_t / static_cast<double>(step_count_));
  u.inv_count = static_cast<float>(1.0 / static_cast<double>(step_count_));
  u.eta = static_cast<float>(eta_t);
  u.mu = static_cast<float>(cfg_.momentum);
  static int ublocks = -1;  // few CTAs: the update shares the SMs with the backward GEMMs
  if (ublocks < 0) {
    const char* e = getenv("EDL_CE_UPDATE_BLOCKS");
    ublocks = e ? atoi(e) : 148;
  }
  u.blocks = ublocks;
  EDL_TRY(shard_update(u, r->side));
  ce_mark("L" + std::to_string(l) + " update done (side)", r->side);
  EDL_CUDA_TRY(cudaEventRecord(r->ev_upd[l], r->side));
  EDL_CUDA_TRY(cudaStreamWaitEvent(r->side3, r->ev_upd[l], 0));
  for (int p = 0; p < n_rep; ++p) {
    if (p == me || n8 == 0) continue;
    EDL_CUDA_TRY(cudaMemcpyAsync(peers_[p].W + base + lo * 8, r->W + base + lo * 8, n8 * 16,
                                 cudaMemcpyDeviceToDevice, r->side3));
  }
  sg.kind = 1;
  EDL_TRY(ce_signal(sg, r->side3));
  ce_mark("L" + std::to_string(l) + " AG pushed (side3)", r->side3);
  ++r->layer_colls;
  launches_ += 4;
  return EDL_OK;
}

void Job::own_segments(int me, int n_rep, CollArgs* a) const {
  a->n_seg = 0;
  for (int l = 0; l < L_; ++l) {
    size_t lo, hi;
    shard_range(static_cast<size_t>(in_[l]) * out_[l] / 8, n_rep, me, &lo, &hi);
    if (hi <= lo) continue;
    a->seg_lo8[a->n_seg] = off_[l] / 8 + lo;
    a->seg_hi8[a->n_seg] = off_[l] / 8 + hi;
    ++a->n_seg;
  }
}

// Launches the layer updates not issued yet (a worker with an empty batch ends the step
// early) and makes the replica's main stream wait for the side stream.
int Job::finish_layer_colls(Replica* r) {
  const int want = fused_update_ ? L_ - 1 : L_;
  while (r->layer_colls < want) {
    const int l = L_ - 1 - r->layer_colls;  // layers go L-1 .. 0 (fused: .. 1)
    EDL_TRY(launch_layer_coll(r, l));
  }
  if (overlap_mode_ == 5 || overlap_mode_ == 6) {  // the push follows once every copy landed
    cudaStream_t cs[3] = {r->side2, r->side3, r->side};
    const int n_st = static_cast<int>(peers_.size()) - 1 < 3 ? static_cast<int>(peers_.size()) - 1 : 3;
    for (int i = 0; i < n_st; ++i) {
      EDL_CUDA_TRY(cudaEventRecord(r->ev_rs[i], cs[i]));  // reuse: per-layer events idle here
      EDL_CUDA_TRY(cudaStreamWaitEvent(r->stream, r->ev_rs[i], 0));
    }
    return EDL_OK;
  }
  if (overlap_mode_ == 2) {  // every peer's weights of every layer have landed here
    EDL_CUDA_TRY(cudaEventRecord(r->ev_rs[0], r->side3));  // reuse: side3 drained
    EDL_CUDA_TRY(cudaStreamWaitEvent(r->side, r->ev_rs[0], 0));
    CeWait cw;
    cw.flags = r->flags;
    cw.n_rep = static_cast<int>(peers_.size());
    cw.me = rep_index(r);
    cw.kind = 1;
    cw.l_lo = 0;
    cw.l_hi = L_;
    cw.epoch = ce_epoch_;
    EDL_TRY(ce_wait(cw, r->side));
    ce_mark("all AG in (side)", r->side);
    launches_ += 1;
  }
  EDL_CUDA_TRY(cudaEventRecord(r->ev_side, r->side));
  EDL_CUDA_TRY(cudaStreamWaitEvent(r->stream, r->ev_side, 0));
  return EDL_OK;
}

int Job::run_worker_linear(Worker* w, int slot) {
  Replica* r = w->rep;
  DeviceGuard dg(r->device);
  const int64_t rows = static_cast<int64_t>(w->plan.size());
  EDL_CUDA_TRY(cudaEventRecord(w->ev_w0[slot], r->stream));
  cudaEvent_t m = (profile_ && r == primary()) ? mark_begin(r->stream) : nullptr;
  if (rows > 0) {
    EdlRun* host = w->runs_host + static_cast<size_t>(slot) * w->runs_cap;
    EDL_CUDA_TRY(cudaMemcpyAsync(w->runs_dev, host, sizeof(EdlRun) * w->n_runs,
                                 cudaMemcpyHostToDevice, r->stream));
    EDL_TRY(gather(r->ds, w->runs_dev, w->n_runs, rows, r->xb, r->yb, r->stream));
    launches_ += 1;
  }
  m = mark(slot, 0, m, r->stream);
  EDL_TRY(linear_local_gradient(cfg_.model, r->w, r->xb, r->yb, rows, cfg_.data.dim, w->g, r->ws,
                                r->stream));
  m = mark(slot, 3, m, r->stream);
  EDL_TRY(linear_batch_loss_from_z(cfg_.model, r->ws + rows, r->yb, rows, w->loss, r->stream));
  m = mark(slot, 2, m, r->stream);
  (void)m;
  if (w->delay_us > 0) {
    EDL_TRY(spin(static_cast<uint64_t>(w->delay_us * 1e3), r->stream));
    launches_ += 1;
  }
  EDL_CUDA_TRY(cudaEventRecord(w->ev_w1[slot], r->stream));
  launches_ += (rows > 0 ? 2 : 1) + (rows > 0 ? 2 : 1);
  return EDL_OK;
}

// Protocol step 3.
int Job::reduce_and_update(uint64_t count, uint64_t t, int slot, const double** loss_src) {
  const double eta_t = cfg_.eta / (1.0 + cfg_.decay * static_cast<double>(t));  // trainer.hpp:27
  const int n_rep = static_cast<int>(peers_.size());
  *loss_src = primary()->loss_sum;
  if (mlp_ && fused_update_ && n_rep == 1 && ring_.size() == 1) {
    // one ring member on one GPU: the update ran inside the wgrad GEMMs and the ordered loss
    // sum over one member is its own loss -- nothing to launch (read that loss directly)
    *loss_src = workers_[ring_[0]]->loss + (t & 1);
    return EDL_OK;
  }
  if (n_rep > 1 && !peers_ready())
    return fail(EDL_EINVAL, "job: peer handles missing (call edl_job_import for every peer)");
  if (ring_.size() > static_cast<size_t>(kCollMaxSources))
    return fail(EDL_EINVAL, "job: ring larger than the collective supports");
  Replica* prim = primary();
  cudaEvent_t m = ag_defer_ && !ag_ce_ ? nullptr : mark_begin(prim->stream);
  const uint32_t epoch = ++coll_epoch_;  // one collective per mini-batch, same on every GPU
  for (int me = 0; me < n_rep; ++me) {
    if (!peers_[me].local) continue;  // launched by its own process
    Replica* r = peers_[me].rep;
    DeviceGuard dg(r->device);
    if (mlp_) {
      // one fused kernel per replica: [barrier] ordered loss sum, reduce-scatter of the bf16
      // gradients of every ring member, sharded SGD on the fp32 master, all-gather of the
      // bf16 weights into every replica [barrier]
      CollArgs a;
      for (const auto& id : ring_) {
        a.grads[a.n_src++] = workers_[id]->grad;
        a.losses[a.n_loss++] = workers_[id]->loss + (t & 1);  // run_worker_mlp's slot
      }
      for (const auto& p : peers_) {
        a.flags[a.n_dst] = p.flags;
        a.w_dst[a.n_dst++] = p.W;
      }
      a.me = me;
      a.n_rep = n_rep;
      a.epoch = epoch;
      own_segments(me, n_rep, &a);
      a.master = r->master;
      a.mom = r->mom;
      a.scale = count ? static_cast<float>(eta_t / static_cast<double>(count)) : 0.f;
      a.inv_count = count ? static_cast<float>(1.0 / static_cast<double>(count)) : 0.f;
      a.eta = static_cast<float>(eta_t);
      a.mu = static_cast<float>(cfg_.momentum);
      a.update = (count > 0 && !fused_update_ &&
                  (!overlap_ || overlap_mode_ == 3 || overlap_mode_ >= 5)) ? 1 : 0;
      a.loss_out = r->loss_sum;
      if (a.update && (overlap_mode_ == 3 || overlap_mode_ >= 5 || push_eligible())) {
        a.push = 1;  // every NVLink byte a store
        // slices already pushed by the GEMMs (3) or the copy engines (5)
        a.skip_push = overlap_mode_ == 3 || overlap_mode_ >= 5 ? 1 : 0;
        a.n_layer = L_;
        for (int l = 0; l < L_; ++l) {
          a.lay_off8[l] = off_[l] / 8;
          a.lay_len8[l] = static_cast<size_t>(in_[l]) * out_[l] / 8;
        }
        for (size_t k = 0; k < ring_.size(); ++k) a.src_rep[k] = host_index(ring_[k]);
        for (int p = 0; p < n_rep; ++p) a.recv_peer[p] = peers_[p].recv;
        a.recv_me = r->recv;
        for (const auto& id : ring_)
          if (host_index(id) == me) a.own_grad = workers_[id]->grad;
      }
      if (ag_ce_ && a.push && a.skip_push) {
        // copy-engine all-gather: the push collective (full grid, after the backward) sums
        // and updates this GPU's shard and writes its bf16 weights locally only; the copy
        // engines then store the shard into every peer layer by layer (forward order, one
        // stream per peer offset so several copy engines run), each layer followed by a flag
        // store that releases the peer's next forward GEMM of that layer.  The copies use
        // no SMs, so they run under the next mini-batch's gather and forward.
        a.w_dst[0] = r->W;
        a.n_dst = 1;
        EDL_TRY(allreduce_sgd(a, r->stream));
        EDL_TRY(launch_ag_ce(r, me, epoch));
      } else if (ag_defer_ && a.push && a.skip_push) {
        // deferred all-gather: the push collective runs on the side stream after this
        // mini-batch's backward, concurrently with the next mini-batch's gather / forward;
        // per-layer flags release the forward GEMMs layer by layer.  A small grid (one CTA
        // per SM) co-resides with the forward GEMMs instead of blocking their CTAs.
        static int ag_blocks = -1;
        if (ag_blocks < 0) {
          const char* e = getenv("EDL_AG_BLOCKS");
          ag_blocks = e ? atoi(e) : 148;
        }
        a.blocks = ag_blocks;
        a.ag_signal = 1;
        EDL_CUDA_TRY(cudaEventRecord(r->ev_bwd, r->stream));
        EDL_CUDA_TRY(cudaStreamWaitEvent(r->side, r->ev_bwd, 0));
        cudaEvent_t ms = (r == prim) ? mark_begin(r->side) : nullptr;
        EDL_TRY(allreduce_sgd(a, r->side));
        if (ms) mark(slot, 4, ms, r->side);
        EDL_CUDA_TRY(cudaEventRecord(r->ev_push, r->side));
        r->ag_wait_epoch = epoch;
        r->side_pending = true;
      } else {
        EDL_TRY(allreduce_sgd(a, r->stream));
      }
    } else {
      LinearCollArgs a;
      for (const auto& id : ring_) {
        a.g[a.n_src] = workers_[id]->g;
        a.losses[a.n_src] = workers_[id]->loss;
        ++a.n_src;
      }
      for (size_t i = 0; i < peers_.size(); ++i) a.flags[i] = peers_[i].flags;
      a.me = me;
      a.n_rep = n_rep;
      a.epoch = epoch;
      a.dim = cfg_.data.dim;
      a.total = r->total;
      a.w = r->w;
      a.eta = eta_t;
      a.loss_out = r->loss_sum;
      EDL_TRY(linear_allreduce_sgd(a, r->stream));
    }
    launches_ += 1;
  }
  if (!ag_defer_ || ag_ce_) m = mark(slot, 4, m, prim->stream);
  (void)m;
  return EDL_OK;
}

int Job::launch_ag_ce(Replica* r, int me, uint32_t epoch) {
  const int n_rep = static_cast<int>(peers_.size());
  // each peer copy in `split` chunks (EDL_AG_CE_SPLIT, default 1), chunks and peers spread
  // over up to three streams so several copy engines run at once
  static int split = -1;
  if (split < 0) {
    const char* e = getenv("EDL_AG_CE_SPLIT");
    split = e && *e ? atoi(e) : 1;
    split = split < 1 ? 1 : (split > 3 ? 3 : split);
  }
  EDL_CUDA_TRY(cudaEventRecord(r->ev_bwd, r->stream));  // the shard update is done
  cudaStream_t ss[3] = {r->side, r->side2, r->side3};
  const int n_s = (n_rep - 1) * split < 3 ? (n_rep - 1) * split : 3;
  for (int s = 0; s < n_s; ++s) EDL_CUDA_TRY(cudaStreamWaitEvent(ss[s], r->ev_bwd, 0));
  for (int l = 0; l < L_; ++l) {
    size_t lo;
    const size_t n8 = shard8(l, me, &lo);
    const size_t at = off_[l] + lo * 8;
    AgSignal sg;
    sg.me = me;
    sg.layer = l;
    sg.epoch = epoch;
    sg.flags[sg.n_dst++] = r->flags;  // my own shard is final in my W
    int k = 0;
    for (int j = 1; j < n_rep; ++j) {
      const int p = (me + j) % n_rep;  // rotated: every GPU feeds a different peer at once
      for (int c = 0; c < split; ++c, ++k) {
        const size_t c0 = n8 * c / split, c1 = n8 * (c + 1) / split;
        if (c1 > c0)
          EDL_CUDA_TRY(cudaMemcpyAsync(peers_[p].W + at + c0 * 8, r->W + at + c0 * 8,
                                       (c1 - c0) * 16, cudaMemcpyDeviceToDevice, ss[k % 3]));
      }
      sg.flags[sg.n_dst++] = peers_[p].flags;
    }
    // the flag stores follow every copy of the layer (stream memory ops, no SM)
    cudaEvent_t evl[2] = {r->ev_rs[l], r->ev_upd[l]};
    for (int s = 1; s < n_s; ++s) {
      EDL_CUDA_TRY(cudaEventRecord(evl[s - 1], ss[s]));
      EDL_CUDA_TRY(cudaStreamWaitEvent(r->side, evl[s - 1], 0));
    }
    EDL_TRY(ag_signal(sg, r->side));
  }
  // `side` ends after every copy (join_side / the next routed wgrad wait on ev_push)
  EDL_CUDA_TRY(cudaEventRecord(r->ev_push, r->side));
  r->ag_wait_epoch = epoch;
  r->side_pending = true;
  return EDL_OK;
}

int Job::join_side() {
  for (auto& [dev, r] : reps_) {
    if (!r->side_pending && !r->ag_wait_epoch) continue;
    DeviceGuard g(dev);
    if (r->side_pending) EDL_CUDA_TRY(cudaStreamWaitEvent(r->stream, r->ev_push, 0));
    r->side_pending = false;
    r->ag_wait_epoch = 0;
  }
  return EDL_OK;
}

// Newcomers start their forward GEMMs on per-layer weight flags (the sources ship the model
// layer by layer on the copy engines) when the job has one source replica; EDL_JOIN_PIPELINE
// =0 never (the newcomer waits on the host for the whole model), =2 with any number of
// sources (measured at 2->4: 0.91 vs 0.84 ms stall, so not the default there)
bool Job::join_pipeline_enabled(int n_src) const {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EDL_JOIN_PIPELINE");
    on = e ? atoi(e) : 1;
    // per-layer side-stream collectives (EDL_OVERLAP=1) take their epochs before the forward
    const char* o = getenv("EDL_OVERLAP");
    if (o && atoi(o) == 1) on = 0;
  }
  return on == 2 || (on == 1 && n_src == 1);
}

// Newcomer (one process per GPU): wait until every source has written its join words (after
// all of its copies), adopt the collective epoch, and rebuild the fp32 master of this
// replica's shard when the source shipped the low halves.
int Job::finish_join() {
  if (!join_.pending) return EDL_OK;
  Replica* r = reps_.begin()->second.get();
  DeviceGuard g(r->device);
  std::vector<uint32_t> words(kJoinFlagWords);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    EDL_CUDA_TRY(cudaMemcpy(words.data(), r->flags + kJoinFlagOffset,
                            sizeof(uint32_t) * kJoinFlagWords, cudaMemcpyDeviceToHost));
    bool all = true;
    for (int j = 0; j < join_.n_src; ++j) all = all && words[2 * j + 1] == join_.version;
    if (all) break;
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
      return fail(EDL_TIMEOUT, "scale_out: the model did not arrive from the ring");
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  coll_epoch_ = words[0];
  for (int j = 1; j < join_.n_src; ++j)
    if (words[2 * j] != coll_epoch_)
      return fail(EDL_VERSION_MISMATCH, "scale_out: sources disagree on the collective epoch");
  if (mlp_ && join_.n_src == 1 && words[2 * kCollMaxReplicas] == 1u) {
    // the source shipped the weights and the low halves of my shard: rebuild its fp32
    r->lo_live = true;  // (W, lo) is this shard's master until the join below
    EDL_TRY(join_own_shard(r, join_.me_new, join_.n_new));
  }
  join_.pending = false;
  return EDL_OK;
}

// Scale-out across processes from a single replica that holds the split master (the fused
// single-replica update ran up to the switch): every process decides the same from the
// configuration and the ring, so sources and newcomers agree without a message.
bool Job::lo_reshard(const Event& ev) const {
  static int env = -1;  // EDL_LO_RESHARD=0: ship the fp32 master as before
  if (env < 0) {
    const char* e = getenv("EDL_LO_RESHARD");
    env = e ? atoi(e) != 0 : 1;
  }
  if (!env || !mlp_ || dry_ || !ev.out || cfg_.momentum != 0.0 || cfg_.appx_recovery ||
      !split_master_enabled() || peers_.size() != 1)
    return false;
  bool multi = joining_;
  for (const auto& w : ev.prepared) multi = multi || (w && w->remote);
  return multi;
}

// fp32 master of replica r's shard (me of n) from its weights and low halves
int Job::join_own_shard(Replica* r, int me, int n) {
  if (!r->lo_live) return EDL_OK;
  if (!r->mlo) return fail(EDL_EINVAL, "split master: no low-half buffer");
  DeviceGuard g(r->device);
  CollArgs a;
  own_segments(me, n, &a);
  for (int k = 0; k < a.n_seg; ++k) {
    const size_t at = a.seg_lo8[k] * 8, len = (a.seg_hi8[k] - a.seg_lo8[k]) * 8;
    EDL_TRY(master_join(r->W + at, r->mlo + at, r->master + at, len, r->stream));
  }
  r->lo_live = false;
  return EDL_OK;
}

int Job::master_sync() {
  for (auto& [dev, r] : reps_) {
    if (!r->lo_live) continue;
    DeviceGuard g(dev);
    EDL_TRY(master_join(r->W, r->mlo, r->master, P_, r->stream));
    r->lo_live = false;
  }
  return EDL_OK;
}

int Job::run_sgd_plan(const GemmPlan& p, Replica* r) {
  if (!p.lo) return gemm_plan_run(p, r->stream, step_scale_);
  if (!p.lo_master) return fail(EDL_EINVAL, "split master: plan without the fp32 master map");
  const bool in_split = r->lo_live, out_split = sgd_out_split_ && split_step_;
  if (in_split && out_split) return gemm_plan_run(p, r->stream, step_scale_);
  GemmPlan q = p;
  if (!in_split && !out_split) {  // plain fp32 master kernel
    q.tm = p.pm.m[0];
    q.lo = 0;
  } else {
    q.lo = in_split ? 2 : 3;
  }
  return gemm_plan_run(q, r->stream, step_scale_);
}

int Job::master_current() {
  EDL_TRY(join_side());
  return master_sync();
}

// All-gather of the sharded fp32 master among the local replicas, enqueued on their streams
// (no host sync): before a topology switch changes the sharding, and for checkpoints.
int Job::consolidate_master() {
  EDL_TRY(master_current());  // the deferred push collective / split master
  if (!mlp_ || peers_.size() < 2 || dry_) return EDL_OK;
  const uint32_t epoch = ++coll_epoch_;
  const int n_rep = static_cast<int>(peers_.size());
  for (int me = 0; me < n_rep; ++me) {
    if (!peers_[me].local) continue;
    Replica* r = peers_[me].rep;
    DeviceGuard dg(r->device);
    CollArgs a;
    for (const auto& p : peers_) {
      a.m_dst[a.n_dst] = p.master;
      a.v_dst[a.n_dst] = p.mom;
      a.flags[a.n_dst] = p.flags;
      ++a.n_dst;
    }
    a.me = me;
    a.n_rep = n_rep;
    a.epoch = epoch;
    own_segments(me, n_rep, &a);
    a.master = r->master;
    a.mom = r->mom;  // each replica's momentum is current only on its own shard, too
    EDL_TRY(master_allgather(a, r->stream));
  }
  return EDL_OK;
}

// Model broadcast to a joining GPU: peer copies over NVLink from the
// lowest existing replica, ordered after the source's work so far; the source's next write
// to its model is its next collective, whose barrier waits for the newcomer.
int Job::broadcast_model(Replica* src, Replica* dst) {
  EDL_TRY(master_current());  // the deferred push collective / split master
  if (dry_ || src == dst) return EDL_OK;
  {
    DeviceGuard dg(src->device);
    EDL_CUDA_TRY(cudaEventRecord(src->ev_sync, src->stream));
  }
  DeviceGuard dg(dst->device);
  EDL_CUDA_TRY(cudaStreamWaitEvent(dst->stream, src->ev_sync, 0));
  if (mlp_) {
    EDL_CUDA_TRY(cudaMemcpyPeerAsync(dst->master, dst->device, src->master, src->device,
                                     sizeof(float) * P_, dst->stream));
    // the working weights are bf16(master) everywhere (init, fused SGD, push collective all
    // round to nearest): rebuild them locally instead of moving another 2 B/param over NVLink
    EDL_TRY(master_to_bf16(dst->master, dst->W, P_, dst->stream));
    if (src->mom && dst->mom)
      EDL_CUDA_TRY(cudaMemcpyPeerAsync(dst->mom, dst->device, src->mom, src->device,
                                       sizeof(float) * P_, dst->stream));
  } else {
    EDL_CUDA_TRY(cudaMemcpyPeerAsync(dst->w, dst->device, src->w, src->device,
                                     sizeof(double) * P_, dst->stream));
  }
  // the newcomer must not start computing before it holds the model (same stream: ordered)
  EDL_CUDA_TRY(cudaEventRecord(dst->ev_sync, dst->stream));
  return EDL_OK;
}

void Job::collect_completed() {
  while (!inflight_.empty()) {
    Pending& p = inflight_.front();
    Replica* r = p.rep;
    if (cudaEventQuery(r->ev_end[p.slot]) != cudaSuccess) break;
    EdlStepReport rep{};
    rep.t = p.t;
    rep.version = p.version;
    rep.ring_size = p.ring_size;
    rep.switched = p.switched;
    rep.count = p.count;
    rep.loss = p.count ? r->host_loss[p.slot] / static_cast<double>(p.count) : 0.0;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r->ev_begin[p.slot], r->ev_end[p.slot]);
    rep.step_ms = ms;
    rep.stall_ms = 0.0;
    if (p.have_prev) {
      float st = 0.f;
      if (cudaEventElapsedTime(&st, p.prev_end, r->ev_begin[p.slot]) == cudaSuccess)
        rep.stall_ms = st;
      cudaGetLastError();  // events of a previous primary on another GPU are not comparable
    }
    std::vector<cudaEvent_t> used;
    for (const Mark& mk : marks_[p.slot]) {
      float pm = 0.f;
      if (cudaEventElapsedTime(&pm, mk.a, mk.b) == cudaSuccess) phase_ms_[mk.phase] += pm;
      used.push_back(mk.a);
      used.push_back(mk.b);
    }
    std::sort(used.begin(), used.end());
    used.erase(std::unique(used.begin(), used.end()), used.end());
    ev_pool_.insert(ev_pool_.end(), used.begin(), used.end());
    if (!marks_[p.slot].empty()) ++phase_steps_;
    marks_[p.slot].clear();
    step_ms_.push_back(rep.step_ms);
    if (step_ms_.size() > 64) step_ms_.erase(step_ms_.begin());
    std::vector<std::pair<std::string, double>> wt;
    for (const auto& [id, w] : p.timed) {
      float wms = 0.f;
      DeviceGuard g(w->rep ? w->rep->device : r->device);
      if (w->ev_w0[p.slot] &&
          cudaEventElapsedTime(&wms, w->ev_w0[p.slot], w->ev_w1[p.slot]) == cudaSuccess)
        wt.emplace_back(id, static_cast<double>(wms));
      cudaGetLastError();
    }
    wtimes_.push_back(std::move(wt));
    if (wtimes_.size() > kTimeWindow) wtimes_.pop_front();
    last_ = rep;
    inflight_.pop_front();
  }
  for (auto it = graveyard_.begin(); it != graveyard_.end();) {
    if (cudaEventQuery(it->first) == cudaSuccess) {
      free_worker(it->second.get());
      cudaEventDestroy(it->first);
      it = graveyard_.erase(it);
    } else {
      ++it;
    }
  }
}

double Job::median_step_ms() const {
  if (step_ms_.empty()) return 0.0;
  std::vector<double> v = step_ms_;
  std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
  return v[v.size() / 2];
}

// Host-only mini-batch (EdlJobConfig::dry_run): the full control protocol — topology
// installs, lease draws, assignment log — without device work.  Lets every process of a
// multi-process job (or a CPU test) replay the leader's decisions.
int Job::step_dry(EdlStepReport* out) {
  bool switched = false;
  EDL_TRY(install_due(&switched));
  return step_host_only(switched, out);
}

// The lease protocol of one mini-batch without device work: dry-run jobs, and a newcomer
// process replaying the ring's draws until its switch (every process holds the leader's
// decisions, so the newcomer's lease state is the ring's when it joins).
int Job::step_host_only(bool switched, EdlStepReport* out) {
  if (cfg_.appx_recovery && dry_) EDL_TRY(take_pre_snapshot());
  uint64_t count = 0;
  for (size_t k = 0; k < ring_.size(); ++k) {
    Worker* w = workers_[ring_[k]].get();
    w->plan = draw(w, splits_[k]);
    count += w->plan.size();
  }
  if (cfg_.keep_log) {
    for (const auto& id : ring_) {
      LogRec rec;
      rec.t = t_;
      rec.worker = id;
      rec.samples = workers_[id]->plan;
      log_.push_back(std::move(rec));
    }
  }
  EdlStepReport rep{};
  rep.t = t_;
  rep.version = version_;
  rep.ring_size = static_cast<int32_t>(ring_.size());
  rep.switched = switched ? 1 : 0;
  rep.count = count;
  rep.loss = NAN;
  last_ = rep;
  if (out) *out = rep;
  ++t_;
  ++launched_;
  return EDL_OK;
}

namespace {
// EDL_HOST_TRACE=1: host time of the step's phases on stderr (switch-stall diagnostics)
struct HostTrace {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  std::string line;
  HostTrace() {
    static int env = -1;
    if (env < 0) {
      const char* e = getenv("EDL_HOST_TRACE");
      env = e ? atoi(e) : 0;
    }
    on = env != 0;
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    line += std::string(" ") + what + "=" +
            std::to_string(std::chrono::duration<double, std::micro>(now - last).count()).substr(0, 6);
    last = now;
  }
};
}  // namespace

int Job::step(EdlStepReport* out) {
  HostTrace ht;
  if (dry_) return step_dry(out);
  const int slot = static_cast<int>(launched_ % kSlots);
  // pinned staging for this slot is free once the mini-batch that used it kSlots ago is done
  if (slot_end_[slot]) EDL_CUDA_TRY(cudaEventSynchronize(slot_end_[slot]));
  // a loss read on the side stream two mini-batches ago (same parity slot of the worker's
  // loss) must be done before this mini-batch's gather zeroes that slot
  for (auto& [dev, rr] : reps_) {
    if (!rr->loss_on_side) continue;
    const int back = static_cast<int>((launched_ + kSlots - 2) % kSlots);
    if (launched_ >= 2 && rr->ev_end[back]) {
      DeviceGuard dg(dev);
      EDL_CUDA_TRY(cudaStreamWaitEvent(rr->stream, rr->ev_end[back], 0));
    }
  }
  collect_completed();

  if (exited_) return fail(EDL_EINVAL, "job: this process's workers have left the ring");
  bool switched = false;
  ht.mark("pre");
  // the previous switch's model copies to newcomers (side3) before this mini-batch
  for (auto& [dev, rr] : reps_) {
    if (!rr->copies_pending) continue;
    DeviceGuard dg(dev);
    EDL_CUDA_TRY(cudaEventRecord(rr->ev_sync, rr->side3));
    EDL_CUDA_TRY(cudaStreamWaitEvent(rr->stream, rr->ev_sync, 0));
    rr->copies_pending = false;
  }
  EDL_TRY(install_due(&switched));
  ht.mark("install");
  if (joining_) return step_host_only(switched, out);  // newcomer before its switch
  if (peers_.empty() || !peers_[rep_index()].local) {
    // one process per GPU, scale-in: this process's members left at this switch (their
    // leases were reclaimed above, the model was consolidated into the survivors):
    // notify_batch_end answers Exit; no device work from here on
    exited_ = true;
    if (out) {
      *out = EdlStepReport{};
      out->t = t_;
      out->version = version_;
      out->ring_size = static_cast<int32_t>(ring_.size());
      out->switched = 1;
      out->loss = NAN;
    }
    return EDL_OK;
  }
  Replica* prim = primary();
  DeviceGuard g(prim->device);
  if (cfg_.appx_recovery) EDL_TRY(take_pre_snapshot());

  // protocol step 2: lease draws in ring order, runs for the gather kernel
  uint64_t count = 0;
  for (size_t k = 0; k < ring_.size(); ++k) {
    Worker* w = workers_[ring_[k]].get();
    w->plan = draw(w, splits_[k]);  // every process replays every member's draw
    count += w->plan.size();
    if (w->remote) continue;
    EdlRun* host = w->runs_host + static_cast<size_t>(slot) * w->runs_cap;
    int n = 0;
    for (size_t i = 0; i < w->plan.size(); ++i) {
      const uint64_t id = w->plan[i].second;
      if (n > 0 && host[n - 1].first + host[n - 1].count == id)
        host[n - 1].count++;
      else
        host[n++] = EdlRun{id, 1};
    }
    w->n_runs = n;
  }

  // one ring member, plain SGD: no collective, the update runs inside the wgrad GEMMs
  fused_update_ = mlp_ && ring_.size() == 1 && cfg_.momentum == 0.0 && peers_.size() == 1;
  if (count > 0)
    step_scale_ = static_cast<float>(
        cfg_.eta / (1.0 + cfg_.decay * static_cast<double>(t_)) / static_cast<double>(count));

  static int overlap_env = -1;
  if (overlap_env < 0) {
    const char* e = getenv("EDL_OVERLAP");
    overlap_env = e && *e ? atoi(e) : -1;
  }
  // overlapped update (EDL_OVERLAP=1: side-stream collective kernels per layer, 2: copy-engine
  // transfers per layer).  Off by default: measured on B200 the
  // single fused collective after the backward is as fast at N=2 and faster at N=4, because
  // the overlapped transfers / update kernels slow the backward GEMMs they share the GPU with.
  overlap_mode_ = 0;
  if (mlp_ && count > 0 && overlap_env > 0) {
    overlap_mode_ = (peers_.size() > 1 || overlap_env == 1) ? overlap_env : 0;
    if (overlap_mode_ == 2 && !ce_fits()) overlap_mode_ = 1;
    if (overlap_mode_ == 3 && !rs_eligible()) overlap_mode_ = 0;
    if ((overlap_mode_ == 5 || overlap_mode_ == 6) && !rs_eligible()) overlap_mode_ = 0;
    if (overlap_mode_ == 6 && peers_.size() < 3) overlap_mode_ = 5;
  }
  // default with several GPUs (EDL_OVERLAP unset): the reduce-scatter rides in the wgrad GEMM
  // epilogues (TMA stores into the owners' recv over NVLink, under the backward) and one push
  // collective does the shard update + all-gather.  Measured on B200: 1.18M vs 1.10M
  // samples/s at N=2, 1.89M vs 1.77M at N=4 over the single push collective.
  // With two GPUs the reduce-scatter goes on the copy engines instead (mode 5: plain wgrad
  // GEMMs, per-layer peer copies under the rest of the backward): measured 1.33M vs 1.22M
  // samples/s at N=2.  From three GPUs on it is split (mode 6): the nearest peers' rows are
  // stored from the wgrad epilogues, the others' by the copy engines: N=4 2.01M vs 1.91M
  // (mode 3) and 1.82M (mode 5).
  if (mlp_ && count > 0 && overlap_env < 0 && peers_.size() > 1 && rs_eligible())
    overlap_mode_ = peers_.size() == 2 ? 5 : 6;
  if (overlap_mode_ == 4 && !xchg_eligible()) overlap_mode_ = rs_eligible() ? 3 : 0;
  overlap_ = overlap_mode_ != 0;
  // deferred all-gather (mode 3, EDL_AG_DEFER=1): the push collective of this mini-batch
  // overlaps the next mini-batch's forward.  Opt-in: measured on B200 the push kernel on a
  // grid small enough to co-reside with the forward GEMMs (148 CTAs) moves 290-360 GB/s
  // against ~530 GB/s with its full grid after the backward, and the forward is paced by it
  // (N=2 1.00M vs 1.12M samples/s, N=4 1.81M vs 1.83M)
  static int defer_env = -1;
  if (defer_env < 0) {
    const char* e = getenv("EDL_AG_DEFER");
    defer_env = e && *e ? atoi(e) : 0;
  }
  ag_defer_ = (overlap_mode_ == 3 || overlap_mode_ == 5) && defer_env != 0 && !cfg_.appx_recovery;
  // EDL_AG_DEFER=2: the all-gather half on the copy engines (launch_ag_ce).  Opt-in: measured
  // on B200 at N=2 the copies slow the forward GEMMs they overlap (GEMM time per mini-batch
  // 0.61 -> 0.74 ms) more than they save on the push kernel (0.26 -> 0.20 ms): 1.10M vs
  // 1.23M samples/s; splitting each copy over 2-3 copy engines was slower still
  ag_ce_ = ag_defer_ && defer_env == 2;
  if (!ag_defer_) EDL_TRY(join_side());
  // split master: the fused update keeps the master as (W, lo) from one fused mini-batch to
  // the next.  The launch before a switch writes the fp32 master instead (kLo = 2) and the
  // first fused launch after one reads it (kLo = 3), so a switch costs no conversion pass;
  // any other reader of the master joins it first (master_sync)
  split_step_ = fused_update_ && !overlap_;
  sgd_out_split_ = true;
  for (const auto& ev : events_)
    if (ev->switch_t >= 0 && ev->switch_t <= static_cast<int64_t>(t_) + 1 && !lo_reshard(*ev))
      sgd_out_split_ = false;
  if (!split_step_) EDL_TRY(master_sync());
  step_count_ = count;
  if (overlap_mode_ == 1) {  // same epochs on every process
    layer_epoch0_ = coll_epoch_ + 1;
    coll_epoch_ += static_cast<uint32_t>(fused_update_ ? L_ - 1 : L_);
  }
  if (overlap_mode_ == 2) ++ce_epoch_;  // same on every process
  static int trace_env = -1;
  if (trace_env < 0) {
    const char* e = getenv("EDL_CE_TRACE");
    trace_env = e ? atoi(e) : 0;
  }
  ce_trace_ = trace_env != 0 && overlap_mode_ == 2;
  if (ce_trace_) {  // print the previous step's timeline, start this one's
    if (!ce_marks_.empty()) {
      for (auto& [dev, rr] : reps_) {
        DeviceGuard g(dev);
        cudaStreamSynchronize(rr->stream);
      }
      for (size_t i = 0; i < ce_marks_.size(); ++i)
        fprintf(stderr, "[ce-trace rank %d] %8.1f us  %s\n", my_rank_,
                1e-3 * static_cast<double>(ce_stamps_[i] - ce_stamps_[0]), ce_marks_[i].c_str());
      ce_marks_.clear();
    }
    ce_mark("step begin (main)", prim->stream);
  }
  std::map<Replica*, Worker*> last_on;  // last local worker of each replica, in ring order
  for (const auto& id : ring_) {
    Worker* w = workers_[id].get();
    if (!w->remote) last_on[w->rep] = w;
  }
  for (auto& [rr, lw] : last_on) rr->layer_colls = 0;

  // device work: each worker on its replica's stream (GPUs run concurrently)
  EDL_CUDA_TRY(cudaEventRecord(prim->ev_begin[slot], prim->stream));
  for (const auto& id : ring_) {
    Worker* w = workers_[id].get();
    if (w->remote) continue;  // computed by its own process
    EDL_TRY(mlp_ ? run_worker_mlp(w, slot, last_on[w->rep] == w) : run_worker_linear(w, slot));
  }
  ht.mark("workers");
  EDL_TRY(finish_join());  // a newcomer's first mini-batch: its epoch and master shard
  const double* loss_src = nullptr;
  EDL_TRY(reduce_and_update(count, t_, slot, &loss_src));
  ht.mark("update");
  if (ht.on)
    fprintf(stderr, "[host rank %d t=%llu%s]%s\n", my_rank_, static_cast<unsigned long long>(t_),
            switched ? " switch" : "", ht.line.c_str());
  // with the deferred all-gather the mini-batch ends on the side streams (push collective);
  // the single-replica fused path reads its loss on the side stream too (EDL_LOSS_SIDE), so
  // the next mini-batch's first kernel follows this one's last without the copy between them
  static int loss_side = -1;
  if (loss_side < 0) {
    const char* e = getenv("EDL_LOSS_SIDE");
    loss_side = e ? atoi(e) : 1;
  }
  const bool side_tail = !ag_defer_ && loss_side && fused_update_ && mlp_ && prim->side;
  cudaStream_t tail = ag_defer_ ? prim->side : prim->stream;
  if (side_tail) {
    EDL_CUDA_TRY(cudaEventRecord(prim->ev_bwd, prim->stream));
    EDL_CUDA_TRY(cudaStreamWaitEvent(prim->side, prim->ev_bwd, 0));
    tail = prim->side;
    prim->loss_on_side = true;
  }
  EDL_CUDA_TRY(cudaMemcpyAsync(&prim->host_loss[slot], loss_src, sizeof(double),
                               cudaMemcpyDeviceToHost, tail));
  // the primary's end event covers every local replica's share of the mini-batch
  for (const auto& p : peers_) {
    if (!p.local || p.rep == prim) continue;
    DeviceGuard dg(p.rep->device);
    EDL_CUDA_TRY(cudaEventRecord(p.rep->ev_done[slot], ag_defer_ ? p.rep->side : p.rep->stream));
    EDL_CUDA_TRY(cudaStreamWaitEvent(tail, p.rep->ev_done[slot], 0));
  }
  EDL_CUDA_TRY(cudaEventRecord(prim->ev_end[slot], tail));
  slot_end_[slot] = prim->ev_end[slot];

  Pending p{prim, t_, slot, count, version_, static_cast<int>(ring_.size()), switched ? 1 : 0,
            last_end_ != nullptr, last_end_, {}};
  for (const auto& id : ring_) {
    Worker* w = workers_[id].get();
    if (!w->remote) p.timed.emplace_back(id, w);
  }
  inflight_.push_back(p);
  last_end_ = prim->ev_end[slot];

  if (cfg_.keep_log) {
    for (const auto& id : ring_) {
      LogRec rec;
      rec.t = t_;
      rec.worker = id;
      rec.samples = workers_[id]->plan;
      log_.push_back(std::move(rec));
    }
  }
  if (out) {
    *out = EdlStepReport{};
    out->t = t_;
    out->version = version_;
    out->ring_size = static_cast<int32_t>(ring_.size());
    out->switched = switched ? 1 : 0;
    out->count = count;
    out->loss = NAN;
  }
  ++t_;
  ++launched_;
  return EDL_OK;
}

int Job::sync(EdlStepReport* out) {
  if (dry_) {
    if (out) *out = last_;
    return EDL_OK;
  }
  // host wait for both streams; a deferred push stays "pending" (its flags and ev_push are
  // complete, so the next mini-batch's waits pass at once)
  for (auto& [dev, r] : reps_) {
    DeviceGuard g(dev);
    EDL_CUDA_TRY(cudaStreamSynchronize(r->stream));
    if (r->side) EDL_CUDA_TRY(cudaStreamSynchronize(r->side));
    if (r->side3) EDL_CUDA_TRY(cudaStreamSynchronize(r->side3));
  }
  collect_completed();
  if (out) *out = last_;
  return EDL_OK;
}

// scale_out / scale_in / scripted event.  explicit_switch < 0: scheduler-facing call,
// switch at t + max(1, ceil(T_a / T_b)) and Retry while another scaling op is pending.
// Scale-out across processes, at the switch (after consolidate_master: every live replica
// holds the whole model).  Sources (processes hosting a current member): copy slice j/n of
// the fp32 master and bf16 weights into every newcomer's replica over NVLink (peer copies
// on the job stream, so they precede this replica's next update), then store the collective
// epoch and the new topology version into the newcomer's join words.  Newcomer: wait on the
// host until every source's version word has arrived, adopt the epoch.  Everyone: the
// newcomers join the ring (ascending id) and the replica list.
int Job::add_copy(MultiCopyArgs* cp, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (!bytes) return EDL_OK;
  if (cp->n == kMaxCopySegs) {
    EDL_TRY(multi_copy(*cp, s));
    launches_ += 1;
    cp->n = 0;
  }
  cp->seg[cp->n++] = CopySeg{dst, src, bytes};
  return EDL_OK;
}

static bool same_replica(const PeerRep& a, const PeerRep& b) {
  if (a.local != b.local) return false;
  return a.local ? a.rep == b.rep : a.rank == b.rank;
}

// Bytes of old replica i's shard that lie in other replicas' new shards (old = replicas and
// sharding before a switch, after = after it; own_segments sharding per layer).
double Job::reshard_piece_bytes(const std::vector<PeerRep>& old, int i,
                                const std::vector<PeerRep>& after, bool mom, bool lo) const {
  const int n_old = static_cast<int>(old.size()), n_new = static_cast<int>(after.size());
  double b = 0;
  for (int l = 0; l < L_; ++l) {
    const size_t len8 = static_cast<size_t>(in_[l]) * out_[l] / 8;
    size_t olo, ohi;
    shard_range(len8, n_old, i, &olo, &ohi);
    for (int j = 0; j < n_new; ++j) {
      if (same_replica(after[j], old[i])) continue;
      size_t nlo, nhi;
      shard_range(len8, n_new, j, &nlo, &nhi);
      const size_t a8 = std::max(olo, nlo), b8 = std::min(ohi, nhi);
      if (b8 > a8) b += (b8 - a8) * 8.0 * (lo ? 2.0 : mom ? 8.0 : 4.0);
    }
  }
  return b;
}

// Re-sharding copies source i (replica `old[i]`, this replica `r`) issues at a switch.  The
// fp32 master (and momentum) is current on each replica only for its own shard; after the
// switch every replica -- old or new -- only needs its NEW shard, so the old owner of each
// piece of a new shard copies exactly that piece to its new owner.  The bf16 weights are
// current and identical on every old replica: each new replica (`fresh`) gets them from all
// sources, in shares that even out each source's NVLink egress with the master pieces it
// sends (every process computes the same split; source i ships the [wlo_i, whi_i) part, in
// units of 8 parameters, of the weights of all fresh replicas laid end to end).  A newcomer
// receives 2 B/param of weights plus 4 B (8 with momentum) per parameter of its shard,
// instead of the whole fp32 model after an all-gather ("broadcast the model").
int Job::add_reshard_copies(MultiCopyArgs* cp, const std::vector<PeerRep>& old, int i,
                            const std::vector<PeerRep>& after, const std::vector<PeerRep>& fresh,
                            Replica* r, bool lo, bool skip_w) {
  const int n_old = static_cast<int>(old.size());
  const bool mom = r->mom != nullptr;
  if (lo && (mom || !r->mlo || !r->lo_live))
    return fail(EDL_EINVAL, "reshard: low-half transfer needs this replica's split master");
  const size_t p8 = P_ / 8, jn = fresh.size();  // MLP layers: in % 8 == 0, so P_ % 8 == 0
  std::vector<double> mb(n_old);
  double sum_m = 0;
  for (int k = 0; k < n_old; ++k) sum_m += (mb[k] = reshard_piece_bytes(old, k, after, mom, lo));
  const double wtot = static_cast<double>(jn * p8) * 16.0;  // bytes of weights to ship
  std::vector<double> quota(n_old);
  double qsum = 0;
  for (int k = 0; k < n_old; ++k) qsum += (quota[k] = std::max(0.0, (wtot + sum_m) / n_old - mb[k]));
  size_t wlo = 0, whi = 0, acc = 0;
  for (int k = 0; k <= i; ++k) {
    const size_t share = qsum > 0 ? static_cast<size_t>(quota[k] / qsum * (jn * p8))
                                  : (jn * p8) / n_old;
    wlo = acc;
    acc = (k == n_old - 1) ? jn * p8 : std::min(jn * p8, acc + share);
    whi = acc;
  }
  if (skip_w) whi = wlo;  // the caller ships the weights itself (layer by layer)
  for (size_t pos = wlo; pos < whi;) {  // split the range at replica boundaries
    const size_t q = pos / p8, off = pos % p8, end = std::min(whi, (q + 1) * p8);
    EDL_TRY(add_copy(cp, fresh[q].W + off * 8, r->W + off * 8,
                     sizeof(__nv_bfloat16) * (end - pos) * 8, r->stream));
    pos = end;
  }
  const int n_new = static_cast<int>(after.size());
  for (int l = 0; l < L_; ++l) {
    const size_t len8 = static_cast<size_t>(in_[l]) * out_[l] / 8, base = off_[l];
    size_t olo, ohi;  // my old shard of layer l
    shard_range(len8, n_old, i, &olo, &ohi);
    for (int j = 0; j < n_new; ++j) {
      if (same_replica(after[j], old[i])) continue;  // my new shard: already mine
      size_t nlo, nhi;
      shard_range(len8, n_new, j, &nlo, &nhi);
      const size_t a8 = std::max(olo, nlo), b8 = std::min(ohi, nhi);
      if (b8 <= a8) continue;
      const size_t at = base + a8 * 8, n = (b8 - a8) * 8;
      if (lo) {  // the new owner rebuilds its fp32 shard from the weights and these halves
        if (!after[j].mlo) return fail(EDL_EINVAL, "reshard: a newcomer has no split-master buffer");
        EDL_TRY(add_copy(cp, after[j].mlo + at, r->mlo + at, sizeof(uint16_t) * n, r->stream));
        continue;
      }
      EDL_TRY(add_copy(cp, after[j].master + at, r->master + at, sizeof(float) * n, r->stream));
      if (mom) {
        if (!after[j].mom) return fail(EDL_EINVAL, "reshard: a replica has no momentum buffer");
        EDL_TRY(add_copy(cp, after[j].mom + at, r->mom + at, sizeof(float) * n, r->stream));
      }
    }
  }
  return EDL_OK;
}

// One process, several GPUs: after the membership change every replica of the new ring
// (old ones re-sharded, `fresh` ones joining) gets exactly what it needs from the old
// replicas (add_reshard_copies), each source's copies in one SM copy kernel on its stream,
// and every new-ring replica's stream waits for all of them.
int Job::reshard_local(const std::vector<PeerRep>& old, const std::vector<Replica*>& fresh) {
  std::vector<PeerRep> fr;
  for (const auto& p : peers_)
    if (std::find(fresh.begin(), fresh.end(), p.rep) != fresh.end()) fr.push_back(p);
  bool same = old.size() == peers_.size() && fr.empty();
  for (size_t i = 0; same && i < old.size(); ++i) same = old[i].rep == peers_[i].rep;
  if (same) return EDL_OK;  // the sharding did not change
  for (size_t i = 0; i < old.size(); ++i) {
    Replica* r = old[i].rep;
    DeviceGuard g(r->device);
    MultiCopyArgs cp;
    EDL_TRY(add_reshard_copies(&cp, old, static_cast<int>(i), peers_, fr, r, false, false));
    EDL_TRY(multi_copy(cp, r->stream));
    launches_ += 1;
    EDL_CUDA_TRY(cudaEventRecord(r->ev_sync, r->stream));
  }
  for (const auto& p : peers_) {
    DeviceGuard g(p.rep->device);
    for (const auto& o : old)
      if (o.rep != p.rep) EDL_CUDA_TRY(cudaStreamWaitEvent(p.rep->stream, o.rep->ev_sync, 0));
  }
  return EDL_OK;
}

// Scale-in across processes: the survivors' new shards from the old owners (leavers
// included, they are still in the ring at this boundary), then a barrier of every old
// replica so nobody updates before the pieces it needs have landed.
int Job::reshard_in_mp(const Event* ev) {
  std::vector<PeerRep> after;
  for (size_t i = 0; i < peers_.size(); ++i) {
    bool keeps = false;
    for (const auto& id : ring_)
      keeps = keeps || (std::find(ev->ids.begin(), ev->ids.end(), id) == ev->ids.end() &&
                        host_index(id) == static_cast<int>(i));
    if (keeps) after.push_back(peers_[i]);
  }
  const int me = rep_index();
  Replica* r = peers_[me].rep;
  DeviceGuard g(r->device);
  MultiCopyArgs cp;
  EDL_TRY(add_reshard_copies(&cp, peers_, me, after, {}, r, false, false));
  EDL_TRY(multi_copy(cp, r->stream));
  CollArgs a;
  for (const auto& p : peers_) a.flags[a.n_dst++] = p.flags;
  a.me = me;
  a.n_rep = static_cast<int>(peers_.size());
  a.epoch = ++coll_epoch_;
  EDL_TRY(replica_barrier(a, r->stream));
  launches_ += 2;
  return EDL_OK;
}

int Job::install_out_mp(Event* ev) {
  const uint64_t new_version = version_ + 1;
  std::vector<PeerRep> joiners;  // newcomer replicas (imported, or this process's own)
  for (const auto& w : ev->prepared)
    for (const auto& p : known_peers_) {
      const bool hosts = w->remote ? p.rank == w->host_rank && !p.local
                                   : p.local && p.rep == w->rep;
      if (!hosts) continue;
      bool dup = false;
      for (const auto& q : joiners) dup = dup || q.rank == p.rank;
      if (!dup) joiners.push_back(p);
    }
  for (const auto& w : ev->prepared)
    if (w->remote && !w->imported)
      return fail(EDL_EINVAL, "scale_out: newcomer " + w->id + " has not exported its handles");
  const int n_src = static_cast<int>(peers_.size());  // the current replicas, rank order
  if (joining_) {
    // this process's newcomer: its buffers are filled by the sources
    std::vector<PeerRep> after = peers_;
    for (const auto& q : joiners) after.push_back(q);
    std::sort(after.begin(), after.end(),
              [](const PeerRep& a, const PeerRep& b) { return a.rank < b.rank; });
    int me_new = 0;
    for (size_t k = 0; k < after.size(); ++k)
      if (after[k].rank == my_rank_) me_new = static_cast<int>(k);
    join_ = JoinWait{true, new_version, n_src, me_new, static_cast<int>(after.size())};
    // one source: the first mini-batch's forward GEMMs wait on the per-layer flags the
    // source writes after each layer's weights, and the join words are read only before its
    // collective (finish_join); with several sources read them now
    if (!(mlp_ && join_pipeline_enabled(n_src))) {
      EDL_TRY(finish_join());
    } else {
      // start once the sources have begun shipping (layer 0's flags): a newcomer that runs
      // ahead in host-only steps waits here, not inside its first GEMM
      Replica* r = reps_.begin()->second.get();
      DeviceGuard g(r->device);
      const auto t0 = std::chrono::steady_clock::now();
      for (;;) {
        std::vector<uint32_t> f(static_cast<size_t>(n_src));
        EDL_CUDA_TRY(cudaMemcpy(f.data(), ag_layer_flags(r->flags, 0), sizeof(uint32_t) * n_src,
                                cudaMemcpyDeviceToHost));
        bool all = true;
        for (uint32_t v : f) all = all && v >= static_cast<uint32_t>(new_version);
        if (all) break;
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
          return fail(EDL_TIMEOUT, "scale_out: the model did not start arriving from the ring");
        std::this_thread::sleep_for(std::chrono::microseconds(10));
      }
    }
    joining_ = false;
  } else {
    const int me = rep_index();
    Replica* r = peers_[me].rep;
    DeviceGuard g(r->device);
    bool ship_lo = false;
    cudaStream_t word_stream = r->stream;
    if (mlp_) {
      // Targeted re-sharding instead of consolidating the whole model: the bf16 weights are
      // current and identical on every replica, so each source ships slice me/n of them to
      // every newcomer; the fp32 master (and momentum) is only current on each replica's
      // own shard, and after the switch every replica -- old or new -- only needs its NEW
      // shard (own_segments under n_new), so the old owner of each piece of a new shard
      // copies exactly that piece to its new owner.  A newcomer receives 2 B/param of
      // weights plus 4 B (8 with momentum) per parameter of its shard instead of the whole
      // fp32 model, and no replica all-gathers ("broadcast the model").
      MultiCopyArgs cp;
      std::vector<PeerRep> after = peers_;  // the replicas after the switch, rank order
      for (const auto& q : joiners) after.push_back(q);
      std::sort(after.begin(), after.end(),
                [](const PeerRep& a, const PeerRep& b) { return a.rank < b.rank; });
      // (a split-master source that has not run a fused mini-batch yet holds the fp32 one)
      bool lo = lo_reshard(*ev) && r->lo_live && r->mlo;
      for (const auto& q : joiners) lo = lo && q.mlo;
      if (lo_reshard(*ev) && !lo) EDL_TRY(master_sync());
      ship_lo = lo;
      // one source: the weights go out layer by layer, each layer followed by its flag word
      // in every newcomer, whose forward GEMMs start on those flags (join_pipeline)
      const bool pipe = join_pipeline_enabled(n_src);
      EDL_TRY(add_reshard_copies(&cp, peers_, me, after, joiners, r, lo, pipe));
      // pipelined join (pipe): the newcomers' model goes out on the copy engines from a side
      // stream, layer by layer, so this replica's own switch mini-batch starts at once and
      // the newcomers' forward follows the weights as they land; nothing here waits for the
      // copies: the newcomers read the join words written after them before their
      // collective, and this replica's next model write is its push collective, past a
      // barrier they enter only after that.  Several sources: one SM copy kernel each ahead
      // of the mini-batch (measured faster than the copy engines when the newcomer waits for
      // the whole model: 1->2 stall 0.98 vs 1.08 ms; EDL_RESHARD_CE=1 selects them)
      static int ce_env = -1;
      if (ce_env < 0) {
        const char* e = getenv("EDL_RESHARD_CE");
        ce_env = e ? atoi(e) != 0 : 0;
      }
      if (ce_env || pipe) {
        EDL_CUDA_TRY(cudaEventRecord(r->ev_sync, r->stream));
        EDL_CUDA_TRY(cudaStreamWaitEvent(r->side3, r->ev_sync, 0));
        for (int l = 0; pipe && l < L_; ++l) {
          // source me of n_src ships its 1/n_src of every layer (16-byte aligned pieces)
          const size_t len8 = static_cast<size_t>(in_[l]) * out_[l] / 8;
          size_t lo8, hi8;
          shard_range(len8, n_src, me, &lo8, &hi8);
          const size_t at = off_[l] + lo8 * 8, bytes = (hi8 - lo8) * 16;
          for (const auto& q : joiners)
            if (bytes)
              EDL_CUDA_TRY(cudaMemcpyAsync(q.W + at, r->W + at, bytes, cudaMemcpyDeviceToDevice,
                                           r->side3));
          for (const auto& q : joiners)
            EDL_TRY(stream_write_u32(ag_layer_flags(q.flags, l) + me,
                                     static_cast<uint32_t>(new_version), r->side3));
        }
        for (int k = 0; k < cp.n; ++k)
          EDL_CUDA_TRY(cudaMemcpyAsync(cp.seg[k].dst, cp.seg[k].src, cp.seg[k].bytes,
                                       cudaMemcpyDeviceToDevice, r->side3));
        word_stream = r->side3;
        r->copies_pending = true;
      } else {
        EDL_TRY(multi_copy(cp, r->stream));  // SM stores over NVLink, one launch
        launches_ += 1;
      }
      if (lo) {  // my own new shard: fp32 master from (W, lo) here
        int me_new = 0;
        for (size_t k = 0; k < after.size(); ++k)
          if (after[k].rank == my_rank_) me_new = static_cast<int>(k);
        EDL_TRY(join_own_shard(r, me_new, static_cast<int>(after.size())));
        launches_ += 1;
      }
    }
    for (const auto& q : joiners) {
      EDL_TRY(stream_write_u32(q.flags + kJoinFlagOffset + 2 * kCollMaxReplicas + me,
                               ship_lo ? 1u : 0u, word_stream));
      EDL_TRY(stream_write_u32(q.flags + kJoinFlagOffset + 2 * me, coll_epoch_, word_stream));
      EDL_TRY(stream_write_u32(q.flags + kJoinFlagOffset + 2 * me + 1,
                               static_cast<uint32_t>(new_version), word_stream));
    }
  }
  std::vector<size_t> order(ev->ids.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return ev->ids[a] < ev->ids[b]; });
  for (size_t i : order) {
    const std::string& id = ev->ids[i];
    ring_.push_back(id);
    lm_->enroll(id);
    workers_[id] = std::move(ev->prepared[i]);
  }
  return EDL_OK;
}

int Job::scale(bool out, const std::vector<std::string>& ids, const std::vector<int>& devices,
               int64_t explicit_switch, int64_t* switch_t) {
  if (ids.empty()) return fail(EDL_EINVAL, "scale: empty worker set");
  if (explicit_switch < 0 && !events_.empty())
    return fail(EDL_RETRY, "a scaling operation is in progress");
  // one process per GPU (every process schedules the same event at an explicit switch
  // step): scale-in -- the leavers' processes exit the job at the switch; scale-out -- the
  // newcomers are hosted by their own processes (Job::create_joining, device -1 here)
  bool remote_new = false;
  for (int d : devices) remote_new = remote_new || d < 0;
  if (!dry_ && out && remote_new) {
    if (!mlp_) return fail(EDL_EINVAL, "scale_out across processes: MLP jobs only in this build");
    if (explicit_switch < 0)
      return fail(EDL_EINVAL, "scale_out across processes needs an explicit switch step");
    for (int d : devices)
      if (d >= 0) return fail(EDL_EINVAL, "scale_out across processes: newcomers are remote (-1)");
    auto ev = std::make_unique<Event>();
    ev->out = true;
    ev->ids = ids;
    ev->devices = devices;
    ev->switch_t = explicit_switch;
    for (const auto& id : ids) {
      if (find_worker(id)) return fail(EDL_EINVAL, "scale_out: worker already in the job");
      auto w = std::make_unique<Worker>();
      w->id = id;
      w->remote = true;  // its process exports the handles (import_handles before the switch)
      ev->prepared.push_back(std::move(w));
    }
    if (switch_t) *switch_t = ev->switch_t;
    auto pos = std::upper_bound(events_.begin(), events_.end(), ev->switch_t,
                                [](int64_t s, const std::unique_ptr<Event>& e) { return s < e->switch_t; });
    events_.insert(pos, std::move(ev));
    return EDL_OK;
  }
  auto ev = std::make_unique<Event>();
  ev->out = out;
  ev->ids = ids;
  ev->devices = devices;
  if (explicit_switch >= 0) {
    if (explicit_switch < static_cast<int64_t>(t_))
      return fail(EDL_EINVAL, "schedule: switch step already passed");
    // scripted event: the membership it meets at its switch is the ring after every event
    // installed before it (switch order, ties in scheduling order) -- it must not empty the
    // ring nor remove a non-member / add a member
    std::set<std::string> m(ring_.begin(), ring_.end());
    auto apply = [&](bool o, const std::vector<std::string>& v) -> int {
      for (const auto& id : v) {
        if (o && m.count(id)) return fail(EDL_EINVAL, "schedule: " + id + " already a member");
        if (!o && !m.count(id))
          return fail(EDL_UNKNOWN_WORKER, "schedule: " + id + " not a member at its switch");
        if (o) m.insert(id); else m.erase(id);
      }
      if (m.empty()) return fail(EDL_EINVAL, "schedule: no worker would remain");
      return EDL_OK;
    };
    bool placed = false;
    for (const auto& e : events_) {
      if (!placed && e->switch_t > explicit_switch) {
        EDL_TRY(apply(out, ids));
        placed = true;
      }
      if (e->switch_t != std::numeric_limits<int64_t>::max()) EDL_TRY(apply(e->out, e->ids));
    }
    if (!placed) EDL_TRY(apply(out, ids));
    ev->switch_t = explicit_switch;
  } else if (out) {
    ev->await_ready = true;  // switch_t chosen when the newcomers are Ready
    ev->switch_t = std::numeric_limits<int64_t>::max();
  } else {
    ev->switch_t = static_cast<int64_t>(t_) + switch_delay_steps();
  }
  if (out) {
    for (const auto& id : ids)
      if (workers_.count(id) && explicit_switch < 0)
        return fail(EDL_EINVAL, "scale_out: worker already in the job");
    if (devices.size() != ids.size()) return fail(EDL_EINVAL, "scale_out: one device per worker");
    for (int d : devices)
      if (d < 0) return fail(EDL_EINVAL, "scale_out: newcomers need a local GPU");
    // Execution-context preparation off the training thread (§4.2): a
    // new GPU gets its CUDA context, HBM dataset, model buffers, peer mappings and staging
    // here while the job keeps stepping; the switch only copies the model.
    ev->prepared.resize(ids.size());
    Event* raw = ev.get();
    // the job's replicas now (reps_ is only read here: install_due inserts into it on the
    // training thread while this preparation runs; GPUs that join through an earlier
    // pending event get their peer access at that install)
    std::map<int, Replica*> have;
    for (auto& [d, r] : reps_) have[d] = r.get();
    ev->prep = std::make_unique<std::thread>([this, raw, have]() {
      struct ReadyOnExit {
        std::atomic<bool>& f;
        ~ReadyOnExit() { f.store(true, std::memory_order_release); }
      } ready_on_exit{raw->ready};
      // new GPUs are prepared in parallel, one thread each (context, dataset, buffers)
      std::map<int, Replica*> made;
      std::vector<std::unique_ptr<Replica>> fresh;
      for (int d : raw->devices) {
        if (have.count(d) || made.count(d)) continue;
        fresh.push_back(std::make_unique<Replica>());
        fresh.back()->device = d;
        made[d] = fresh.back().get();
      }
      std::vector<int> rcs(fresh.size(), EDL_OK);
      std::vector<std::thread> builders;
      for (size_t k = 0; k < fresh.size(); ++k)
        builders.emplace_back([this, &fresh, &rcs, k]() { rcs[k] = build_replica(fresh[k].get()); });
      for (auto& b : builders) b.join();
      for (size_t k = 0; k < fresh.size(); ++k) {
        if (rcs[k] != EDL_OK) {
          raw->prep_rc = rcs[k];
          for (auto& f : fresh) raw->new_reps.push_back(std::move(f));
          return;
        }
        // peer mappings with the job's GPUs and with this event's other newcomers
        std::vector<int> others;
        for (const auto& [d, r] : have) others.push_back(d);
        for (size_t o = 0; o < k; ++o) others.push_back(fresh[o]->device);
        const int rc = enable_peer_devices(fresh[k]->device, others);
        if (rc != EDL_OK) raw->prep_rc = rc;
      }
      for (auto& f : fresh) raw->new_reps.push_back(std::move(f));
      if (raw->prep_rc != EDL_OK) return;
      for (size_t i = 0; i < raw->ids.size(); ++i) {
        const int d = raw->devices[i];
        auto it = have.find(d);
        Replica* r = it != have.end() ? it->second : made[d];
        auto w = std::make_unique<Worker>();
        w->id = raw->ids[i];
        const int rc = build_worker(w.get(), r);
        if (rc != EDL_OK) {
          raw->prep_rc = rc;
          return;
        }
        raw->prepared[i] = std::move(w);
      }
    });
  } else {
    // Scripted events are validated when they are installed (the ring may change before).
    if (explicit_switch < 0) {
      size_t leaving = 0;
      for (const auto& id : ids) {
        if (!workers_.count(id)) return fail(EDL_UNKNOWN_WORKER, "scale_in: unknown worker " + id);
        ++leaving;
      }
      if (leaving >= ring_.size()) return fail(EDL_EINVAL, "scale_in: no worker would remain");
    }
  }
  if (switch_t) *switch_t = ev->await_ready ? -1 : ev->switch_t;
  auto pos = std::upper_bound(events_.begin(), events_.end(), ev->switch_t,
                              [](int64_t s, const std::unique_ptr<Event>& e) { return s < e->switch_t; });
  events_.insert(pos, std::move(ev));
  return EDL_OK;
}

int Job::params(const std::string& worker, void* host, size_t bytes) {
  EDL_TRY(master_current());  // the deferred push collective / split master
  auto it = workers_.find(worker);
  if (it == workers_.end()) return fail(EDL_UNKNOWN_WORKER, "params: unknown worker " + worker);
  if (it->second->remote) return fail(EDL_EINVAL, "params: worker hosted by another process");
  Replica* r = it->second->rep;
  bool all_local = true;
  for (const auto& p : peers_) all_local = all_local && p.local;
  if (all_local) EDL_TRY(consolidate_master());  // multi-process: call edl_job_gather_master
  for (auto& [dev, rr] : reps_) {
    DeviceGuard g(dev);
    EDL_CUDA_TRY(cudaStreamSynchronize(rr->stream));
  }
  DeviceGuard g(r->device);
  const size_t need = mlp_ ? sizeof(float) * P_ : sizeof(double) * P_;
  if (bytes < need) return fail(EDL_EINVAL, "params: buffer too small");
  EDL_CUDA_TRY(cudaMemcpy(host, mlp_ ? static_cast<void*>(r->master) : static_cast<void*>(r->w),
                          need, cudaMemcpyDeviceToHost));
  return EDL_OK;
}

// Checkpoint restore (stop-resume baseline, recovery): every replica takes the parameters;
// MLP replicas re-derive their bf16 working weights from the fp32 master.
int Job::set_params(const void* host, size_t bytes) {
  EDL_TRY(master_current());  // the deferred push collective / split master
  const size_t need = mlp_ ? sizeof(float) * P_ : sizeof(double) * P_;
  if (bytes < need) return fail(EDL_EINVAL, "set_params: buffer too small");
  for (auto& [dev, r] : reps_) {
    DeviceGuard g(dev);
    EDL_CUDA_TRY(cudaStreamSynchronize(r->stream));
    if (mlp_) {
      EDL_CUDA_TRY(cudaMemcpy(r->master, host, need, cudaMemcpyHostToDevice));
      EDL_TRY(master_to_bf16(r->master, r->W, P_, r->stream));
      EDL_CUDA_TRY(cudaStreamSynchronize(r->stream));
    } else {
      EDL_CUDA_TRY(cudaMemcpy(r->w, host, need, cudaMemcpyHostToDevice));
    }
  }
  return EDL_OK;
}

std::string Job::log_text() const {  // write_log_file, trainer.cpp:79-100
  std::ostringstream o;
  for (const auto& r : log_) {
    if (r.kind == LogRec::Batch) {
      o << "batch " << r.t << " " << r.worker << " " << r.samples.size();
      for (const auto& [e, id] : r.samples) o << " " << e << ":" << id;
      o << "\n";
    } else if (r.kind == LogRec::Topo) {
      o << "topo " << r.t << " " << r.version << " " << r.ring.size();
      for (const auto& w : r.ring) o << " " << w;
      o << "\n";
    } else {
      o << "restore " << r.t << "\n";
    }
  }
  return o.str();
}

std::string Job::ring_csv() const {
  std::string s;
  for (size_t i = 0; i < ring_.size(); ++i) s += (i ? "," : "") + ring_[i];
  return s;
}

// ------------------------------------------------------------------ multi-process plumbing
// One process per GPU: every process hosts its own replica + worker(s) and replays the
// lease protocol for the whole ring; the per-step exchange goes through CUDA IPC mappings
// of the peers' gradient / weight / flag / loss buffers (NVLink peer memory), so no NCCL
// call sits on the data path.

int Job::rep_index() const {
  for (size_t i = 0; i < peers_.size(); ++i)
    if (peers_[i].local) return static_cast<int>(i);
  return 0;
}

int Job::rep_index(const Replica* r) const {
  for (size_t i = 0; i < peers_.size(); ++i)
    if (peers_[i].rep == r) return static_cast<int>(i);
  return -1;
}

bool Job::peers_ready() const {
  for (const auto& [id, w] : workers_)
    if (w->remote && !w->imported) return false;
  return true;
}

namespace {
constexpr uint32_t kBlobMagic = 0x48444c45;  // "EDLH"
struct BlobW {
  std::vector<uint8_t> b;
  bool dry = false;  // dry-run jobs publish the layout without device handles
  template <class T>
  void pod(const T& v) {
    const auto* p = reinterpret_cast<const uint8_t*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  void text(const std::string& s) {
    pod<uint32_t>(static_cast<uint32_t>(s.size()));
    b.insert(b.end(), s.begin(), s.end());
  }
  int handle(const void* ptr) {
    cudaIpcMemHandle_t h{};
    const uint8_t has = ptr != nullptr && !dry;
    pod(has);
    if (has) EDL_CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
    pod(h);
    return EDL_OK;
  }
};
struct BlobR {
  const uint8_t* p;
  size_t n, at = 0;
  bool ok = true;
  template <class T>
  T pod() {
    T v{};
    if (at + sizeof(T) > n) {
      ok = false;
      return v;
    }
    std::memcpy(&v, p + at, sizeof(T));
    at += sizeof(T);
    return v;
  }
  std::string text() {
    const uint32_t k = pod<uint32_t>();
    if (at + k > n) {
      ok = false;
      return {};
    }
    std::string s(reinterpret_cast<const char*>(p + at), k);
    at += k;
    return s;
  }
};
}  // namespace

constexpr uint32_t kStateMagic = 0x45444c53;  // "EDLS"

// Host protocol state at this mini-batch boundary (the leader's decisions so far): t_cur,
// topology version, ring, the lease manager snapshot (datapipeline.cpp:115 layout) and every
// ring member's current shard cursor.  A newcomer process adopts it instead of replaying the
// job's whole history (the newcomer receives the pending topology).
int Job::export_host_state(std::vector<uint8_t>* out) const {
  if (!events_.empty()) return fail(EDL_RETRY, "state: a scaling operation is pending");
  BlobW w;
  w.pod(kStateMagic);
  w.pod<uint64_t>(t_);
  w.pod<uint64_t>(version_);
  w.pod(static_cast<uint32_t>(ring_.size()));
  for (const auto& id : ring_) {
    w.text(id);
    const Cursor& c = workers_.at(id)->cur;
    w.pod<uint8_t>(c.has ? 1 : 0);
    w.pod(c.part);
    w.pod(c.off);
    w.pod(c.len);
    w.pod(c.first);
    w.pod(c.epoch);
  }
  const std::vector<uint8_t> lease = lm_->snapshot();
  w.pod<uint64_t>(lease.size());
  w.b.insert(w.b.end(), lease.begin(), lease.end());
  *out = std::move(w.b);
  return EDL_OK;
}

int Job::adopt_host_state(const uint8_t* blob, size_t len, int64_t switch_t) {
  if (!joining_ || t_ != 0 || launched_ != 0 || events_.size() != 1)
    return fail(EDL_EINVAL, "adopt_state: only a newcomer process before its first step");
  BlobR rd{blob, len};
  if (rd.pod<uint32_t>() != kStateMagic) return fail(EDL_EINVAL, "adopt_state: not a state blob");
  const uint64_t t = rd.pod<uint64_t>();
  const uint64_t version = rd.pod<uint64_t>();
  const uint32_t n = rd.pod<uint32_t>();
  std::vector<std::string> ring;
  std::vector<Cursor> cur;
  for (uint32_t i = 0; i < n && rd.ok; ++i) {
    ring.push_back(rd.text());
    Cursor c;
    c.has = rd.pod<uint8_t>() != 0;
    c.part = rd.pod<uint32_t>();
    c.off = rd.pod<uint64_t>();
    c.len = rd.pod<uint64_t>();
    c.first = rd.pod<uint64_t>();
    c.epoch = rd.pod<uint64_t>();
    cur.push_back(c);
  }
  const uint64_t llen = rd.pod<uint64_t>();
  if (!rd.ok || rd.at + llen > len) return fail(EDL_ETRUNCATED, "adopt_state: truncated");
  if (ring != ring_) return fail(EDL_EINVAL, "adopt_state: the ring changed since the command");
  if (switch_t <= static_cast<int64_t>(t)) return fail(EDL_EINVAL, "adopt_state: switch passed");
  // validated: replace the placeholder state (parse the leases into a copy first)
  auto lm = std::make_unique<LeaseManager>(*lm_);
  LeaseStatus ls;
  try {
    ls = lm->restore(blob + rd.at, llen);
  } catch (const std::exception&) {
    return fail(EDL_ETRUNCATED, "adopt_state: truncated lease state");
  }
  if (ls != LeaseStatus::Ok) return fail(EDL_SHAPE_MISMATCH, "adopt_state: lease state rejected");
  lm_ = std::move(lm);
  for (size_t i = 0; i < ring.size(); ++i) workers_.at(ring[i])->cur = cur[i];
  t_ = t;
  version_ = version;
  events_.front()->switch_t = switch_t;
  log_.clear();
  if (cfg_.keep_log) {  // this process's log starts at the adopted boundary
    LogRec r;
    r.kind = LogRec::Topo;
    r.t = t_ == 0 ? 0 : t_ - 1;
    r.version = version_;
    r.ring = ring_;
    log_.push_back(r);
  }
  resplit();
  return EDL_OK;
}

int Job::export_handles(std::vector<uint8_t>* out) const {
  const Replica* r = reps_.begin()->second.get();
  DeviceGuard g(dry_ ? 0 : r->device);
  BlobW w;
  w.dry = dry_;
  w.pod(kBlobMagic);
  w.pod<int32_t>(my_rank_);
  w.pod<int32_t>(r->device);
  w.pod<uint64_t>(P_);
  EDL_TRY(w.handle(r->W));
  EDL_TRY(w.handle(r->master));
  EDL_TRY(w.handle(r->flags));
  EDL_TRY(w.handle(r->recv));
  EDL_TRY(w.handle(r->mom));
  EDL_TRY(w.handle(r->mlo));
  std::vector<const Worker*> mine;  // local members + this process's scheduled newcomers
  for (const auto& [id, wk] : workers_)
    if (!wk->remote) mine.push_back(wk.get());
  for (const auto& ev : events_)
    if (ev->out)
      for (const auto& wk : ev->prepared)
        if (wk && !wk->remote) mine.push_back(wk.get());
  w.pod(static_cast<uint32_t>(mine.size()));
  for (const Worker* wk : mine) {
    const std::string& id = wk->id;
    w.text(id);
    EDL_TRY(w.handle(wk->grad));
    EDL_TRY(w.handle(wk->g));
    EDL_TRY(w.handle(wk->loss));
  }
  *out = std::move(w.b);
  return EDL_OK;
}

int Job::import_handles(const uint8_t* blob, size_t len) {
  Replica* r = reps_.begin()->second.get();
  DeviceGuard g(dry_ ? 0 : r->device);
  BlobR rd{blob, len};
  if (rd.pod<uint32_t>() != kBlobMagic) return fail(EDL_EINVAL, "import: not an edl handle blob");
  PeerRep peer;
  peer.rank = rd.pod<int32_t>();
  // a second copy of a known replica (or of this process's own) would raise the replica
  // count the collective barriers wait for
  if (rd.ok && peer.rank == my_rank_)
    return fail(EDL_EINVAL, "import: blob of this process's own replica");
  for (auto it = known_peers_.begin(); rd.ok && it != known_peers_.end(); ++it) {
    if (it->rank != peer.rank) continue;
    // a replica whose process left the ring and now re-joins: its old entry (mappings of
    // memory that process has freed) is replaced; a live one is a duplicate
    bool hosts = false;
    for (const auto& [id, w] : workers_) hosts = hosts || (w->remote && w->host_rank == peer.rank);
    if (hosts || it->local)
      return fail(EDL_EINVAL, "import: replica rank " + std::to_string(peer.rank) +
                                  " already imported");
    known_peers_.erase(it);
    break;
  }
  peer.device = rd.pod<int32_t>();
  if (rd.pod<uint64_t>() != P_) return fail(EDL_SHAPE_MISMATCH, "import: model shape differs");
  auto open = [&](void** dst) -> int {
    const uint8_t has = rd.pod<uint8_t>();
    const cudaIpcMemHandle_t h = rd.pod<cudaIpcMemHandle_t>();
    *dst = nullptr;
    if (!has || !rd.ok) return EDL_OK;
    EDL_CUDA_TRY(cudaIpcOpenMemHandle(dst, h, cudaIpcMemLazyEnablePeerAccess));
    ipc_mapped_.push_back(*dst);
    return EDL_OK;
  };
  void* p = nullptr;
  EDL_TRY(open(&p));
  peer.W = static_cast<__nv_bfloat16*>(p);
  EDL_TRY(open(&p));
  peer.master = static_cast<float*>(p);
  EDL_TRY(open(&p));
  peer.flags = static_cast<uint32_t*>(p);
  EDL_TRY(open(&p));
  peer.recv = static_cast<__nv_bfloat16*>(p);
  EDL_TRY(open(&p));
  peer.mom = static_cast<float*>(p);
  EDL_TRY(open(&p));
  peer.mlo = static_cast<uint16_t*>(p);
  const uint32_t n = rd.pod<uint32_t>();
  for (uint32_t i = 0; i < n && rd.ok; ++i) {
    const std::string id = rd.text();
    Worker* w = find_worker(id);  // a ring member or a scheduled newcomer
    if (!w || !w->remote)
      return fail(EDL_UNKNOWN_WORKER, "import: " + id + " is not a remote member of this ring");
    w->imported = true;
    w->host_rank = peer.rank;
    EDL_TRY(open(&p));
    w->grad = static_cast<__nv_bfloat16*>(p);
    EDL_TRY(open(&p));
    w->g = static_cast<double*>(p);
    EDL_TRY(open(&p));
    w->loss = static_cast<double*>(p);
  }
  if (!rd.ok) return fail(EDL_ETRUNCATED, "import: truncated handle blob");
  if (known_peers_.size() >= static_cast<size_t>(kCollMaxReplicas))
    return fail(EDL_EINVAL, "import: too many replicas");
  known_peers_.push_back(peer);
  std::sort(known_peers_.begin(), known_peers_.end(),
            [](const PeerRep& a, const PeerRep& b) { return a.rank < b.rank; });
  rebuild_peers();
  return EDL_OK;
}

int Job::gather_master() {
  EDL_TRY(master_current());  // the deferred push collective / split master
  if (!mlp_ || peers_.size() < 2 || dry_) return EDL_OK;
  Replica* r = primary();
  bool all_local = true;
  for (const auto& p : peers_) all_local = all_local && p.local;
  if (all_local) {
    EDL_TRY(consolidate_master());
  } else {
    DeviceGuard g(r->device);
    CollArgs a;
    for (const auto& p : peers_) {
      a.m_dst[a.n_dst] = p.master;
      a.v_dst[a.n_dst] = p.mom;
      a.flags[a.n_dst] = p.flags;
      ++a.n_dst;
    }
    a.me = rep_index(r);
    a.n_rep = static_cast<int>(peers_.size());
    a.epoch = ++coll_epoch_;
    own_segments(a.me, a.n_rep, &a);
    a.master = r->master;
    a.mom = r->mom;
    EDL_TRY(master_allgather(a, r->stream));
  }
  for (auto& [dev, rr] : reps_) {
    DeviceGuard g(dev);
    EDL_CUDA_TRY(cudaStreamSynchronize(rr->stream));
  }
  return EDL_OK;
}

}  // namespace edl
