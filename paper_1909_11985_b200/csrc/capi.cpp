// extern "C" surface (include/edl_b200.h).  No exceptions cross this boundary: every
// reference exception class maps to an EDL_E* code + edl_last_error() text.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "edl_internal.hpp"
#include "kernels.hpp"
#include "lease.hpp"
#include "runtime.hpp"

struct EdlLeaseManager {
  edl::LeaseManager lm;
};
struct EdlDataset {
  edl::Dataset* ds;
};
struct EdlJob {
  edl::Job* job;
};

namespace {

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    return edl::fail(EDL_EINVAL, e.what());
  } catch (const std::out_of_range& e) {
    return edl::fail(EDL_OUT_OF_RANGE, e.what());
  } catch (const std::bad_alloc& e) {
    return edl::fail(EDL_ENOMEM, e.what());
  } catch (const std::runtime_error& e) {
    const std::string m = e.what();
    return edl::fail(m.find("truncated") != std::string::npos ? EDL_ETRUNCATED : EDL_EIO, m);
  } catch (const std::exception& e) {
    return edl::fail(EDL_EINVAL, e.what());
  }
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

int copy_text(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return EDL_OK;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ leases
int32_t edl_default_partition_count(int32_t w) { return edl::default_partitions(w); }

int edl_lease_create(uint64_t size, int32_t partitions, uint64_t seed, const char* locator,
                     EdlLeaseManager** out) {
  return guarded([&]() -> int {
    if (partitions <= 0) return edl::fail(EDL_EINVAL, "partitions must be positive");
    *out = new EdlLeaseManager{edl::LeaseManager(size, partitions, seed, locator ? locator : "")};
    return EDL_OK;
  });
}
void edl_lease_destroy(EdlLeaseManager* lm) { delete lm; }
int edl_lease_register(EdlLeaseManager* lm, const char* w) {
  return guarded([&]() -> int {
    lm->lm.enroll(w);
    return EDL_OK;
  });
}
int edl_lease_unregister(EdlLeaseManager* lm, const char* w) {
  return guarded([&]() -> int {
    lm->lm.retire(w);
    return EDL_OK;
  });
}
int edl_lease_is_registered(const EdlLeaseManager* lm, const char* w) {
  return lm->lm.enrolled(w) ? 1 : 0;
}
int edl_lease_next(EdlLeaseManager* lm, const char* w, EdlNextShard* out) {
  return guarded([&]() -> int {
    const edl::Lease l = lm->lm.next(w);
    *out = EdlNextShard{};
    out->kind = static_cast<int32_t>(l.kind);
    out->meta = EdlPartitionMeta{l.meta.index, l.meta.offset, l.meta.length};
    out->resume_offset = l.resume;
    out->epoch = l.epoch;
    if (l.status != edl::LeaseStatus::Ok)
      return edl::fail(static_cast<int>(l.status), std::string("unknown worker ") + w);
    return EDL_OK;
  });
}
int edl_lease_report(EdlLeaseManager* lm, const char* w, uint32_t part, uint64_t off) {
  return guarded([&]() -> int {
    const auto st = lm->lm.progress(w, part, off);
    if (st == edl::LeaseStatus::Ok) return EDL_OK;
    return edl::fail(static_cast<int>(st), st == edl::LeaseStatus::UnknownWorker
                                               ? "unknown worker"
                                               : "stale shard");
  });
}
int edl_lease_reclaim(EdlLeaseManager* lm, const char* w) {
  return guarded([&]() -> int {
    lm->lm.reclaim(w);
    return EDL_OK;
  });
}
int edl_lease_reclaim_at(EdlLeaseManager* lm, const char* w, const uint32_t* parts,
                         const uint64_t* offs, size_t n) {
  return guarded([&]() -> int {
    std::vector<std::pair<uint32_t, uint64_t>> v;
    for (size_t i = 0; i < n; ++i) v.emplace_back(parts[i], offs[i]);
    lm->lm.reclaim_at(w, v);
    return EDL_OK;
  });
}
int edl_lease_reclaim_missing(EdlLeaseManager* lm, const char* const* live, size_t n) {
  return guarded([&]() -> int {
    std::set<std::string> s;
    for (size_t i = 0; i < n; ++i) s.insert(live[i]);
    lm->lm.reclaim_missing(s);
    return EDL_OK;
  });
}
int edl_lease_partition_meta(const EdlLeaseManager* lm, uint32_t index, EdlPartitionMeta* out) {
  if (index >= static_cast<uint32_t>(lm->lm.partitions()))
    return edl::fail(EDL_OUT_OF_RANGE, "partition index");
  const auto m = lm->lm.meta(index);
  *out = EdlPartitionMeta{m.index, m.offset, m.length};
  return EDL_OK;
}
size_t edl_lease_worker_shards(const EdlLeaseManager* lm, const char* w, uint32_t* parts,
                               uint64_t* offs, size_t cap) {
  const auto v = lm->lm.held_by(w);
  for (size_t i = 0; i < v.size() && i < cap; ++i) {
    parts[i] = v[i].first;
    offs[i] = v[i].second;
  }
  return v.size();
}
int edl_lease_snapshot(const EdlLeaseManager* lm, uint8_t* buf, size_t cap, size_t* len) {
  return guarded([&]() -> int {
    const auto s = lm->lm.snapshot();
    if (len) *len = s.size();
    if (buf) std::memcpy(buf, s.data(), s.size() < cap ? s.size() : cap);
    return EDL_OK;
  });
}
int edl_lease_restore(EdlLeaseManager* lm, const uint8_t* buf, size_t len) {
  return guarded([&]() -> int {
    const auto st = lm->lm.restore(buf, len);
    if (st == edl::LeaseStatus::Ok) return EDL_OK;
    return edl::fail(EDL_SHAPE_MISMATCH, "snapshot shape mismatch (size or d)");
  });
}
uint64_t edl_lease_epoch(const EdlLeaseManager* lm) { return lm->lm.epoch(); }
uint64_t edl_lease_epochs_completed(const EdlLeaseManager* lm) { return lm->lm.epochs_completed(); }
uint64_t edl_lease_cursor(const EdlLeaseManager* lm) { return lm->lm.cursor(); }
size_t edl_lease_permutation(const EdlLeaseManager* lm, uint32_t* out, size_t cap) {
  const auto& p = lm->lm.permutation();
  for (size_t i = 0; i < p.size() && i < cap; ++i) out[i] = p[i];
  return p.size();
}
size_t edl_lease_reclaimed_count(const EdlLeaseManager* lm) { return lm->lm.reclaimed_count(); }
size_t edl_lease_in_flight_count(const EdlLeaseManager* lm) { return lm->lm.in_flight_count(); }

// ------------------------------------------------------------------ runtime arithmetic
int edl_split_batch(int64_t B, int32_t p, int64_t* out) {
  if (p < 1 || B < p) return edl::fail(EDL_EINVAL, "split_batch: B < p");
  for (int32_t r = 0; r < p; ++r) out[r] = B / p + (r < B % p ? 1 : 0);
  return EDL_OK;
}
int64_t edl_switch_delay(double ta, double tb) {
  if (!(tb > 0)) return 1;
  const double k = std::ceil(ta / tb);
  return k < 1 ? 1 : static_cast<int64_t>(k);
}
double edl_eta_at(double eta, double decay, uint64_t t) {
  return eta / (1.0 + decay * static_cast<double>(t));
}

// ------------------------------------------------------------------ dataset
int edl_dataset_create_synthetic(const EdlSyntheticSpec* spec, int32_t dtype, int32_t num_classes,
                                 EdlDataset** out) {
  return guarded([&]() -> int {
    edl::Dataset* ds = nullptr;
    const int rc = edl::dataset_create(*spec, dtype, num_classes, &ds);
    if (rc != EDL_OK) return rc;
    *out = new EdlDataset{ds};
    return EDL_OK;
  });
}
void edl_dataset_destroy(EdlDataset* ds) {
  if (!ds) return;
  edl::dataset_destroy(ds->ds);
  delete ds;
}
uint64_t edl_dataset_size(const EdlDataset* ds) { return ds->ds->spec.size; }
int32_t edl_dataset_dim(const EdlDataset* ds) { return ds->ds->spec.dim; }
const void* edl_dataset_features(const EdlDataset* ds) { return ds->ds->x; }
const void* edl_dataset_labels(const EdlDataset* ds) { return ds->ds->y; }
int edl_dataset_true_weights(const EdlDataset* ds, double* out) {
  std::memcpy(out, ds->ds->w_true.data(), sizeof(double) * ds->ds->w_true.size());
  return EDL_OK;
}
int edl_dataset_get(const EdlDataset* ds, uint64_t index, double* f, double* label) {
  return edl::dataset_get(ds->ds, index, f, label);
}
int edl_gather(const EdlDataset* ds, const EdlRun* runs_dev, int32_t n_runs, int64_t n_rows,
               void* x_out, void* y_out, void* stream) {
  return edl::gather(ds->ds, runs_dev, n_runs, n_rows, x_out, y_out, S(stream));
}

// ------------------------------------------------------------------ linear trainer
int edl_local_gradient(int32_t kind, const double* w, const double* x, const double* y, int64_t n,
                       int32_t dim, double* grad_out, void* stream) {
  if (dim <= 0 || n < 0) return edl::fail(EDL_EINVAL, "gradient dimension mismatch");
  // no workspace: one fused launch, nothing allocated on the call path
  return edl::linear_local_gradient(kind, w, x, y, n, dim, grad_out, nullptr, S(stream));
}
int edl_batch_loss(int32_t kind, const double* w, const double* x, const double* y, int64_t n,
                   int32_t dim, double* loss_out, void* stream) {
  if (dim <= 0 || n < 0) return edl::fail(EDL_EINVAL, "loss dimension mismatch");
  return edl::linear_batch_loss(kind, w, x, y, n, dim, loss_out, nullptr, S(stream));
}
int edl_sgd_step(double* w, const double* g, int64_t count, double eta, int32_t dim,
                 void* stream) {
  return edl::linear_sgd(w, g, count, eta, dim, S(stream));
}
int edl_master_split(const float* master, uint16_t* lo, void* W, size_t n, void* stream) {
  return edl::master_split(master, lo, static_cast<__nv_bfloat16*>(W), n, S(stream));
}
int edl_master_join(const void* W, const uint16_t* lo, float* master, size_t n, void* stream) {
  return edl::master_join(static_cast<const __nv_bfloat16*>(W), lo, master, n, S(stream));
}
int edl_ring_allreduce_f64(const double* const* inputs, int32_t n, size_t len, int32_t op,
                           double* out, void* stream) {
  return edl::ring_allreduce_f64(inputs, n, len, op, out, S(stream));
}

// ------------------------------------------------------------------ job
void edl_job_config_default(EdlJobConfig* c) {
  *c = EdlJobConfig{};
  c->model = EDL_MODEL_LEAST_SQUARES;
  c->data = EdlSyntheticSpec{8192, 64, 1, 0.01, 0};
  c->num_classes = 4096;
  c->layers = 8;
  c->hidden = 4096;
  c->eta = 0.05;  // HyperParams defaults, trainer.hpp:20-25
  c->decay = 0.0;
  c->momentum = 0.0;
  c->batch = 64;
  c->per_worker_batch = 0;
  c->lease_seed = 7;
  c->partitions = 0;
  c->max_workers = 1;
  c->init_seed = 0;
  c->t_a_ms = 500.0;
  c->keep_log = 1;
  c->dry_run = 0;
  const char* appx = std::getenv("USE_APPX_RECOVERY");  // SPEC.md:384, default consistent
  c->appx_recovery = (appx && std::atoi(appx) != 0) ? 1 : 0;
}

int edl_job_create(const EdlJobConfig* cfg, const char* const* ring, const int32_t* devices,
                   int32_t n, EdlJob** out) {
  return guarded([&]() -> int {
    std::vector<std::string> r;
    std::vector<int> d;
    for (int32_t i = 0; i < n; ++i) {
      r.emplace_back(ring[i]);
      d.push_back(devices ? devices[i] : 0);
    }
    edl::Job* j = nullptr;
    const int rc = edl::Job::create(*cfg, r, d, &j);
    if (rc != EDL_OK) return rc;
    *out = new EdlJob{j};
    return EDL_OK;
  });
}
int edl_job_create_joining(const EdlJobConfig* cfg, const char* const* ring, int32_t n,
                           const char* const* newcomers, int32_t n_new, const char* self_id,
                           int32_t device, int32_t rank, int64_t switch_t, EdlJob** out) {
  return guarded([&]() -> int {
    if (!self_id) return edl::fail(EDL_EINVAL, "create_joining: no worker id");
    std::vector<std::string> r, nc;
    for (int32_t i = 0; i < n; ++i) r.emplace_back(ring[i]);
    for (int32_t i = 0; i < n_new; ++i) nc.emplace_back(newcomers[i]);
    edl::Job* j = nullptr;
    const int rc = edl::Job::create_joining(*cfg, r, nc, self_id, device, rank, switch_t, &j);
    if (rc != EDL_OK) return rc;
    *out = new EdlJob{j};
    return EDL_OK;
  });
}
void edl_job_destroy(EdlJob* job) {
  if (!job) return;
  delete job->job;
  delete job;
}
int edl_job_step(EdlJob* job, EdlStepReport* rep) {
  return guarded([&]() -> int { return job->job->step(rep); });
}
int edl_job_sync(EdlJob* job, EdlStepReport* rep) {
  return guarded([&]() -> int { return job->job->sync(rep); });
}
static std::vector<std::string> ids_of(const char* const* ids, int32_t n) {
  std::vector<std::string> v;
  for (int32_t i = 0; i < n; ++i) v.emplace_back(ids[i]);
  return v;
}
static std::vector<int> devs_of(const int32_t* d, int32_t n) {
  std::vector<int> v;
  for (int32_t i = 0; i < n; ++i) v.push_back(d ? d[i] : 0);
  return v;
}
int edl_job_scale_out(EdlJob* job, const char* const* ids, const int32_t* devices, int32_t n,
                      int64_t* switch_t) {
  return guarded([&]() -> int {
    return job->job->scale(true, ids_of(ids, n), devs_of(devices, n), -1, switch_t);
  });
}
int edl_job_scale_in(EdlJob* job, const char* const* ids, int32_t n, double allowance_ms,
                     int64_t* switch_t) {
  (void)allowance_ms;  // leavers exit in-process at switch_t; the allowance cannot be exceeded
  return guarded([&]() -> int { return job->job->scale(false, ids_of(ids, n), {}, -1, switch_t); });
}
int edl_job_schedule(EdlJob* job, int64_t switch_t, int32_t out, const char* const* ids,
                     const int32_t* devices, int32_t n) {
  return guarded([&]() -> int {
    if (switch_t < 0) return edl::fail(EDL_EINVAL, "switch_t must be >= 0");
    return job->job->scale(out != 0, ids_of(ids, n), out ? devs_of(devices, n) : std::vector<int>{},
                           switch_t, nullptr);
  });
}
int edl_job_params(EdlJob* job, const char* worker, void* host, size_t bytes) {
  return guarded([&]() -> int { return job->job->params(worker, host, bytes); });
}
size_t edl_job_param_count(const EdlJob* job) { return job->job->param_count(); }
uint64_t edl_job_t(const EdlJob* job) { return job->job->t(); }
double edl_job_median_step_ms(const EdlJob* job) { return job->job->median_step_ms(); }
int edl_job_log(const EdlJob* job, char* buf, size_t cap, size_t* len) {
  return copy_text(job->job->log_text(), buf, cap, len);
}
int edl_job_ring(const EdlJob* job, char* buf, size_t cap, size_t* len) {
  return copy_text(job->job->ring_csv(), buf, cap, len);
}
int edl_job_lease_snapshot(const EdlJob* job, uint8_t* buf, size_t cap, size_t* len) {
  std::vector<uint8_t> s;
  job->job->lease_snapshot(&s);
  if (len) *len = s.size();
  if (buf) std::memcpy(buf, s.data(), s.size() < cap ? s.size() : cap);
  return EDL_OK;
}

}  // extern "C"

extern "C" {
void* edl_job_stream(const EdlJob* job) { return job->job->stream(); }
void edl_job_set_profile(EdlJob* job, int32_t on) { job->job->set_profile(on != 0); }
int edl_job_exchange_mode(const EdlJob* job) { return job->job->exchange_mode(); }
int edl_job_join(EdlJob* job) { return job->job->join_side(); }
void edl_job_counters(const EdlJob* job, double* phase_ms, uint64_t* steps, uint64_t* launches) {
  job->job->phase_totals(phase_ms, steps, launches);
}
void edl_job_reset_counters(EdlJob* job) { job->job->reset_counters(); }
int edl_job_export(const EdlJob* job, uint8_t* buf, size_t cap, size_t* len) {
  return guarded([&]() -> int {
    std::vector<uint8_t> b;
    const int rc = job->job->export_handles(&b);
    if (rc != EDL_OK) return rc;
    if (len) *len = b.size();
    if (buf) std::memcpy(buf, b.data(), b.size() < cap ? b.size() : cap);
    return EDL_OK;
  });
}
int edl_job_export_state(const EdlJob* job, uint8_t* buf, size_t cap, size_t* len) {
  return guarded([&]() -> int {
    std::vector<uint8_t> b;
    const int rc = job->job->export_host_state(&b);
    if (rc != EDL_OK) return rc;
    if (len) *len = b.size();
    if (buf) std::memcpy(buf, b.data(), b.size() < cap ? b.size() : cap);
    return EDL_OK;
  });
}
int edl_job_adopt_state(EdlJob* job, const uint8_t* blob, size_t len, int64_t switch_t) {
  return guarded([&]() -> int { return job->job->adopt_host_state(blob, len, switch_t); });
}
int edl_job_import(EdlJob* job, const uint8_t* blob, size_t len) {
  return guarded([&]() -> int { return job->job->import_handles(blob, len); });
}
int edl_job_set_params(EdlJob* job, const void* host, size_t bytes) {
  return guarded([&]() -> int { return job->job->set_params(host, bytes); });
}
int edl_job_gather_master(EdlJob* job) {
  return guarded([&]() -> int { return job->job->gather_master(); });
}
}  // extern "C"

extern "C" {
int edl_detect_straggler(const double* durations, int32_t n_batches, int32_t n_workers,
                         int32_t window, double factor, int32_t* worker) {
  return guarded([&]() -> int {
    if (!worker || (n_batches > 0 && n_workers > 0 && !durations))
      return edl::fail(EDL_EINVAL, "detect_straggler: null argument");
    *worker = edl::detect_straggler(durations, n_batches, n_workers, window, factor);
    return EDL_OK;
  });
}
int edl_job_worker_ms(const EdlJob* job, const char* worker, double* out, size_t cap,
                      size_t* n) {
  return guarded([&]() -> int {
    std::vector<double> v;
    job->job->worker_ms(worker, &v);
    if (n) *n = v.size();
    if (out) std::memcpy(out, v.data(), sizeof(double) * (v.size() < cap ? v.size() : cap));
    return EDL_OK;
  });
}
int edl_job_straggler(const EdlJob* job, int32_t window, double factor, char* buf, size_t cap,
                      size_t* len) {
  return guarded([&]() -> int { return copy_text(job->job->straggler(window, factor), buf, cap, len); });
}
int edl_job_set_worker_delay(EdlJob* job, const char* worker, double us) {
  return guarded([&]() -> int { return job->job->set_worker_delay(worker, us); });
}
}  // extern "C"

extern "C" {
int edl_job_save_checkpoint(EdlJob* job, const char* path) {
  return guarded([&]() -> int { return job->job->save_checkpoint(path ? path : ""); });
}
int edl_job_load_checkpoint(EdlJob* job, const char* path) {
  return guarded([&]() -> int { return job->job->load_checkpoint(path ? path : ""); });
}
int edl_job_fail(EdlJob* job, const char* const* ids, int32_t n, int32_t approximate,
                 EdlRecovery* out) {
  return guarded([&]() -> int {
    std::vector<std::string> v;
    for (int32_t i = 0; i < n; ++i) v.emplace_back(ids[i]);
    EdlRecovery r{};
    const int rc = job->job->recover(v, approximate != 0, &r);
    if (out) *out = r;
    return rc;
  });
}
}  // extern "C"
