// ORACLE — TEST INFRASTRUCTURE ONLY (see restate.hpp header).
//
// oracle/_ref/libedlref.so: the same C API as liboracle.so (capi_common.inc, prefix ref_)
// but every component is the REFERENCE's own class, compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile (headers shimmed for g++ 13, SURVEY.md
// Appendix B).  Used to (a) generate tests/golden/ fixtures, (b) pin the restatement, and
// (c) time the reference CPU path for bench.py --impl reference.
#include <chrono>
#include <memory>
#include <span>
#include <thread>
#include <variant>

#include "edl/allreduce.hpp"
#include "edl/clock.hpp"
#include "edl/datapipeline.hpp"
#include "edl/dataset.hpp"
#include "edl/trainer.hpp"
#include "edl/transport.hpp"
#include "job_driver.hpp"
#include "restate.hpp"

namespace {

orc::Pipe conv(edl::PipeStatus s) {
  switch (s) {
    case edl::PipeStatus::Ok: return orc::Pipe::Ok;
    case edl::PipeStatus::UnknownWorker: return orc::Pipe::UnknownWorker;
    case edl::PipeStatus::StaleShard: return orc::Pipe::StaleShard;
    case edl::PipeStatus::ShapeMismatch: return orc::Pipe::ShapeMismatch;
  }
  return orc::Pipe::Ok;
}

edl::ModelKind kind_of(orc::Model m) {
  return m == orc::Model::LeastSquares ? edl::ModelKind::LeastSquares : edl::ModelKind::Logistic;
}

struct LeaseT {
  edl::ShardManager sm;
  LeaseT(uint64_t size, int d, uint64_t seed, const std::string& loc) : sm(size, d, seed, loc) {}
  void add_worker(const std::string& w) { sm.register_worker(w); }
  void remove_worker(const std::string& w) { sm.unregister_worker(w); }
  bool has_worker(const std::string& w) const { return sm.is_registered(w); }
  orc::PartitionMeta meta(uint32_t p) const {
    auto m = sm.partition_meta(p);
    return {m.index, m.offset, m.length};
  }
  orc::Next next(const std::string& w) {
    auto r = sm.next_shard(w);
    orc::Next n;
    n.status = conv(r.status);
    if (const auto* s = std::get_if<edl::Shard>(&r.value)) {
      n.kind = orc::NextKind::Shard;
      n.meta = {s->meta.index, s->meta.offset, s->meta.length};
      n.resume = s->resume_offset;
    } else if (const auto* e = std::get_if<edl::EpochEnd>(&r.value)) {
      n.kind = orc::NextKind::EpochEnd;
      n.epoch = e->epoch;
    } else {
      n.kind = orc::NextKind::Pending;
    }
    return n;
  }
  orc::Pipe report(const std::string& w, uint32_t p, uint64_t off) {
    edl::ProgressRecord rec;
    rec.worker = w;
    rec.partition = p;
    rec.next_sample_offset = off;
    return conv(sm.report_progress(rec));
  }
  void reclaim(const std::string& w) { sm.reclaim(w); }
  void reclaim_at(const std::string& w, const std::vector<std::pair<uint32_t, uint64_t>>& o) {
    sm.reclaim_at(w, o);
  }
  void reclaim_missing(const std::set<std::string>& live) { sm.reclaim_missing(live); }
  std::vector<std::pair<uint32_t, uint64_t>> worker_shards(const std::string& w) const {
    return sm.worker_shards(w);
  }
  std::vector<uint8_t> snapshot() const { return sm.snapshot(); }
  orc::Pipe restore(const uint8_t* b, size_t n) {
    return conv(sm.restore(std::span<const uint8_t>(b, n)));
  }
  uint64_t epoch() const { return sm.epoch(); }
  uint64_t epochs_completed() const { return sm.epochs_completed(); }
  uint64_t cursor() const { return sm.cursor(); }
  const std::vector<uint32_t>& permutation() const { return sm.permutation(); }
  size_t reclaimed_count() const { return sm.reclaimed_count(); }
  size_t in_flight_count() const { return sm.in_flight_count(); }
};

struct DataT {
  using SampleT = edl::Sample;
  static edl::Sample make_sample(uint64_t id, std::vector<double> f, double label) {
    edl::Sample s;
    s.id = id;
    s.features = std::move(f);
    s.label = label;
    return s;
  }
  edl::SyntheticDataset ds;
  explicit DataT(edl::SyntheticDataset::Spec s) : ds(s) {}
  edl::Sample get(uint64_t i) const { return ds.get(i); }
  std::vector<double> true_weights() const { return ds.true_weights(); }
  std::string locator() const { return ds.locator(); }
};

struct TrainT {
  static void add_grad(orc::Model m, const std::vector<double>& w, const edl::Sample& s, double* g) {
    edl::accumulate_gradient(kind_of(m), w, s, std::span<double>(g, w.size()));
  }
  static double loss(orc::Model m, const std::vector<double>& w, const std::vector<edl::Sample>& b) {
    return edl::batch_loss(kind_of(m), w, b);
  }
  static void sgd(std::vector<double>& w, const double* g, uint64_t count, double eta) {
    edl::sgd_step(w, std::span<const double>(g, w.size()), count, eta);
  }
  static std::vector<double> ring_sum(const std::vector<std::vector<double>>& v) {
    return edl::ring_order_reduce(v, edl::ReduceOp::Sum);
  }
  static int coverage_file(const char* path, uint64_t n, uint64_t* fe, std::string* d) {
    auto c = edl::check_coverage(edl::effective_log(edl::read_log_file(path)), n);
    *fe = c.full_epochs;
    *d = c.detail;
    return c.ok ? 1 : 0;
  }
  static int replay_file(const char* path, int model, const DataT& ds, std::vector<double>& w,
                         double eta, double decay, bool ring, std::string* e, uint64_t* batches) {
    edl::HyperParams hp;
    hp.eta = eta;
    hp.decay = decay;
    auto r = edl::oracle_replay(edl::effective_log(edl::read_log_file(path)),
                                model == 0 ? edl::ModelKind::LeastSquares : edl::ModelKind::Logistic,
                                ds.ds, w, hp,
                                ring ? edl::ReplayOrder::RingOrder : edl::ReplayOrder::Concatenated);
    w = r.w;
    *e = r.error;
    *batches = r.batches;
    return r.ok ? 1 : 0;
  }
};

std::unique_ptr<DataT> make_data(uint64_t size, int dim, uint64_t seed, double noise, bool sign) {
  edl::SyntheticDataset::Spec s;
  s.size = size;
  s.dim = dim;
  s.seed = seed;
  s.noise = noise;
  s.sign_labels = sign;
  return std::make_unique<DataT>(s);
}
std::unique_ptr<LeaseT> make_lease(uint64_t size, int d, uint64_t seed, const std::string& loc) {
  return std::make_unique<LeaseT>(size, d, seed, loc);
}

}  // namespace

#define EDL_PFX(name) ref_##name
#include "capi_common.inc"

extern "C" {

// The reference's actual threaded ring_allreduce (allreduce.cpp:60-130) over an
// InProcFabric, one thread per rank; pins ring_order_reduce == ring_allreduce (AC1).
// Returns transfers performed by rank 0, or -1 on a non-Ok status.
int ref_ring_allreduce_threads(const double* in, int n, size_t len, double* out) {
  edl::SystemClock clock;
  edl::InProcFabric::Options opts;
  opts.max_payload = size_t(1) << 40;
  edl::InProcFabric fabric(clock, opts);
  edl::Topology topo;
  topo.version = 1;
  for (int r = 0; r < n; ++r) topo.ring.push_back("w" + std::to_string(r));
  std::vector<std::shared_ptr<edl::Mailbox>> boxes;
  for (int r = 0; r < n; ++r) boxes.push_back(fabric.attach(topo.ring[r]));
  std::vector<edl::ReduceOutcome> res(static_cast<size_t>(n));
  std::vector<std::thread> th;
  for (int r = 0; r < n; ++r) {
    th.emplace_back([&, r] {
      edl::FabricChunkIO io(fabric, boxes[r]->channel(0), topo.ring[r], topo.successor(r));
      res[r] = edl::ring_allreduce(std::span<const double>(in + r * len, len), topo, topo.ring[r],
                                   edl::ReduceOp::Sum, io, 0, std::chrono::seconds(30));
    });
  }
  for (auto& t : th) t.join();
  for (int r = 0; r < n; ++r) {
    if (res[r].status != edl::ReduceStatus::Ok) return -1;
    std::memcpy(out + r * len, res[r].data.data(), sizeof(double) * len);
  }
  return res[0].transfers;
}

}  // extern "C"
