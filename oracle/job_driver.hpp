// ORACLE — TEST INFRASTRUCTURE ONLY (see restate.hpp header).
//
// Deterministic mini-batch protocol of an elastic data-parallel SGD job, driven over
// partition leases.  The reference runtime that would own this loop is absent
// (SPEC.md:272-392), so the protocol is fixed here once (SURVEY.md
// §8(a')) and the product runtime (paper_1909_11985_b200/csrc/runtime.cpp) follows it
// verbatim:
//   * each step t, pending topology events with switch_t == t are installed first
//     (notify_batch_end of step t-1): scale-out appends newcomers in
//     ascending id order and registers them; scale-in reclaims each leaver's shards in
//     ring order (datapipeline.cpp:73-84) and unregisters it; version += 1; the switch is
//     logged as `topo <t-1> <version> ...` (ring effective from t, trainer.cpp:222-226);
//   * workers draw in ring-rank order: when the current shard is exhausted the worker
//     reports offset=length (erasing it) and calls next_shard; EpochEnd -> ask again;
//     ShardPending -> the worker contributes fewer samples this step; after its draw a
//     worker with a shard still in flight reports its offset (datapipeline.cpp:43-71);
//   * samples are tagged with the epoch current at lease time; id = meta.offset + off;
//   * per-worker batch = split_batch(B, p), or a fixed per-worker
//     batch for the static-scaling sweeps (BASELINE.json configs[1]);
//   * per-worker [grad_sum, count] vectors are combined in ring order
//     (ring_order_reduce == ring_allreduce, allreduce.cpp:60-148) and applied with
//     sgd_step(eta_at(t)) (trainer.cpp:244-271);
//   * failure recovery: consistent = restore a JobCheckpoint (params,
//     t_cur, pipeline state) with the remaining workers: the lease state is restored, every
//     checkpointed member's in-flight shards are reclaimed at their reported offsets
//     (datapipeline.cpp:73-84) so the survivors resume them, leavers are unregistered,
//     the ring becomes the survivors (version + 1, `restore <t-1>` + `topo` records);
//     approximate = roll params, leases, cursors and log back to the start of the failed
//     mini-batch (after its topology install), remove the failed workers as a scale-in
//     would, and redo that mini-batch.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "restate.hpp"

namespace orc {

struct Cursor {
  bool has = false;
  uint32_t part = 0;
  uint64_t off = 0, len = 0, first = 0, epoch = 0;
};

struct JobCfg {
  int model = 0;  // 0 least squares, 1 logistic, 2 no arithmetic (plan/log only)
  double eta = 0.05, decay = 0.0;
  int64_t B = 64;
  int64_t per_worker = 0;  // > 0: fixed per-worker batch instead of split_batch(B, p)
};

// LM: lease manager adapter (next/report/reclaim/add_worker/remove_worker/epoch).
// DS: dataset adapter (get -> orc::Sample).  TR: trainer ops (add_grad/loss/sgd/ring_sum).
template <class LM, class DS, class TR>
class JobDriver {
 public:
  JobDriver(LM& lm, const DS& ds, JobCfg cfg, std::vector<std::string> ring, std::vector<double> w0)
      : lm_(lm), ds_(ds), cfg_(cfg), ring_(std::move(ring)), w_(std::move(w0)) {
    for (const auto& w : ring_) lm_.add_worker(w);
    version_ = 1;
    resplit();
    Rec r;
    r.kind = Rec::Topo;
    r.t = 0;
    r.version = version_;
    r.ring = ring_;
    log_.push_back(r);
  }

  // scale_out / scale_in scheduled at an explicit switch step (the scheduler-side k is
  // computed by switch_delay).
  void schedule(int64_t switch_t, bool out, std::vector<std::string> ids) {
    events_.push_back({switch_t, out, std::move(ids)});
    std::stable_sort(events_.begin(), events_.end(),
                     [](const Ev& a, const Ev& b) { return a.switch_t < b.switch_t; });
  }

  // One mini-batch; returns mean loss over the global batch (0 if empty).
  double step(uint64_t* count_out) {
    install_due();
    pre_ = snapshot();  // boundary state for approximate recovery
    const size_t p = ring_.size();
    plan_.assign(p, {});
    for (size_t r = 0; r < p; ++r) plan_[r] = draw(ring_[r], splits_[r]);
    const size_t dim = w_.size();
    double mean = 0.0;
    uint64_t count = 0;
    if (cfg_.model == 0 || cfg_.model == 1) {
      const Model m = cfg_.model == 0 ? Model::LeastSquares : Model::Logistic;
      std::vector<std::vector<double>> parts(p, std::vector<double>(dim + 1, 0.0));
      double loss = 0.0;
      for (size_t r = 0; r < p; ++r) {
        std::vector<typename DS::SampleT> batch;
        batch.reserve(plan_[r].size());
        for (const auto& [e, id] : plan_[r]) batch.push_back(ds_.get(id));
        for (const auto& s : batch) TR::add_grad(m, w_, s, parts[r].data());
        parts[r][dim] = static_cast<double>(batch.size());
        loss += TR::loss(m, w_, batch);
      }
      std::vector<double> total = TR::ring_sum(parts);
      count = static_cast<uint64_t>(total[dim]);
      if (count > 0) {
        mean = loss / static_cast<double>(count);
        TR::sgd(w_, total.data(), count, eta_at(cfg_.eta, cfg_.decay, t_));
      }
    } else {
      for (const auto& pl : plan_) count += pl.size();
    }
    for (size_t r = 0; r < p; ++r) {
      Rec rec;
      rec.t = t_;
      rec.worker = ring_[r];
      rec.samples = plan_[r];
      log_.push_back(std::move(rec));
    }
    ++t_;
    if (count_out) *count_out = count;
    return mean;
  }

  // State at a mini-batch boundary (JobCheckpoint).
  struct Snap {
    uint64_t t = 0, version = 0;
    std::vector<std::string> ring;
    std::vector<uint8_t> lease;
    std::map<std::string, Cursor> cur;
    std::vector<double> w;
    size_t log_len = 0;
  };
  Snap snapshot() const {
    Snap s;
    s.t = t_;
    s.version = version_;
    s.ring = ring_;
    s.lease = lm_.snapshot();
    s.cur = cur_;
    s.w = w_;
    s.log_len = log_.size();
    return s;
  }

  // Consistent recovery: resume from checkpoint `s` with workers `ring`.
  void restore(const Snap& s, std::vector<std::string> ring) {
    lm_.restore(s.lease.data(), s.lease.size());
    for (const auto& w : s.ring) {
      lm_.reclaim(w);
      if (std::find(ring.begin(), ring.end(), w) == ring.end()) lm_.remove_worker(w);
    }
    for (const auto& w : ring)
      if (std::find(s.ring.begin(), s.ring.end(), w) == s.ring.end()) lm_.add_worker(w);
    cur_.clear();
    events_.clear();
    w_ = s.w;
    t_ = s.t;
    ring_ = std::move(ring);
    version_ = std::max(version_, s.version) + 1;
    if (t_ > 0) {
      Rec r;
      r.kind = Rec::Restore;
      r.t = t_ - 1;
      log_.push_back(r);
    }
    Rec r;
    r.kind = Rec::Topo;
    r.t = t_ == 0 ? 0 : t_ - 1;
    r.version = version_;
    r.ring = ring_;
    log_.push_back(r);
    resplit();
  }

  // Approximate recovery: the last mini-batch failed; `failed` leave and it is redone.
  void fail_approximate(const std::vector<std::string>& failed) {
    lm_.restore(pre_.lease.data(), pre_.lease.size());
    cur_ = pre_.cur;
    w_ = pre_.w;
    t_ = pre_.t;
    ring_ = pre_.ring;
    version_ = pre_.version;
    log_.resize(pre_.log_len);
    std::vector<std::string> keep;
    for (const auto& w : ring_) {
      if (std::find(failed.begin(), failed.end(), w) != failed.end()) {
        lm_.reclaim(w);
        lm_.remove_worker(w);
        cur_.erase(w);
      } else {
        keep.push_back(w);
      }
    }
    ring_ = keep;
    ++version_;
    Rec r;
    r.kind = Rec::Topo;
    r.t = t_ == 0 ? 0 : t_ - 1;
    r.version = version_;
    r.ring = ring_;
    log_.push_back(r);
    resplit();
  }

  const std::vector<std::string>& ring() const { return ring_; }
  const std::vector<int64_t>& splits() const { return splits_; }
  const std::vector<std::vector<std::pair<uint64_t, uint64_t>>>& plan() const { return plan_; }
  const std::vector<Rec>& log() const { return log_; }
  const std::vector<double>& params() const { return w_; }
  uint64_t t() const { return t_; }
  uint64_t version() const { return version_; }

 private:
  struct Ev {
    int64_t switch_t;
    bool out;
    std::vector<std::string> ids;
  };

  void resplit() {
    const int p = static_cast<int>(ring_.size());
    if (cfg_.per_worker > 0)
      splits_.assign(static_cast<size_t>(p), cfg_.per_worker);
    else
      splits_ = split_batch(cfg_.B, p);
  }

  void install_due() {
    bool changed = false;
    while (!events_.empty() && events_.front().switch_t <= static_cast<int64_t>(t_)) {
      Ev ev = events_.front();
      events_.erase(events_.begin());
      if (ev.out) {
        std::vector<std::string> add = ev.ids;
        std::sort(add.begin(), add.end());
        for (const auto& w : add) {
          if (std::find(ring_.begin(), ring_.end(), w) != ring_.end()) continue;
          ring_.push_back(w);
          lm_.add_worker(w);
        }
      } else {
        std::vector<std::string> keep;
        for (const auto& w : ring_) {
          if (std::find(ev.ids.begin(), ev.ids.end(), w) != ev.ids.end()) {
            lm_.reclaim(w);
            lm_.remove_worker(w);
            cur_.erase(w);
          } else {
            keep.push_back(w);
          }
        }
        ring_ = keep;
      }
      ++version_;
      changed = true;
      Rec r;
      r.kind = Rec::Topo;
      r.t = t_ == 0 ? 0 : t_ - 1;
      r.version = version_;
      r.ring = ring_;
      log_.push_back(r);
    }
    if (changed) resplit();
  }

  std::vector<std::pair<uint64_t, uint64_t>> draw(const std::string& w, int64_t need) {
    std::vector<std::pair<uint64_t, uint64_t>> out;
    Cursor& c = cur_[w];
    while (need > 0) {
      if (!c.has) {
        Next n = lm_.next(w);
        if (n.kind == NextKind::EpochEnd) continue;
        if (n.kind == NextKind::Pending || n.status != Pipe::Ok) break;
        c.has = true;
        c.part = n.meta.index;
        c.off = n.resume;
        c.len = n.meta.length;
        c.first = n.meta.offset;
        c.epoch = lm_.epoch();
      }
      const uint64_t k = std::min<uint64_t>(static_cast<uint64_t>(need), c.len - c.off);
      for (uint64_t j = 0; j < k; ++j) out.emplace_back(c.epoch, c.first + c.off + j);
      c.off += k;
      need -= static_cast<int64_t>(k);
      if (c.off >= c.len) {
        lm_.report(w, c.part, c.len);
        c.has = false;
      }
    }
    if (c.has) lm_.report(w, c.part, c.off);
    return out;
  }

  LM& lm_;
  const DS& ds_;
  JobCfg cfg_;
  std::vector<std::string> ring_;
  std::vector<int64_t> splits_;
  std::vector<double> w_;
  std::vector<Ev> events_;
  std::map<std::string, Cursor> cur_;
  std::vector<std::vector<std::pair<uint64_t, uint64_t>>> plan_;
  std::vector<Rec> log_;
  uint64_t t_ = 0;
  uint64_t version_ = 1;
  Snap pre_;
};

}  // namespace orc
