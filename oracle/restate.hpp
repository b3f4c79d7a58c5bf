// ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product (libedl_b200.so).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
//
// Independent CPU restatement of the reference EDL hot-path components, written from
// SURVEY.md §8(a) (not from the reference source).  Each function cites the reference
// file:line (relative to /root/reference/proj) whose behaviour it restates.  Pinned by
// tests/test_oracle_golden.py against vectors produced by the reference itself
// (oracle/_ref, tests/golden/).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <numeric>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- synthetic data
// splitmix64 finaliser, src/dataset.cpp:13-18
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// top 53 bits -> [0,1), src/dataset.cpp:20-23
inline double unit_double(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

struct SynthSpec {
  uint64_t size = 0;
  int dim = 0;
  uint64_t seed = 0;
  double noise = 0.0;
  bool sign_labels = false;
};

struct Sample {
  uint64_t id = 0;
  std::vector<double> features;
  double label = 0.0;
};

// SyntheticDataset, src/dataset.cpp:27-54
class Synth {
 public:
  using SampleT = Sample;
  static Sample make_sample(uint64_t id, std::vector<double> f, double label) {
    return Sample{id, std::move(f), label};
  }
  explicit Synth(SynthSpec s) : spec_(s) {
    w_true_.resize(static_cast<size_t>(s.dim));
    uint64_t st = splitmix64(s.seed ^ 0x77ee55aa11cc33ddULL);  // :29
    for (auto& w : w_true_) {
      st = splitmix64(st);
      w = 2.0 * unit_double(st) - 1.0;
    }
  }
  uint64_t size() const { return spec_.size; }
  int dim() const { return spec_.dim; }
  const std::vector<double>& true_weights() const { return w_true_; }
  Sample get(uint64_t i) const {
    if (i >= spec_.size) throw std::out_of_range("sample index");  // :37
    Sample s;
    s.id = i;
    s.features.resize(static_cast<size_t>(spec_.dim));
    uint64_t st = splitmix64(spec_.seed ^ (i * 0xd1342543de82ef95ULL + 1));  // :41
    for (auto& f : s.features) {
      st = splitmix64(st);
      f = 2.0 * unit_double(st) - 1.0;
    }
    // sequential dot, no FMA contraction (built with -ffp-contract=off) :48-49
    double yy = 0.0;
    for (int k = 0; k < spec_.dim; ++k)
      yy += w_true_[static_cast<size_t>(k)] * s.features[static_cast<size_t>(k)];
    if (spec_.noise > 0.0) {  // :50-53
      st = splitmix64(st);
      yy += spec_.noise * (2.0 * unit_double(st) - 1.0);
    }
    s.label = spec_.sign_labels ? (yy >= 0.0 ? 1.0 : -1.0) : yy;
    return s;
  }
  std::string locator() const {  // :56-58
    return "synthetic:" + std::to_string(spec_.seed) + ":" + std::to_string(spec_.size);
  }

 private:
  SynthSpec spec_;
  std::vector<double> w_true_;
};

// ---------------------------------------------------------------- partition leasing
inline int default_partition_count(int w) { return std::max(4 * w, 64); }  // datapipeline.cpp:9-11

struct PartitionMeta {
  uint32_t index = 0;
  uint64_t offset = 0;
  uint64_t length = 0;
};
enum class NextKind { Shard, EpochEnd, Pending };
enum class Pipe { Ok, UnknownWorker, StaleShard, ShapeMismatch };
struct Next {
  Pipe status = Pipe::Ok;
  NextKind kind = NextKind::Pending;
  PartitionMeta meta;
  uint64_t resume = 0;
  uint64_t epoch = 0;
};

// ShardManager, include/edl/datapipeline.hpp:58-127, src/datapipeline.cpp:13-178
class Leases {
 public:
  Leases(uint64_t size, int d, uint64_t seed, std::string locator)
      : size_(size), d_(d), locator_(std::move(locator)), rng_(seed) {
    reshuffle();
  }
  void add_worker(const std::string& w) { workers_.insert(w); }
  void remove_worker(const std::string& w) { workers_.erase(w); }
  bool has_worker(const std::string& w) const { return workers_.count(w) != 0; }

  PartitionMeta meta(uint32_t p) const {  // :34-41
    PartitionMeta m;
    m.index = p;
    m.offset = size_ * p / static_cast<uint64_t>(d_);
    m.length = size_ * (p + 1) / static_cast<uint64_t>(d_) - m.offset;
    return m;
  }

  Next next(const std::string& w) {  // :43-62
    Next r;
    if (!workers_.count(w)) {
      r.status = Pipe::UnknownWorker;
      return r;
    }
    if (!returned_.empty()) {  // reclaimed-first
      auto [p, off] = returned_.front();
      returned_.pop_front();
      live_[p] = {w, off};
      r.kind = NextKind::Shard;
      r.meta = meta(p);
      r.resume = off;
      return r;
    }
    if (pos_ < static_cast<uint64_t>(d_)) {
      uint32_t p = order_[pos_];
      ++pos_;
      live_[p] = {w, 0};
      r.kind = NextKind::Shard;
      r.meta = meta(p);
      return r;
    }
    if (!live_.empty()) {
      r.kind = NextKind::Pending;
      return r;
    }
    r.kind = NextKind::EpochEnd;
    r.epoch = epoch_;
    ++epoch_;
    ++done_;
    reshuffle();
    return r;
  }

  Pipe report(const std::string& w, uint32_t p, uint64_t off) {  // :64-71
    if (!workers_.count(w)) return Pipe::UnknownWorker;
    auto it = live_.find(p);
    if (it == live_.end() || it->second.worker != w) return Pipe::StaleShard;
    it->second.off = off;
    if (off >= meta(p).length) live_.erase(it);
    return Pipe::Ok;
  }

  void reclaim(const std::string& w) {  // :73-84 (ascending partition order, std::map)
    for (auto it = live_.begin(); it != live_.end();) {
      if (it->second.worker == w) {
        if (it->second.off < meta(it->first).length) returned_.emplace_back(it->first, it->second.off);
        it = live_.erase(it);
      } else {
        ++it;
      }
    }
  }
  void reclaim_at(const std::string& w, const std::vector<std::pair<uint32_t, uint64_t>>& offs) {
    for (const auto& [p, off] : offs) {  // :86-93
      auto it = live_.find(p);
      if (it != live_.end() && it->second.worker == w) it->second.off = off;
    }
    reclaim(w);
  }
  void reclaim_missing(const std::set<std::string>& live) {  // :95-104
    std::vector<std::string> gone;
    for (const auto& w : workers_)
      if (!live.count(w)) gone.push_back(w);
    for (const auto& w : gone) {
      reclaim(w);
      workers_.erase(w);
    }
  }
  std::vector<std::pair<uint32_t, uint64_t>> worker_shards(const std::string& w) const {
    std::vector<std::pair<uint32_t, uint64_t>> out;  // :106-113
    for (const auto& [p, a] : live_)
      if (a.worker == w) out.emplace_back(p, a.off);
    return out;
  }

  // Little-endian snapshot, src/datapipeline.cpp:115-142 / include/edl/bytes.hpp:14-51
  std::vector<uint8_t> snapshot() const {
    std::vector<uint8_t> b;
    auto raw = [&](const void* p, size_t n) {
      const auto* c = static_cast<const uint8_t*>(p);
      b.insert(b.end(), c, c + n);
    };
    auto u32 = [&](uint32_t v) { raw(&v, 4); };
    auto u64 = [&](uint64_t v) { raw(&v, 8); };
    auto str = [&](const std::string& s) {
      u32(static_cast<uint32_t>(s.size()));
      raw(s.data(), s.size());
    };
    u64(size_);
    int64_t d = d_;
    raw(&d, 8);
    str(locator_);
    u64(epoch_);
    u64(done_);
    u64(pos_);
    u64(order_.size());
    for (uint32_t p : order_) u32(p);
    u64(returned_.size());
    for (const auto& [p, off] : returned_) {
      u32(p);
      u64(off);
    }
    u64(live_.size());
    for (const auto& [p, a] : live_) {
      u32(p);
      str(a.worker);
      u64(a.off);
    }
    u64(workers_.size());
    for (const auto& w : workers_) str(w);
    std::ostringstream rs;
    rs << rng_;
    str(rs.str());
    return b;
  }
  // src/datapipeline.cpp:144-178; throws std::runtime_error on truncation (bytes.hpp:112)
  Pipe restore(const uint8_t* data, size_t n) {
    size_t pos = 0;
    auto need = [&](size_t k) {
      if (pos + k > n) throw std::runtime_error("truncated payload");
    };
    auto rd = [&](void* dst, size_t k) {
      need(k);
      std::memcpy(dst, data + pos, k);
      pos += k;
    };
    auto u32 = [&]() { uint32_t v; rd(&v, 4); return v; };
    auto u64 = [&]() { uint64_t v; rd(&v, 8); return v; };
    auto str = [&]() {
      uint32_t k = u32();
      need(k);
      std::string s(reinterpret_cast<const char*>(data + pos), k);
      pos += k;
      return s;
    };
    uint64_t size = u64();
    int64_t d;
    rd(&d, 8);
    if (size != size_ || static_cast<int>(d) != d_) return Pipe::ShapeMismatch;
    locator_ = str();
    epoch_ = u64();
    done_ = u64();
    pos_ = u64();
    order_.resize(u64());
    for (auto& p : order_) p = u32();
    returned_.clear();
    uint64_t rn = u64();
    for (uint64_t i = 0; i < rn; ++i) {
      uint32_t p = u32();
      uint64_t off = u64();
      returned_.emplace_back(p, off);
    }
    live_.clear();
    uint64_t fn = u64();
    for (uint64_t i = 0; i < fn; ++i) {
      uint32_t p = u32();
      Live a;
      a.worker = str();
      a.off = u64();
      live_[p] = a;
    }
    workers_.clear();
    uint64_t wn = u64();
    for (uint64_t i = 0; i < wn; ++i) workers_.insert(str());
    std::istringstream rs(str());
    rs >> rng_;
    return Pipe::Ok;
  }

  uint64_t epoch() const { return epoch_; }
  uint64_t epochs_completed() const { return done_; }
  uint64_t cursor() const { return pos_; }
  const std::vector<uint32_t>& permutation() const { return order_; }
  size_t reclaimed_count() const { return returned_.size(); }
  size_t in_flight_count() const { return live_.size(); }

 private:
  void reshuffle() {  // fresh_permutation, :19-24
    order_.resize(static_cast<size_t>(d_));
    std::iota(order_.begin(), order_.end(), 0u);
    std::shuffle(order_.begin(), order_.end(), rng_);
    pos_ = 0;
  }
  struct Live {
    std::string worker;
    uint64_t off = 0;
  };
  uint64_t size_;
  int d_;
  std::string locator_;
  std::mt19937_64 rng_;
  uint64_t epoch_ = 0, done_ = 0, pos_ = 0;
  std::vector<uint32_t> order_;
  std::deque<std::pair<uint32_t, uint64_t>> returned_;
  std::map<uint32_t, Live> live_;
  std::set<std::string> workers_;
};

// ---------------------------------------------------------------- linear trainer
enum class Model { LeastSquares = 0, Logistic = 1 };

inline double eta_at(double eta, double decay, uint64_t t) {  // trainer.hpp:27-29
  return eta / (1.0 + decay * static_cast<double>(t));
}

// accumulate_gradient, src/trainer.cpp:14-28 (sequential; -ffp-contract=off)
inline void add_grad(Model m, const std::vector<double>& w, const Sample& s, double* g) {
  if (w.size() != s.features.size()) throw std::invalid_argument("gradient dimension mismatch");
  double zz = 0.0;
  for (size_t i = 0; i < w.size(); ++i) zz += w[i] * s.features[i];
  double sc;
  if (m == Model::LeastSquares) {
    sc = zz - s.label;
  } else {
    double mm = -s.label * zz;
    sc = -s.label / (1.0 + std::exp(-mm));
  }
  for (size_t i = 0; i < w.size(); ++i) g[i] += sc * s.features[i];
}

// batch_loss, src/trainer.cpp:41-54
inline double loss_of(Model m, const std::vector<double>& w, const std::vector<Sample>& b) {
  double total = 0.0;
  for (const auto& s : b) {
    double zz = 0.0;
    for (size_t i = 0; i < w.size(); ++i) zz += w[i] * s.features[i];
    if (m == Model::LeastSquares) {
      double e = zz - s.label;
      total += 0.5 * e * e;
    } else {
      total += std::log1p(std::exp(-s.label * zz));
    }
  }
  return total;
}

// sgd_step, src/trainer.cpp:56-61
inline void sgd(std::vector<double>& w, const double* g, uint64_t count, double eta) {
  if (count == 0) throw std::invalid_argument("sgd_step with zero sample count");
  const double sc = eta / static_cast<double>(count);
  for (size_t i = 0; i < w.size(); ++i) w[i] -= sc * g[i];
}

// ---------------------------------------------------------------- collective order
inline std::pair<size_t, size_t> chunk(size_t len, int n, int c) {  // allreduce.cpp:33-37
  return {len * static_cast<size_t>(c) / n, len * static_cast<size_t>(c + 1) / n};
}
// ring_order_reduce, allreduce.cpp:132-148 (== ring_allreduce bit for bit)
inline std::vector<double> ring_sum(const std::vector<std::vector<double>>& in, bool average) {
  const int n = static_cast<int>(in.size());
  const size_t len = in.at(0).size();
  std::vector<double> out(len, 0.0);
  for (int c = 0; c < n; ++c) {
    auto [lo, hi] = chunk(len, n, c);
    for (size_t i = lo; i < hi; ++i) {
      double acc = in[c][i];
      for (int k = 1; k < n; ++k) acc = acc + in[(c + k) % n][i];
      out[i] = acc;
    }
  }
  if (average)
    for (auto& v : out) v /= n;
  return out;
}

// ---------------------------------------------------------------- runtime arithmetic
// split_batch
inline std::vector<int64_t> split_batch(int64_t B, int p) {
  if (p < 1 || B < p) throw std::invalid_argument("split_batch: B < p");
  std::vector<int64_t> out(static_cast<size_t>(p), B / p);
  for (int64_t r = 0; r < B % p; ++r) out[static_cast<size_t>(r)] += 1;
  return out;
}
// k = max(1, ceil(T_a / T_b))
inline int64_t switch_delay(double ta, double tb) {
  if (!(tb > 0)) return 1;
  return std::max<int64_t>(1, static_cast<int64_t>(std::ceil(ta / tb)));
}

// ---------------------------------------------------------------- assignment log
// LogRecord / write_log_file / read_log_file, trainer.hpp:59-90, trainer.cpp:79-142
struct Rec {
  enum Kind { Batch, Topo, Restore } kind = Batch;
  uint64_t t = 0;
  std::string worker;
  std::vector<std::pair<uint64_t, uint64_t>> samples;
  uint64_t version = 0;
  std::vector<std::string> ring;
};

inline std::string log_text(const std::vector<Rec>& recs) {
  std::ostringstream o;
  for (const auto& r : recs) {
    if (r.kind == Rec::Batch) {
      o << "batch " << r.t << " " << r.worker << " " << r.samples.size();
      for (const auto& [e, id] : r.samples) o << " " << e << ":" << id;
      o << "\n";
    } else if (r.kind == Rec::Topo) {
      o << "topo " << r.t << " " << r.version << " " << r.ring.size();
      for (const auto& w : r.ring) o << " " << w;
      o << "\n";
    } else {
      o << "restore " << r.t << "\n";
    }
  }
  return o.str();
}

inline std::vector<Rec> parse_log(const std::string& text) {
  std::vector<Rec> out;
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string tag;
    ls >> tag;
    Rec r;
    size_t n = 0;
    if (tag == "batch") {
      ls >> r.t >> r.worker >> n;
      for (size_t i = 0; i < n; ++i) {
        std::string pr;
        ls >> pr;
        auto c = pr.find(':');
        r.samples.emplace_back(std::stoull(pr.substr(0, c)), std::stoull(pr.substr(c + 1)));
      }
    } else if (tag == "topo") {
      r.kind = Rec::Topo;
      ls >> r.t >> r.version >> n;
      for (size_t i = 0; i < n; ++i) {
        std::string w;
        ls >> w;
        r.ring.push_back(w);
      }
    } else if (tag == "restore") {
      r.kind = Rec::Restore;
      ls >> r.t;
    } else {
      throw std::runtime_error("unknown log record: " + tag);
    }
    out.push_back(std::move(r));
  }
  return out;
}

// effective_log, trainer.cpp:63-77
inline std::vector<Rec> effective(const std::vector<Rec>& raw) {
  std::vector<Rec> out;
  for (const auto& r : raw) {
    if (r.kind == Rec::Restore) {
      std::erase_if(out, [&](const Rec& x) { return x.kind != Rec::Restore && x.t > r.t; });
      continue;
    }
    out.push_back(r);
  }
  return out;
}

// check_coverage, trainer.cpp:144-186
struct Coverage {
  bool ok = false;
  uint64_t full_epochs = 0;
  std::string detail;
};
inline Coverage coverage(const std::vector<Rec>& log, uint64_t N) {
  Coverage c;
  std::map<uint64_t, std::map<uint64_t, int>> per;
  for (const auto& r : log)
    if (r.kind == Rec::Batch)
      for (const auto& [e, id] : r.samples) per[e][id]++;
  if (per.empty()) {
    c.ok = true;
    return c;
  }
  const uint64_t last = per.rbegin()->first;
  uint64_t expect = 0;
  for (const auto& [e, ids] : per) {
    if (e != expect) {
      c.detail = "epoch " + std::to_string(expect) + " missing entirely";
      return c;
    }
    for (const auto& [id, k] : ids) {
      if (k != 1) {
        c.detail = "epoch " + std::to_string(e) + " sample " + std::to_string(id) +
                   " consumed " + std::to_string(k) + " times";
        return c;
      }
      if (id >= N) {
        c.detail = "epoch " + std::to_string(e) + " sample " + std::to_string(id) + " out of range";
        return c;
      }
    }
    if (ids.size() == N)
      c.full_epochs++;
    else if (e != last) {
      c.detail = "epoch " + std::to_string(e) + " incomplete (" + std::to_string(ids.size()) +
                 "/" + std::to_string(N) + ") but a later epoch ran";
      return c;
    }
    ++expect;
  }
  c.ok = true;
  return c;
}

// oracle_replay, trainer.cpp:188-276
inline bool replay(const std::vector<Rec>& log, Model m, const Synth& ds, std::vector<double>& w,
                   double eta, double decay, bool ring_order, std::string* err,
                   uint64_t* batches) {
  const size_t dim = w.size();
  std::map<uint64_t, std::map<std::string, std::vector<std::pair<uint64_t, uint64_t>>>> by_t;
  std::map<uint64_t, std::vector<std::string>> ring_from;
  for (const auto& r : log) {
    if (r.kind == Rec::Batch) {
      auto& v = by_t[r.t][r.worker];
      v.insert(v.end(), r.samples.begin(), r.samples.end());
    } else if (r.kind == Rec::Topo) {
      ring_from[r.t] = r.ring;
    } else {
      *err = "restore marker in effective log";
      return false;
    }
  }
  *batches = 0;
  if (by_t.empty()) return true;
  uint64_t expect = by_t.begin()->first;
  for (const auto& [t, workers] : by_t) {
    if (t != expect) {
      *err = "mini-batch gap at t=" + std::to_string(t);
      return false;
    }
    expect = t + 1;
    std::vector<std::string> ring;
    for (const auto& [from, rg] : ring_from)
      if (from < t) ring = rg;
    if (ring.empty())
      for (const auto& [wk, ids] : workers) ring.push_back(wk);
    for (const auto& [wk, ids] : workers)
      if (std::find(ring.begin(), ring.end(), wk) == ring.end()) {
        *err = "worker " + wk + " logged batch t=" + std::to_string(t) + " outside ring";
        return false;
      }
    std::vector<double> total(dim + 1, 0.0);
    if (ring_order) {
      std::vector<std::vector<double>> vecs;
      for (const auto& wk : ring) {
        std::vector<double> g(dim + 1, 0.0);
        auto it = workers.find(wk);
        if (it != workers.end()) {
          for (const auto& [e, id] : it->second) add_grad(m, w, ds.get(id), g.data());
          g[dim] = static_cast<double>(it->second.size());
        }
        vecs.push_back(std::move(g));
      }
      total = ring_sum(vecs, false);
    } else {
      for (const auto& wk : ring) {
        auto it = workers.find(wk);
        if (it == workers.end()) continue;
        for (const auto& [e, id] : it->second) add_grad(m, w, ds.get(id), total.data());
      }
      double c = 0;
      for (const auto& [wk, ids] : workers) c += static_cast<double>(ids.size());
      total[dim] = c;
    }
    const uint64_t count = static_cast<uint64_t>(total[dim]);
    if (count > 0) sgd(w, total.data(), count, eta_at(eta, decay, t));
    ++*batches;
  }
  return true;
}

}  // namespace orc
