// Partition leasing (see lease.hpp).  Host C++: the lease state machine is control
// plane (88 ns/op in the reference) and stays on the CPU; its output — runs
// of contiguous sample ids — feeds the device gather kernel (dataset.cu).
#include "lease.hpp"

#include <algorithm>
#include <cstring>
#include <numeric>
#include <sstream>
#include <stdexcept>

namespace edl {

int default_partitions(int w) { return w * 4 > 64 ? w * 4 : 64; }

LeaseManager::LeaseManager(uint64_t dataset_size, int partitions, uint64_t seed,
                           std::string locator)
    : size_(dataset_size), parts_(partitions), locator_(std::move(locator)), rng_(seed) {
  new_epoch_order();
}

// datapipeline.cpp:19-24: iota + std::shuffle with the persistent engine
void LeaseManager::new_epoch_order() {
  perm_.resize(static_cast<size_t>(parts_));
  std::iota(perm_.begin(), perm_.end(), 0u);
  std::shuffle(perm_.begin(), perm_.end(), rng_);
  cursor_ = 0;
}

// datapipeline.cpp:34-41
PartMeta LeaseManager::meta(uint32_t index) const {
  PartMeta m;
  m.index = index;
  const uint64_t d = static_cast<uint64_t>(parts_);
  m.offset = size_ * index / d;
  m.length = size_ * (index + 1) / d - m.offset;
  return m;
}

// datapipeline.cpp:43-62: reclaimed FIFO, then the permutation, then Pending while
// anything is in flight, else EpochEnd + a fresh permutation.
Lease LeaseManager::next(const std::string& worker) {
  Lease out;
  if (!members_.count(worker)) {
    out.status = LeaseStatus::UnknownWorker;
    return out;
  }
  if (!returned_.empty()) {
    const auto [part, off] = returned_.front();
    returned_.pop_front();
    held_[part] = Holder{worker, off};
    out.kind = LeaseKind::Shard;
    out.meta = meta(part);
    out.resume = off;
    return out;
  }
  if (cursor_ < static_cast<uint64_t>(parts_)) {
    const uint32_t part = perm_[cursor_++];
    held_[part] = Holder{worker, 0};
    out.kind = LeaseKind::Shard;
    out.meta = meta(part);
    return out;
  }
  if (!held_.empty()) return out;  // Pending
  out.kind = LeaseKind::EpochEnd;
  out.epoch = epoch_++;
  ++completed_;
  new_epoch_order();
  return out;
}

// datapipeline.cpp:64-71
LeaseStatus LeaseManager::progress(const std::string& worker, uint32_t part, uint64_t off) {
  if (!members_.count(worker)) return LeaseStatus::UnknownWorker;
  auto it = held_.find(part);
  if (it == held_.end() || it->second.worker != worker) return LeaseStatus::StaleShard;
  it->second.offset = off;
  if (off >= meta(part).length) held_.erase(it);
  return LeaseStatus::Ok;
}

// datapipeline.cpp:73-84 (ascending partition index, fully consumed shards vanish)
void LeaseManager::reclaim(const std::string& worker) {
  for (auto it = held_.begin(); it != held_.end();) {
    if (it->second.worker != worker) {
      ++it;
      continue;
    }
    if (it->second.offset < meta(it->first).length) returned_.emplace_back(it->first, it->second.offset);
    it = held_.erase(it);
  }
}

// datapipeline.cpp:86-93
void LeaseManager::reclaim_at(const std::string& worker,
                              const std::vector<std::pair<uint32_t, uint64_t>>& at) {
  for (const auto& [part, off] : at) {
    auto it = held_.find(part);
    if (it != held_.end() && it->second.worker == worker) it->second.offset = off;
  }
  reclaim(worker);
}

// datapipeline.cpp:95-104
void LeaseManager::reclaim_missing(const std::set<std::string>& live) {
  std::vector<std::string> gone;
  std::copy_if(members_.begin(), members_.end(), std::back_inserter(gone),
               [&](const std::string& w) { return live.count(w) == 0; });
  for (const auto& w : gone) {
    reclaim(w);
    members_.erase(w);
  }
}

std::vector<std::pair<uint32_t, uint64_t>> LeaseManager::held_by(const std::string& w) const {
  std::vector<std::pair<uint32_t, uint64_t>> out;
  for (const auto& [part, h] : held_)
    if (h.worker == w) out.emplace_back(part, h.offset);
  return out;
}

namespace {

// Little-endian codec with the reference's field widths (include/edl/bytes.hpp:14-51).
struct Writer {
  std::vector<uint8_t> b;
  template <class T>
  void pod(T v) {
    const auto* p = reinterpret_cast<const uint8_t*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  void text(const std::string& s) {
    pod<uint32_t>(static_cast<uint32_t>(s.size()));
    b.insert(b.end(), s.begin(), s.end());
  }
};

struct Reader {
  const uint8_t* p;
  size_t n, at = 0;
  void need(size_t k) {
    if (at + k > n) throw std::runtime_error("truncated payload");
  }
  template <class T>
  T pod() {
    need(sizeof(T));
    T v;
    std::memcpy(&v, p + at, sizeof(T));
    at += sizeof(T);
    return v;
  }
  std::string text() {
    const uint32_t k = pod<uint32_t>();
    need(k);
    std::string s(reinterpret_cast<const char*>(p + at), k);
    at += k;
    return s;
  }
};

}  // namespace

// Field order of datapipeline.cpp:115-142.
std::vector<uint8_t> LeaseManager::snapshot() const {
  Writer w;
  w.pod<uint64_t>(size_);
  w.pod<int64_t>(parts_);
  w.text(locator_);
  w.pod<uint64_t>(epoch_);
  w.pod<uint64_t>(completed_);
  w.pod<uint64_t>(cursor_);
  w.pod<uint64_t>(perm_.size());
  for (uint32_t v : perm_) w.pod<uint32_t>(v);
  w.pod<uint64_t>(returned_.size());
  for (const auto& [part, off] : returned_) {
    w.pod<uint32_t>(part);
    w.pod<uint64_t>(off);
  }
  w.pod<uint64_t>(held_.size());
  for (const auto& [part, h] : held_) {
    w.pod<uint32_t>(part);
    w.text(h.worker);
    w.pod<uint64_t>(h.offset);
  }
  w.pod<uint64_t>(members_.size());
  for (const auto& m : members_) w.text(m);
  std::ostringstream rs;
  rs << rng_;
  w.text(rs.str());
  return std::move(w.b);
}

// datapipeline.cpp:144-178
LeaseStatus LeaseManager::restore(const uint8_t* data, size_t len) {
  Reader r{data, len};
  const uint64_t size = r.pod<uint64_t>();
  const int parts = static_cast<int>(r.pod<int64_t>());
  if (size != size_ || parts != parts_) return LeaseStatus::ShapeMismatch;
  locator_ = r.text();
  epoch_ = r.pod<uint64_t>();
  completed_ = r.pod<uint64_t>();
  cursor_ = r.pod<uint64_t>();
  perm_.resize(r.pod<uint64_t>());
  for (auto& v : perm_) v = r.pod<uint32_t>();
  returned_.clear();
  for (uint64_t i = 0, k = r.pod<uint64_t>(); i < k; ++i) {
    const uint32_t part = r.pod<uint32_t>();
    returned_.emplace_back(part, r.pod<uint64_t>());
  }
  held_.clear();
  for (uint64_t i = 0, k = r.pod<uint64_t>(); i < k; ++i) {
    const uint32_t part = r.pod<uint32_t>();
    Holder h;
    h.worker = r.text();
    h.offset = r.pod<uint64_t>();
    held_[part] = std::move(h);
  }
  members_.clear();
  for (uint64_t i = 0, k = r.pod<uint64_t>(); i < k; ++i) members_.insert(r.text());
  std::istringstream rs(r.text());
  rs >> rng_;
  return LeaseStatus::Ok;
}

}  // namespace edl
