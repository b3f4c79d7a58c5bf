// Reference-side binding (what an EDL maintainer adds to /root/reference/proj to use the B200
// library): a drop-in for edl::ShardManager (include/edl/datapipeline.hpp:58-127) over the
// C ABI of include/edl_b200.h.  Same constructor, methods, result types and status values;
// the snapshot bytes are the reference's layout (datapipeline.cpp:115-178).
// Compiled against the reference's own header and checked against its ShardManager by
// tests/test_integration_shim.py (integration/shim_check.cpp).
#pragma once

#include <cstdint>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "edl/datapipeline.hpp"
#include "edl_b200.h"

namespace edl {

class B200ShardManager {
 public:
  using NextResult = ShardManager::NextResult;

  B200ShardManager(uint64_t dataset_size, int partitions, uint64_t seed, std::string locator)
      : loc_(std::move(locator)) {
    if (edl_lease_create(dataset_size, partitions, seed, loc_.c_str(), &h_) != EDL_OK)
      throw std::invalid_argument(edl_last_error());
  }
  ~B200ShardManager() { edl_lease_destroy(h_); }
  B200ShardManager(const B200ShardManager&) = delete;
  B200ShardManager& operator=(const B200ShardManager&) = delete;

  void register_worker(const std::string& w) { edl_lease_register(h_, w.c_str()); }
  void unregister_worker(const std::string& w) { edl_lease_unregister(h_, w.c_str()); }
  bool is_registered(const std::string& w) const { return edl_lease_is_registered(h_, w.c_str()); }

  NextResult next_shard(const std::string& w) {
    EdlNextShard n{};
    const int rc = edl_lease_next(h_, w.c_str(), &n);
    if (rc != EDL_OK) return {status(rc), ShardPending{}};
    if (n.kind == EDL_NEXT_SHARD)
      return {PipeStatus::Ok, Shard{meta(n.meta), n.resume_offset}};
    if (n.kind == EDL_NEXT_EPOCH_END) return {PipeStatus::Ok, EpochEnd{n.epoch}};
    return {PipeStatus::Ok, ShardPending{}};
  }
  PipeStatus report_progress(const ProgressRecord& r) {
    return status(edl_lease_report(h_, r.worker.c_str(), r.partition, r.next_sample_offset));
  }
  void reclaim(const std::string& w) { edl_lease_reclaim(h_, w.c_str()); }
  void reclaim_at(const std::string& w, const std::vector<std::pair<uint32_t, uint64_t>>& at) {
    std::vector<uint32_t> p;
    std::vector<uint64_t> o;
    for (const auto& [pi, oi] : at) {
      p.push_back(pi);
      o.push_back(oi);
    }
    edl_lease_reclaim_at(h_, w.c_str(), p.data(), o.data(), p.size());
  }
  void reclaim_missing(const std::set<std::string>& live) {
    std::vector<const char*> v;
    for (const auto& s : live) v.push_back(s.c_str());
    edl_lease_reclaim_missing(h_, v.data(), v.size());
  }
  PartitionMeta partition_meta(uint32_t index) const {
    EdlPartitionMeta m{};
    edl_lease_partition_meta(h_, index, &m);
    return meta(m);
  }
  std::vector<uint8_t> snapshot() const {
    size_t n = 0;
    edl_lease_snapshot(h_, nullptr, 0, &n);
    std::vector<uint8_t> b(n);
    edl_lease_snapshot(h_, b.data(), n, &n);
    return b;
  }
  PipeStatus restore(std::span<const uint8_t> snap) {
    const int rc = edl_lease_restore(h_, snap.data(), snap.size());
    if (rc == EDL_ETRUNCATED) throw std::runtime_error("truncated payload");  // bytes.hpp:112
    return status(rc);
  }
  uint64_t epoch() const { return edl_lease_epoch(h_); }
  uint64_t epochs_completed() const { return edl_lease_epochs_completed(h_); }
  uint64_t cursor() const { return edl_lease_cursor(h_); }
  size_t reclaimed_count() const { return edl_lease_reclaimed_count(h_); }
  size_t in_flight_count() const { return edl_lease_in_flight_count(h_); }
  std::vector<uint32_t> permutation() const {
    std::vector<uint32_t> p(edl_lease_permutation(h_, nullptr, 0));
    edl_lease_permutation(h_, p.data(), p.size());
    return p;
  }
  std::vector<std::pair<uint32_t, uint64_t>> worker_shards(const std::string& w) const {
    const size_t n = edl_lease_worker_shards(h_, w.c_str(), nullptr, nullptr, 0);
    std::vector<uint32_t> p(n);
    std::vector<uint64_t> o(n);
    edl_lease_worker_shards(h_, w.c_str(), p.data(), o.data(), n);
    std::vector<std::pair<uint32_t, uint64_t>> out;
    for (size_t i = 0; i < n; ++i) out.emplace_back(p[i], o[i]);
    return out;
  }

 private:
  static PipeStatus status(int rc) {  // EDL_* -> PipeStatus (same numbering, edl_b200.h)
    switch (rc) {
      case EDL_OK: return PipeStatus::Ok;
      case EDL_UNKNOWN_WORKER: return PipeStatus::UnknownWorker;
      case EDL_STALE_SHARD: return PipeStatus::StaleShard;
      default: return PipeStatus::ShapeMismatch;
    }
  }
  PartitionMeta meta(const EdlPartitionMeta& m) const {
    return PartitionMeta{m.index, loc_, m.offset, m.length};
  }
  EdlLeaseManager* h_ = nullptr;
  std::string loc_;
};

}  // namespace edl
