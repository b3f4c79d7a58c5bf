// Partition leasing: the leader-owned dynamic data assignment of EDL (§4.3).
//
// Drop-in for edl::ShardManager (include/edl/datapipeline.hpp:58-127,
// src/datapipeline.cpp:13-178): the dataset is tiled into d partitions; each epoch
// hands out a fresh std::mt19937_64 + std::shuffle permutation on demand, reclaimed
// partial partitions first; progress is tracked at sample-offset granularity.  The
// permutation stream, hand-out order and snapshot bytes are identical to the
// reference's (tests/test_lease_parity.py pins this against the reference's own output).
#pragma once

#include <cstdint>
#include <deque>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

namespace edl {

struct PartMeta {
  uint32_t index = 0;
  uint64_t offset = 0;
  uint64_t length = 0;
};

enum class LeaseKind { Shard = 0, EpochEnd = 1, Pending = 2 };
enum class LeaseStatus { Ok = 0, UnknownWorker = 6, StaleShard = 7, ShapeMismatch = 8 };

struct Lease {
  LeaseStatus status = LeaseStatus::Ok;
  LeaseKind kind = LeaseKind::Pending;
  PartMeta meta;
  uint64_t resume = 0;
  uint64_t epoch = 0;  // EpochEnd: the epoch that just completed
};

int default_partitions(int max_expected_workers);  // max(4W, 64), datapipeline.cpp:9-11

class LeaseManager {
 public:
  LeaseManager(uint64_t dataset_size, int partitions, uint64_t seed, std::string locator);

  void enroll(const std::string& worker) { members_.insert(worker); }
  void retire(const std::string& worker) { members_.erase(worker); }
  bool enrolled(const std::string& worker) const { return members_.count(worker) != 0; }

  Lease next(const std::string& worker);
  LeaseStatus progress(const std::string& worker, uint32_t part, uint64_t next_offset);
  void reclaim(const std::string& worker);
  void reclaim_at(const std::string& worker, const std::vector<std::pair<uint32_t, uint64_t>>& at);
  void reclaim_missing(const std::set<std::string>& live);
  std::vector<std::pair<uint32_t, uint64_t>> held_by(const std::string& worker) const;
  PartMeta meta(uint32_t index) const;

  std::vector<uint8_t> snapshot() const;
  // Throws std::runtime_error("truncated payload") on a short buffer (bytes.hpp:112).
  LeaseStatus restore(const uint8_t* data, size_t len);

  uint64_t epoch() const { return epoch_; }
  uint64_t epochs_completed() const { return completed_; }
  uint64_t cursor() const { return cursor_; }
  const std::vector<uint32_t>& permutation() const { return perm_; }
  size_t reclaimed_count() const { return returned_.size(); }
  size_t in_flight_count() const { return held_.size(); }
  uint64_t dataset_size() const { return size_; }
  int partitions() const { return parts_; }

 private:
  void new_epoch_order();

  struct Holder {
    std::string worker;
    uint64_t offset = 0;
  };
  uint64_t size_;
  int parts_;
  std::string locator_;
  std::mt19937_64 rng_;
  uint64_t epoch_ = 0;
  uint64_t completed_ = 0;
  uint64_t cursor_ = 0;
  std::vector<uint32_t> perm_;
  std::deque<std::pair<uint32_t, uint64_t>> returned_;
  std::map<uint32_t, Holder> held_;
  std::set<std::string> members_;
};

}  // namespace edl
