// Differential check of integration/b200_shard_manager.hpp against the reference's own
// edl::ShardManager (compiled from /root/reference/proj/src/datapipeline.cpp): random
// scripts of register / next_shard / report_progress / reclaim / reclaim_at /
// reclaim_missing / snapshot / restore on both, every result and the snapshot bytes
// compared.  Prints "SHIM OK <ops>" or the first mismatch.  Test infrastructure
// (tests/test_integration_shim.py builds and runs it).
#include <cstdio>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "b200_shard_manager.hpp"

using namespace edl;

static std::string show(const ShardManager::NextResult& r) {
  char b[128];
  if (auto* s = std::get_if<Shard>(&r.value))
    std::snprintf(b, sizeof b, "%d shard %u %s %lu %lu @%lu", int(r.status), s->meta.index,
                  s->meta.locator.c_str(), (unsigned long)s->meta.offset,
                  (unsigned long)s->meta.length, (unsigned long)s->resume_offset);
  else if (auto* e = std::get_if<EpochEnd>(&r.value))
    std::snprintf(b, sizeof b, "%d epoch_end %lu", int(r.status), (unsigned long)e->epoch);
  else
    std::snprintf(b, sizeof b, "%d pending", int(r.status));
  return b;
}

int main() {
  long ops = 0;
  for (int seed = 0; seed < 40; ++seed) {
    std::mt19937 rng(seed);
    const uint64_t size = 1000 + 97 * seed;
    const int d = 8 + seed % 24;
    ShardManager ref(size, d, 1234 + seed, "synthetic:1");
    B200ShardManager b2(size, d, 1234 + seed, "synthetic:1");
    std::vector<std::string> ws = {"w0", "w1", "w2", "w3"};
    for (int i = 0; i < 2; ++i) {
      ref.register_worker(ws[i]);
      b2.register_worker(ws[i]);
    }
    std::vector<std::pair<uint32_t, uint64_t>> held;  // (partition, length) last handed out
    for (int k = 0; k < 500; ++k, ++ops) {
      const std::string& w = ws[rng() % ws.size()];
      const int op = rng() % 100;
      std::string a, b;
      if (op < 45) {
        auto r1 = ref.next_shard(w);
        auto r2 = b2.next_shard(w);
        a = show(r1);
        b = show(r2);
        if (auto* s = std::get_if<Shard>(&r1.value)) held.push_back({s->meta.index, s->meta.length});
      } else if (op < 75 && !held.empty()) {
        const auto [p, len] = held[rng() % held.size()];
        const uint64_t off = rng() % (len + 1);
        a = std::to_string(int(ref.report_progress({w, p, off})));
        b = std::to_string(int(b2.report_progress({w, p, off})));
      } else if (op < 82) {
        ref.register_worker(w);
        b2.register_worker(w);
      } else if (op < 88) {
        ref.reclaim(w);
        b2.reclaim(w);
      } else if (op < 92) {
        auto s1 = ref.worker_shards(w);
        auto s2 = b2.worker_shards(w);
        a = std::to_string(s1.size());
        b = std::to_string(s2.size());
        if (s1 == s2 && !s1.empty()) {
          ref.reclaim_at(w, s1);
          b2.reclaim_at(w, s2);
        }
      } else if (op < 95) {
        std::set<std::string> live = {ws[0], w};
        ref.reclaim_missing(live);
        b2.reclaim_missing(live);
      } else {
        const auto snap = ref.snapshot();
        if (snap != b2.snapshot()) {
          std::printf("SHIM MISMATCH seed %d op %d: snapshot bytes\n", seed, k);
          return 1;
        }
        ShardManager r3(size, d, 1, "synthetic:1");
        B200ShardManager b3(size, d, 1, "synthetic:1");
        a = std::to_string(int(r3.restore(snap)));
        b = std::to_string(int(b3.restore(snap)));
        if (r3.snapshot() != b3.snapshot()) a += "x";
      }
      if (a != b) {
        std::printf("SHIM MISMATCH seed %d op %d: reference '%s' vs b200 '%s'\n", seed, k,
                    a.c_str(), b.c_str());
        return 1;
      }
    }
    if (ref.snapshot() != b2.snapshot() || ref.epoch() != b2.epoch() ||
        ref.cursor() != b2.cursor() || ref.in_flight_count() != b2.in_flight_count() ||
        ref.reclaimed_count() != b2.reclaimed_count()) {
      std::printf("SHIM MISMATCH seed %d: final state\n", seed);
      return 1;
    }
  }
  std::printf("SHIM OK %ld\n", ops);
  return 0;
}
