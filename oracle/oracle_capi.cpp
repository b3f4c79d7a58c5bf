// ORACLE — TEST INFRASTRUCTURE ONLY (see restate.hpp header).
// liboracle.so: the C API of capi_common.inc over the independent restatement
// (restate.hpp), plus runtime arithmetic the reference only specifies in prose.
#include <fstream>
#include <memory>
#include <sstream>

#include "job_driver.hpp"
#include "restate.hpp"

namespace {

using LeaseT = orc::Leases;
using DataT = orc::Synth;

std::string slurp(const char* path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error(std::string("cannot open assignment log: ") + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

struct TrainT {
  static void add_grad(orc::Model m, const std::vector<double>& w, const orc::Sample& s, double* g) {
    orc::add_grad(m, w, s, g);
  }
  static double loss(orc::Model m, const std::vector<double>& w, const std::vector<orc::Sample>& b) {
    return orc::loss_of(m, w, b);
  }
  static void sgd(std::vector<double>& w, const double* g, uint64_t count, double eta) {
    orc::sgd(w, g, count, eta);
  }
  static std::vector<double> ring_sum(const std::vector<std::vector<double>>& v) {
    return orc::ring_sum(v, false);
  }
  static int coverage_file(const char* path, uint64_t n, uint64_t* fe, std::string* d) {
    auto c = orc::coverage(orc::effective(orc::parse_log(slurp(path))), n);
    *fe = c.full_epochs;
    *d = c.detail;
    return c.ok ? 1 : 0;
  }
  static int replay_file(const char* path, int model, const DataT& ds, std::vector<double>& w,
                         double eta, double decay, bool ring, std::string* e, uint64_t* batches) {
    auto log = orc::effective(orc::parse_log(slurp(path)));
    return orc::replay(log, model == 0 ? orc::Model::LeastSquares : orc::Model::Logistic, ds, w,
                       eta, decay, ring, e, batches)
               ? 1
               : 0;
  }
};

std::unique_ptr<DataT> make_data(uint64_t size, int dim, uint64_t seed, double noise, bool sign) {
  orc::SynthSpec s{size, dim, seed, noise, sign};
  return std::make_unique<DataT>(s);
}
std::unique_ptr<LeaseT> make_lease(uint64_t size, int d, uint64_t seed, const std::string& loc) {
  return std::make_unique<LeaseT>(size, d, seed, loc);
}

}  // namespace

#define EDL_PFX(name) or_##name
#include "capi_common.inc"

extern "C" {
int or_split_batch(int64_t B, int p, int64_t* out) {
  try {
    auto v = orc::split_batch(B, p);
    std::copy(v.begin(), v.end(), out);
    return 0;
  } catch (const std::invalid_argument&) {
    return 2;
  }
}
int64_t or_switch_delay(double ta, double tb) { return orc::switch_delay(ta, tb); }
double or_eta_at(double eta, double decay, uint64_t t) { return orc::eta_at(eta, decay, t); }
int or_default_partition_count(int w) { return orc::default_partition_count(w); }
}
