// mpsg_mpsamp.hpp — header-only drop-in for the reference's C++ sampling entry points.
//
// Include this *after* the reference headers (it uses mpsamp::MpsState, BatchPlan, SamplerOptions,
// SampleBatch, RunStats and the exception hierarchy from proj/include/mpsamp/*.hpp) and call
// mpsg_mpsamp::sample_batch / sample_micro_serial where the reference calls
//
//   mpsamp::sample_batch(const MpsState&, const BatchPlan&, const SamplerOptions&, RunStats*)
//                                                         proj/include/mpsamp/sampler.hpp:84-85
//   mpsamp::detail::sample_micro_serial(const MpsState&, uint64_t first, size_t count,
//                                       const SamplerOptions&, uint8_t* rows, RunStats&)
//                                                         proj/include/mpsamp/sampler.hpp:103-104
//
// Same arguments, same validation (MpsState::validate, PrecisionPolicy::validate,
// BatchPlan::normalize run first, exactly as sampler.cpp:166-169), same output layout
// (N x M u8, 0xFF dead) and the C ABI's return codes rethrown as the reference's exceptions
// (errors.hpp:8-27).  The compute runs on the B200 through include/mpsg.h; link libmpsg.so.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "mpsg.h"

namespace mpsg_mpsamp {

[[noreturn]] inline void rethrow(int rc) {
  const std::string msg = std::string("mpsg: ") + mpsg_last_error();
  switch (rc) {
    case MPSG_ERR_CONFIG: throw mpsamp::ConfigError(msg);
    case MPSG_ERR_NUMERIC: throw mpsamp::NumericError(msg);
    case MPSG_ERR_IO: throw mpsamp::IoError(msg);
    default: throw mpsamp::Error(msg);
  }
}

inline void check(int rc) {
  if (rc != MPSG_OK) rethrow(rc);
}

// RAII handle: the compressed MPS resident on the listed B200s (data-parallel replicas).
class DeviceState {
 public:
  DeviceState(const mpsamp::MpsState& mps, const mpsamp::PrecisionPolicy& policy,
              const std::vector<int>& devices = {}, const mpsg_options* opts = nullptr)
      : m_(mps.num_sites), d_(mps.phys_dim) {
    mps.validate();
    policy.validate();
    std::vector<uint64_t> bonds(mps.bond_dims.begin(), mps.bond_dims.end());
    std::vector<const double*> g(m_), l(m_);
    for (size_t i = 0; i < m_; ++i) {
      // std::complex<double> is layout-compatible with double[2] (interleaved re, im)
      g[i] = reinterpret_cast<const double*>(mps.gammas[i].data());
      l[i] = mps.lambdas[i].data();
    }
    const mpsg_mps_view view{m_, d_, bonds.data(), g.data(), l.data()};
    const mpsg_policy pol{static_cast<int>(policy.compute), static_cast<int>(policy.storage),
                          static_cast<int>(policy.scaling)};
    mpsg_handle h = nullptr;
    check(mpsg_create(&view, &pol, opts, devices.empty() ? nullptr : devices.data(),
                      static_cast<int>(devices.size()), &h));
    h_.reset(h);
  }
  size_t num_sites() const { return m_; }
  size_t phys_dim() const { return d_; }
  mpsg_handle handle() const { return h_.get(); }

 private:
  struct Del {
    void operator()(mpsg_handle h) const { mpsg_destroy(h); }
  };
  size_t m_, d_;
  std::unique_ptr<mpsg_handle_s, Del> h_;
};

inline void merge_stats(const mpsg_stats& s, const std::vector<double>& site, mpsamp::RunStats& rs) {
  rs.flops.contraction_macs += s.contraction_macs;
  rs.flops.measure_weight_macs += s.measure_weight_macs;
  rs.flops.displacement_macs += s.displacement_macs;
  rs.flops.measure_pipeline_ops += s.measure_pipeline_ops;
  rs.dead_samples += s.dead_samples;
  if (rs.site_seconds.size() < site.size()) rs.site_seconds.resize(site.size(), 0.0);
  for (size_t i = 0; i < site.size(); ++i) rs.site_seconds[i] += site[i];
  rs.total_seconds += s.seconds;
}

// detail::sample_micro_serial on a resident DeviceState (sampler.cpp:129-162).
inline void sample_micro_serial(const DeviceState& st, uint64_t first, size_t count,
                                const mpsamp::SamplerOptions& opts, uint8_t* rows,
                                mpsamp::RunStats& stats) {
  if (opts.schedule || opts.site_transform)
    throw mpsamp::ConfigError("mpsg: bond schedules / site transforms are not on the GPU path");
  std::vector<double> site(st.num_sites(), 0.0);
  mpsg_stats s{};
  s.site_seconds = site.data();
  check(mpsg_sample(st.handle(), opts.seed, first, count, rows, &s));
  merge_stats(s, site, stats);
}

// mpsamp::sample_batch (sampler.cpp:164-205) on the B200.
inline mpsamp::SampleBatch sample_batch(const mpsamp::MpsState& mps_in, const mpsamp::BatchPlan& plan_in,
                                        const mpsamp::SamplerOptions& opts_in,
                                        mpsamp::RunStats* stats_out = nullptr,
                                        const std::vector<int>& devices = {}) {
  mps_in.validate();
  opts_in.policy.validate();
  mpsamp::BatchPlan plan = plan_in;
  plan.normalize();
  if (opts_in.site_transform)
    throw mpsamp::ConfigError("mpsg: site transforms are not on the GPU path");
  // a BondSchedule truncates the chain first, with the reference's own apply_schedule
  // (sampler.cpp:173-176)
  mpsamp::MpsState truncated;
  const mpsamp::MpsState* state = &mps_in;
  if (opts_in.schedule) {
    truncated = mpsamp::apply_schedule(mps_in, *opts_in.schedule);
    state = &truncated;
  }
  const mpsamp::MpsState& mps = *state;
  mpsamp::SamplerOptions opts = opts_in;
  opts.schedule.reset();
  mpsg_options o{};
  o.record_site_times = stats_out ? 1 : 0;
  DeviceState st(mps, opts.policy, devices, &o);
  mpsamp::SampleBatch b;
  b.num_samples = plan.total_samples;
  b.num_sites = mps.num_sites;
  b.phys_dim = mps.phys_dim;
  b.seed = opts.seed;
  b.outcomes.assign(plan.total_samples * mps.num_sites, mpsamp::kDeadOutcome);
  mpsamp::RunStats stats;
  sample_micro_serial(st, 0, plan.total_samples, opts, b.outcomes.data(), stats);
  if (stats_out) *stats_out = std::move(stats);
  return b;
}

// run_serial / run_data_parallel (parallel.hpp:24-52) on an MPSB file: the file is streamed into
// the compressed device state (mpsg_create_from_file) and sampled on `p1` B200s (devices 0..p1-1
// unless given).  Returns the batch and merged RunStats like ParallelResult (no CommStats: the
// data path has no collective).  from_storage: keep only the header and Lambda and re-read the site
// payloads from the file on every pass (mpsg_create_from_file_streamed, the reference's SiteStream)
// -- for chains beyond device and host memory.
inline mpsamp::SampleBatch run_data_parallel_file(const std::string& mps_path,
                                                  const mpsamp::BatchPlan& plan_in, size_t p1,
                                                  const mpsamp::SamplerOptions& opts,
                                                  mpsamp::RunStats* stats_out = nullptr,
                                                  std::vector<int> devices = {},
                                                  bool from_storage = false) {
  if (p1 < 1) throw mpsamp::ConfigError("data parallel needs p1 >= 1");
  opts.policy.validate();
  if (opts.site_transform || opts.schedule)
    throw mpsamp::ConfigError("mpsg: schedules / site transforms are not on the file path");
  mpsamp::BatchPlan plan = plan_in;
  plan.normalize();
  if (devices.empty())
    for (size_t i = 0; i < p1; ++i) devices.push_back(static_cast<int>(i));
  const mpsg_policy pol{static_cast<int>(opts.policy.compute), static_cast<int>(opts.policy.storage),
                        static_cast<int>(opts.policy.scaling)};
  mpsg_options o{};
  o.record_site_times = stats_out ? 1 : 0;
  mpsg_handle h = nullptr;
  check((from_storage ? mpsg_create_from_file_streamed : mpsg_create_from_file)(
      mps_path.c_str(), &pol, &o, devices.data(), static_cast<int>(devices.size()), &h));
  std::unique_ptr<mpsg_handle_s, void (*)(mpsg_handle)> guard(h, mpsg_destroy);
  // chain shape from the file header (read_mps_info, mps_io.cpp:212-254)
  mpsamp::MpsFileInfo info = mpsamp::read_mps_info(mps_path);
  mpsamp::SampleBatch b;
  b.num_samples = plan.total_samples;
  b.num_sites = info.num_sites;
  b.phys_dim = info.phys_dim;
  b.seed = opts.seed;
  b.outcomes.assign(plan.total_samples * info.num_sites, mpsamp::kDeadOutcome);
  std::vector<double> site(info.num_sites, 0.0);
  mpsg_stats s{};
  s.site_seconds = site.data();
  check(mpsg_sample(h, opts.seed, 0, plan.total_samples, b.outcomes.data(), &s));
  if (stats_out) merge_stats(s, site, *stats_out);
  return b;
}

}  // namespace mpsg_mpsamp
