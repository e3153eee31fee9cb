// TEST INFRASTRUCTURE: builds the drop-in adapter (include/mpsg_mpsamp.hpp) against the
// reference's own headers and library, exactly as a maintainer would, and checks it.
//   adapter_test cpu  -> validation/error mapping only (no GPU needed)
//   adapter_test gpu  -> c1 = random_mps(16, 32, 4, 42) through mpsg_mpsamp::sample_batch (AUTO at
//                        compute F64 = PRECISE: the caller's Gamma to ~2^-23), compared with
//                        mpsamp::sample_batch on the same MPS and seed (0 strings may differ); and
//                        MPSG_MODE_SPLIT against the reference on the decoded Gamma (0 may differ)
#include <cstdio>
#include <cstring>

#include "mpsamp/errors.hpp"
#include "mpsamp/mps.hpp"
#include "mpsamp/mps_io.hpp"
#include "mpsamp/sampler.hpp"
#include "mpsg_mpsamp.hpp"

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  mpsamp::MpsState mps = mpsamp::random_mps(16, 32, 4, 42);
  mpsamp::SamplerOptions opts;
  opts.seed = 7;
  opts.policy.scaling = mpsamp::ScalingMode::PerSampleMax;
  // 1) reference validation runs first: TF32 storage -> ConfigError (precision.cpp:98-102)
  {
    mpsamp::SamplerOptions bad = opts;
    bad.policy.storage = mpsamp::Precision::TF32;
    try {
      mpsg_mpsamp::sample_batch(mps, mpsamp::BatchPlan::simple(10), bad);
      std::printf("FAIL: no ConfigError\n");
      return 1;
    } catch (const mpsamp::ConfigError&) {
    }
  }
  if (!gpu) {
    // without a B200 the GPU call must fail loudly (mpsamp::Error), never fall back to CPU
    try {
      mpsg_mpsamp::sample_batch(mps, mpsamp::BatchPlan::simple(10), opts);
      if (mpsg_device_count() == 0) {
        std::printf("FAIL: sampled without a device\n");
        return 1;
      }
    } catch (const mpsamp::Error& e) {
      std::printf("ok (no device): %s\n", e.what());
    }
    return 0;
  }
  mpsamp::RunStats st;
  mpsamp::SampleBatch got = mpsg_mpsamp::sample_batch(mps, mpsamp::BatchPlan::simple(1000), opts, &st);
  mpsamp::SampleBatch want = mpsamp::sample_batch(mps, mpsamp::BatchPlan::simple(1000), opts);
  size_t diff = 0;
  for (size_t n = 0; n < 1000; ++n)
    diff += std::memcmp(&got.outcomes[n * 16], &want.outcomes[n * 16], 16) != 0;
  // schedule through the adapter == the reference's truncation sampled directly
  {
    mpsamp::SamplerOptions so = opts;
    so.schedule = mpsamp::BondSchedule::full(mps.bond_dims, 32);
    so.schedule->per_site_chi[5] = 20;
    mpsamp::SampleBatch a = mpsg_mpsamp::sample_batch(mps, mpsamp::BatchPlan::simple(300), so);
    mpsamp::SampleBatch c = mpsg_mpsamp::sample_batch(mpsamp::apply_schedule(mps, *so.schedule),
                                                      mpsamp::BatchPlan::simple(300), opts);
    if (a.outcomes != c.outcomes) {
      std::printf("FAIL: scheduled sampling differs\n");
      return 1;
    }
  }
  // file executor: save with the reference, run through the adapter
  {
    mpsamp::save_mps(mps, "/tmp/mpsg_adapter_c1.mpsb", mpsamp::Precision::F64);
    mpsamp::SampleBatch f = mpsg_mpsamp::run_data_parallel_file("/tmp/mpsg_adapter_c1.mpsb",
                                                                mpsamp::BatchPlan::simple(1000), 1, opts);
    if (f.outcomes != got.outcomes) {
      std::printf("FAIL: file executor differs from in-memory\n");
      return 1;
    }
    // the same file streamed from storage every pass (mpsg_create_from_file_streamed)
    mpsamp::SampleBatch fs = mpsg_mpsamp::run_data_parallel_file("/tmp/mpsg_adapter_c1.mpsb",
                                                                 mpsamp::BatchPlan::simple(1000), 1, opts,
                                                                 nullptr, {}, true);
    if (fs.outcomes != got.outcomes) {
      std::printf("FAIL: storage-streamed file executor differs from in-memory\n");
      return 1;
    }
  }
  // MPSG_MODE_SPLIT (the fp16 format's decoded-Gamma contract): identical strings against the
  // reference run on the decoded Gamma, and the count against the original Gamma recorded
  size_t diff_split_dec = 0, diff_split_orig = 0;
  {
    mpsg_options o{};
    o.mode = MPSG_MODE_SPLIT;
    mpsg_mpsamp::DeviceState ds(mps, opts.policy, {}, &o);
    mpsamp::MpsState dec = mps;
    for (size_t i = 0; i < mps.num_sites; ++i)
      mpsg_mpsamp::check(mpsg_decoded_gamma(ds.handle(), i, reinterpret_cast<double*>(dec.gammas[i].data())));
    std::vector<uint8_t> rows(1000 * 16);
    mpsamp::RunStats rs;
    mpsg_mpsamp::sample_micro_serial(ds, 0, 1000, opts, rows.data(), rs);
    mpsamp::SampleBatch ref_dec = mpsamp::sample_batch(dec, mpsamp::BatchPlan::simple(1000), opts);
    for (size_t n = 0; n < 1000; ++n) {
      diff_split_dec += std::memcmp(&rows[n * 16], &ref_dec.outcomes[n * 16], 16) != 0;
      diff_split_orig += std::memcmp(&rows[n * 16], &want.outcomes[n * 16], 16) != 0;
    }
  }
  // one JSON line (profiles/r2_parity/adapter_c1.json): the default (AUTO -> PRECISE at F64) against the
  // caller's original Gamma, SPLIT against the decoded and the original Gamma
  std::printf("{\"case\": \"c1 random_mps(16, 32, 4, 42), 1000 samples, seed 7, F64 + PerSampleMax\", "
              "\"auto_mode\": %d, \"auto_vs_original_strings_differing\": %zu, "
              "\"split_vs_decoded_strings_differing\": %zu, \"split_vs_original_strings_differing\": %zu, "
              "\"contraction_macs\": %llu, \"reference_contraction_macs\": %llu}\n",
              mpsg_mode(mpsg_mpsamp::DeviceState(mps, opts.policy).handle()), diff, diff_split_dec, diff_split_orig,
              static_cast<unsigned long long>(st.flops.contraction_macs), 45600000ull);
  return (st.flops.contraction_macs == 45600000ull && diff == 0 && diff_split_dec == 0) ? 0 : 1;
}
