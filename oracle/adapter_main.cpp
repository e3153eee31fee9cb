// TEST INFRASTRUCTURE: builds the drop-in adapter (include/mpsg_mpsamp.hpp) against the
// reference's own headers and library, exactly as a maintainer would, and checks it.
//   adapter_test cpu  -> validation/error mapping only (no GPU needed)
//   adapter_test gpu  -> c1 = random_mps(16, 32, 4, 42) through mpsg_mpsamp::sample_batch,
//                        compared with mpsamp::sample_batch on the same MPS and seed
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
  }
  std::printf("adapter gpu: %zu/1000 strings differ from the reference on the original (uncompressed) "
              "Gamma; contraction_macs %llu (reference %llu)\n",
              diff, static_cast<unsigned long long>(st.flops.contraction_macs), 45600000ull);
  return (st.flops.contraction_macs == 45600000ull && diff <= 20) ? 0 : 1;
}
