// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Flat C wrapper around the *unmodified* reference library `mpsamp`, compiled
// from its own sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libmpsamp_ref.so.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py load it, as the checker and
// the CPU comparator.  No reference source is copied here: this file only
// includes the reference headers and calls the reference's public API.
//
// Entry points wrapped (reference file:line):
//   rng::mix64 / key / uniform         proj/include/mpsamp/rng.hpp:12-37
//   round_scalar                        proj/src/precision.cpp:104-112
//   random_mps / capped_bond_dims       proj/src/mps.cpp:78-88,129-181
//   decay_chain / branching_decay_chain proj/src/mps.cpp:183-212
//   sample_batch                        proj/src/sampler.cpp:164-205
//   contract_site / measure / scale     proj/src/contract.cpp:109-121, sampler.cpp:60-118,
//                                       precision.cpp:135-165
//   save_mps / run_data_parallel /      proj/src/mps_io.cpp:167-210, parallel.cpp:240-330,
//   run_tensor_parallel                 parallel.cpp:579-630
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "mpsamp/contract.hpp"
#include "mpsamp/errors.hpp"
#include "mpsamp/mps.hpp"
#include "mpsamp/mps_io.hpp"
#include "mpsamp/parallel.hpp"
#include "mpsamp/precision.hpp"
#include "mpsamp/rng.hpp"
#include "mpsamp/sampler.hpp"

using namespace mpsamp;

namespace {

thread_local std::string g_err;

int map_exception() {
    try {
        throw;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return 2;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

SamplerOptions make_opts(uint64_t seed, int compute, int scaling) {
    SamplerOptions o;
    o.seed = seed;
    o.policy.compute = static_cast<Precision>(compute);
    o.policy.storage = Precision::F64;
    o.policy.scaling = static_cast<ScalingMode>(scaling);
    return o;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_mix64(uint64_t z) { return rng::mix64(z); }
uint64_t ref_rng_key(uint64_t seed, uint64_t stream, uint64_t sample, uint64_t site) {
    return rng::key(seed, stream, sample, site);
}
double ref_rng_uniform(uint64_t seed, uint64_t stream, uint64_t sample, uint64_t site) {
    return rng::uniform(seed, stream, sample, site);
}
double ref_round_scalar(double x, int precision) {
    return round_scalar(x, static_cast<Precision>(precision));
}

// ---- MPS handles ---------------------------------------------------------------------------

void* ref_mps_random(size_t m, size_t chi, size_t d, uint64_t seed, double level_damping,
                     double lambda_decay) {
    try {
        RandomMpsOptions o;
        o.level_damping = level_damping;
        o.lambda_decay = lambda_decay;
        return new MpsState(random_mps(m, chi, d, seed, o));
    } catch (...) {
        map_exception();
        return nullptr;
    }
}

void* ref_mps_decay_chain(size_t m, size_t d, double decades) {
    return new MpsState(decay_chain(m, d, decades));
}

void* ref_mps_branching_decay_chain(size_t m, double decades) {
    return new MpsState(branching_decay_chain(m, decades));
}

// gamma[i]: interleaved (re, im) doubles, shape (bond[i], bond[i+1], d) row-major.
void* ref_mps_from_arrays(size_t m, size_t d, const size_t* bonds, const double* const* gamma,
                          const double* const* lambda) {
    auto* s = new MpsState();
    s->num_sites = m;
    s->phys_dim = d;
    s->bond_dims.assign(bonds, bonds + m + 1);
    for (size_t i = 0; i < m; ++i) {
        const size_t cl = bonds[i], cr = bonds[i + 1];
        std::vector<cdouble> data(cl * cr * d);
        std::memcpy(data.data(), gamma[i], data.size() * sizeof(cdouble));
        s->gammas.emplace_back(std::vector<size_t>{cl, cr, d}, std::move(data));
        s->lambdas.emplace_back(lambda[i], lambda[i] + cr);
    }
    return s;
}

void ref_mps_free(void* h) { delete static_cast<MpsState*>(h); }
size_t ref_mps_num_sites(void* h) { return static_cast<MpsState*>(h)->num_sites; }
size_t ref_mps_phys_dim(void* h) { return static_cast<MpsState*>(h)->phys_dim; }
size_t ref_mps_bond(void* h, size_t i) { return static_cast<MpsState*>(h)->bond_dims.at(i); }
void ref_mps_gamma(void* h, size_t i, double* out) {
    const auto& g = static_cast<MpsState*>(h)->gammas.at(i);
    std::memcpy(out, g.data(), g.size() * sizeof(cdouble));
}
void ref_mps_lambda(void* h, size_t i, double* out) {
    const auto& l = static_cast<MpsState*>(h)->lambdas.at(i);
    std::memcpy(out, l.data(), l.size() * sizeof(double));
}
int ref_mps_validate(void* h) {
    try {
        static_cast<MpsState*>(h)->validate();
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// ---- sampling --------------------------------------------------------------------------------

// Full reference entry point sampler.cpp:164. out: N x M u8 row-major.
int ref_sample_batch(void* h, uint64_t n, uint64_t n1, uint64_t n2, uint64_t seed, int compute,
                     int scaling, uint8_t* out, uint64_t* contraction_macs, uint64_t* dead) {
    try {
        BatchPlan plan;
        plan.total_samples = n;
        plan.macro_batch = n1;
        plan.micro_batch = n2;
        RunStats st;
        SampleBatch b = sample_batch(*static_cast<MpsState*>(h), plan, make_opts(seed, compute, scaling), &st);
        std::memcpy(out, b.outcomes.data(), b.outcomes.size());
        if (contraction_macs) *contraction_macs = st.flops.contraction_macs;
        if (dead) *dead = st.dead_samples;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// sample_batch with the RunStats counters (contract.hpp:12-25, sampler.hpp:46-54):
// out4 = {contraction_macs, displacement_macs, measure_weight_macs, measure_pipeline_ops}
int ref_sample_batch_stats(void* h, uint64_t n, uint64_t seed, int compute, int scaling, uint8_t* out,
                           uint64_t* out4, uint64_t* dead) {
    try {
        RunStats st;
        SampleBatch b = sample_batch(*static_cast<MpsState*>(h), BatchPlan::simple(n),
                                     make_opts(seed, compute, scaling), &st);
        std::memcpy(out, b.outcomes.data(), b.outcomes.size());
        out4[0] = st.flops.contraction_macs;
        out4[1] = st.flops.displacement_macs;
        out4[2] = st.flops.measure_weight_macs;
        out4[3] = st.flops.measure_pipeline_ops;
        if (dead) *dead = st.dead_samples;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// detail::sample_micro_serial sampler.cpp:129 over [first, first+count), run on `threads`
// host threads over disjoint contiguous sub-ranges (equivalent to run_data_parallel with
// p1 = threads because draws are keyed by global sample index).  rows: count x M.
int ref_sample_range(void* h, uint64_t first, uint64_t count, uint64_t seed, int compute,
                     int scaling, int threads, uint8_t* rows) {
    const MpsState& mps = *static_cast<MpsState*>(h);
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(threads);
    SamplerOptions opts = make_opts(seed, compute, scaling);
    const size_t m = mps.num_sites;
    for (int t = 0; t < threads; ++t) {
        uint64_t a = first + count * t / threads, b = first + count * (t + 1) / threads;
        pool.emplace_back([&, t, a, b] {
            try {
                RunStats st;
                if (b > a) detail::sample_micro_serial(mps, a, b - a, opts, rows + (a - first) * m, st);
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs) {
        if (e) {
            try {
                std::rethrow_exception(e);
            } catch (...) {
                return map_exception();
            }
        }
    }
    return 0;
}

// Teacher-forced per-site marginals: drives the reference's own contract_site / measure /
// scale_rows_inplace along a *given* outcome string per sample and records the normalized
// weights p[n, i, k] = w[n,k] / sum_k w[n,k] (sampler.cpp:83-100).  This is the reference's
// conditional distribution at every site for the GPU's (or any) outcome prefix.
// forced: count x M u8 (0xFF = dead from that site on).  marg: count x M x d doubles.
int ref_marginals_forced(void* h, uint64_t count, int compute, int scaling, const uint8_t* forced,
                         double* marg) {
    try {
        const MpsState& mps = *static_cast<MpsState*>(h);
        const size_t m = mps.num_sites, d = mps.phys_dim;
        PrecisionPolicy pol;
        pol.compute = static_cast<Precision>(compute);
        pol.scaling = static_cast<ScalingMode>(scaling);
        ComplexTensor env({count, 1});
        for (size_t n = 0; n < count; ++n) env[n] = cdouble(1.0, 0.0);
        std::vector<uint8_t> alive(count, 1);
        for (size_t i = 0; i < m; ++i) {
            ComplexTensor temp = contract_site(env, mps.gammas[i], pol);
            const size_t chi = temp.extent(1);
            const auto& lam = mps.lambdas[i];
            ComplexTensor next({count, chi});
            for (size_t n = 0; n < count; ++n) {
                double* mrow = marg + (n * m + i) * d;
                const uint8_t k_f = forced[n * m + i];
                if (!alive[n] || k_f == kDeadOutcome) {
                    alive[n] = 0;
                    for (size_t k = 0; k < d; ++k) mrow[k] = -1.0;
                    continue;
                }
                std::vector<double> w(d, 0.0);
                const cdouble* row = temp.data() + n * chi * d;
                for (size_t b = 0; b < chi; ++b) {
                    const double l2 = lam[b] * lam[b];
                    for (size_t k = 0; k < d; ++k) w[k] += l2 * std::norm(row[b * d + k]);
                }
                double total = 0.0;
                for (size_t k = 0; k < d; ++k) total += w[k];
                for (size_t k = 0; k < d; ++k) mrow[k] = total == 0.0 ? -1.0 : w[k] / total;
                for (size_t b = 0; b < chi; ++b) next.at2(n, b) = row[b * d + k_f];
            }
            env = std::move(next);
            scale_rows_inplace(env, pol.scaling, alive);
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// CPU baseline probe: the reference hot step (contract_site -> measurement_draws -> measure ->
// scale_rows_inplace, i.e. one iteration of sampler.cpp:140-158) at site `site` of the given
// state for `count` samples per thread starting from a seeded random environment, run on
// `threads` host threads concurrently.  Returns wall seconds; macs gets the contraction MACs.
double ref_time_site_step(void* h, size_t site, uint64_t count, int threads, int reps,
                          uint64_t* macs) {
    const MpsState& mps = *static_cast<MpsState*>(h);
    const ComplexTensor& g = mps.gammas.at(site);
    const size_t cl = g.extent(0);
    std::vector<ComplexTensor> envs;
    for (int t = 0; t < threads; ++t) {
        ComplexTensor e({count, cl});
        for (size_t j = 0; j < e.size(); ++j) {
            e[j] = cdouble(rng::uniform(99, 1, t, j) - 0.5, rng::uniform(99, 2, t, j) - 0.5);
        }
        envs.push_back(std::move(e));
    }
    PrecisionPolicy pol;
    pol.scaling = ScalingMode::PerSampleMax;
    std::vector<uint64_t> mac(threads, 0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            for (int r = 0; r < reps; ++r) {
                FlopCounters fc;
                ComplexTensor temp = contract_site(envs[t], g, pol, &fc);
                std::vector<double> draws = detail::measurement_draws(7, t * count, count, site);
                std::vector<uint8_t> alive(count, 1);
                MeasureResult mr = measure(temp, mps.lambdas[site], draws, alive, &fc);
                scale_rows_inplace(mr.env, pol.scaling, alive);
                mac[t] += fc.contraction_macs;
            }
        });
    }
    for (auto& th : pool) th.join();
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (macs) {
        *macs = 0;
        for (auto v : mac) *macs += v;
    }
    return s;
}

// ---- file-backed executors (scheme-invariance checks) ----------------------------------------

int ref_save_mps(void* h, const char* path, int storage) {
    try {
        save_mps(*static_cast<MpsState*>(h), path, static_cast<Precision>(storage));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// scheme: 0 serial, 1 data-parallel(p1), 2 single-site TP(p1 x p2), 3 double-site TP(p1 x p2)
int ref_run_scheme(const char* path, int scheme, uint64_t n, uint64_t n1, uint64_t n2, size_t p1,
                   size_t p2, uint64_t seed, int compute, int scaling, uint8_t* out) {
    try {
        BatchPlan plan;
        plan.total_samples = n;
        plan.macro_batch = n1;
        plan.micro_batch = n2;
        SamplerOptions o = make_opts(seed, compute, scaling);
        ParallelResult r;
        switch (scheme) {
            case 0: r = run_serial(path, plan, o); break;
            case 1: r = run_data_parallel(path, plan, p1, o); break;
            case 2: r = run_tensor_parallel(path, plan, p1, p2, false, o); break;
            case 3: r = run_tensor_parallel(path, plan, p1, p2, true, o); break;
            default: throw ConfigError("unknown scheme");
        }
        std::memcpy(out, r.batch.outcomes.data(), r.batch.outcomes.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

}  // extern "C"

extern "C" {
// contract_site (contract.cpp:109) on flat arrays: env (count, chil), gamma (chil, chir, d).
int ref_contract_site(const double* env, size_t count, size_t chil, const double* gamma, size_t chir,
                      size_t d, int compute, double* out) {
    try {
        std::vector<cdouble> e(count * chil), g(chil * chir * d);
        std::memcpy(e.data(), env, e.size() * sizeof(cdouble));
        std::memcpy(g.data(), gamma, g.size() * sizeof(cdouble));
        ComplexTensor et({count, chil}, std::move(e)), gt({chil, chir, d}, std::move(g));
        PrecisionPolicy pol;
        pol.compute = static_cast<Precision>(compute);
        ComplexTensor t = contract_site(et, gt, pol);
        std::memcpy(out, t.data(), t.size() * sizeof(cdouble));
        return 0;
    } catch (...) {
        return map_exception();
    }
}
}

extern "C" {
// load_mps (mps_io.cpp:277-292) -> MpsState handle
void* ref_mps_load(const char* path) {
    try {
        return new MpsState(load_mps(path));
    } catch (...) {
        map_exception();
        return nullptr;
    }
}
// apply_schedule (sampler.cpp:218-246) -> new MpsState handle
void* ref_mps_apply_schedule(void* h, const size_t* per_site_chi, size_t n, size_t chi_max) {
    try {
        BondSchedule s;
        s.per_site_chi.assign(per_site_chi, per_site_chi + n);
        s.chi_max = chi_max;
        return new MpsState(apply_schedule(*static_cast<MpsState*>(h), s));
    } catch (...) {
        map_exception();
        return nullptr;
    }
}
// sample_batch with a BondSchedule in SamplerOptions (sampler.cpp:173-176)
int ref_sample_batch_scheduled(void* h, uint64_t n, uint64_t seed, int scaling, const size_t* chi,
                               size_t nchi, size_t chi_max, uint8_t* out) {
    try {
        SamplerOptions o = make_opts(seed, 0, scaling);
        BondSchedule s;
        s.per_site_chi.assign(chi, chi + nchi);
        s.chi_max = chi_max;
        o.schedule = s;
        SampleBatch b = sample_batch(*static_cast<MpsState*>(h), BatchPlan::simple(n), o);
        std::memcpy(out, b.outcomes.data(), b.outcomes.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}
}

extern "C" {
// decay_probe (sampler.cpp:207-216): per-site mean |env| before scaling. out: M doubles.
int ref_decay_probe(void* h, int compute, int scaling, uint64_t count, uint64_t seed, double* out) {
    try {
        PrecisionPolicy pol;
        pol.compute = static_cast<Precision>(compute);
        pol.scaling = static_cast<ScalingMode>(scaling);
        std::vector<double> t = decay_probe(*static_cast<MpsState*>(h), pol, count, seed);
        std::memcpy(out, t.data(), t.size() * sizeof(double));
        return 0;
    } catch (...) {
        return map_exception();
    }
}
}

// ---- site-streaming sweep (full-length parity on chains larger than host memory) ---------------
//
// The per-site body of detail::sample_micro_serial (sampler.cpp:140-158) -- contract_site ->
// measurement_draws -> measure -> scale_rows_inplace, the reference's own functions -- driven one
// site at a time, so the caller can hand over one decoded Gamma_i at a time (c3 as complex128 is
// 409 GB, beyond host memory) and drop it afterwards.  The samples [first, first + count) are split
// into `threads` contiguous chunks with one environment each (partition-invariant: draws are keyed
// by global sample index, rng.hpp:7-9).  Per site it also returns the reference's conditional
// distribution p[n, k] = w[n, k] / total (the weights of sampler.cpp:83-93, evaluated on the same
// temp) and, per sample, whether the draw lay within `eps` of an interior CDF boundary cum_k
// (k < d - 1, cum accumulated exactly as sampler.cpp:100-104).  With `forced` the outcome column
// is given (teacher forcing) and the environment follows it, as ref_marginals_forced does.
namespace {
struct SiteSweep {
    uint64_t first = 0, count = 0, seed = 0;
    PrecisionPolicy pol;
    std::vector<uint64_t> a, b;             // chunk ranges (relative to first)
    std::vector<ComplexTensor> env;         // per chunk (count_t, chiL)
    std::vector<std::vector<uint8_t>> alive;
    uint64_t macs = 0;
};
}  // namespace

extern "C" {
void* ref_sweep_begin(uint64_t first, uint64_t count, uint64_t seed, int compute, int scaling, int threads) {
    auto* s = new SiteSweep();
    s->first = first;
    s->count = count;
    s->seed = seed;
    s->pol.compute = static_cast<Precision>(compute);
    s->pol.storage = Precision::F64;
    s->pol.scaling = static_cast<ScalingMode>(scaling);
    if (threads < 1) threads = 1;
    for (int t = 0; t < threads; ++t) {
        const uint64_t a = count * t / threads, b = count * (t + 1) / threads;
        if (b <= a) continue;
        s->a.push_back(a);
        s->b.push_back(b);
        ComplexTensor e({b - a, 1});
        for (uint64_t n = 0; n < b - a; ++n) e[n] = cdouble(1.0, 0.0);  // sampler.cpp:136-137
        s->env.push_back(std::move(e));
        s->alive.emplace_back(b - a, 1);
    }
    return s;
}

// gamma: complex128 (chil, chir, d) of site `site`; lambda: chir.  out: count outcomes (0xFF dead);
// marg: count x d (-1 for samples not alive at this site); near: count flags (may be null).
int ref_sweep_site(void* hs, size_t site, const double* gamma, size_t chil, size_t chir, size_t d,
                   const double* lambda, const uint8_t* forced, double eps, uint8_t* out, double* marg,
                   uint8_t* near) {
    auto* s = static_cast<SiteSweep*>(hs);
    try {
        std::vector<cdouble> g(chil * chir * d);
        std::memcpy(g.data(), gamma, g.size() * sizeof(cdouble));
        const ComplexTensor gt({chil, chir, d}, std::move(g));
        const std::vector<double> lam(lambda, lambda + chir);
        const size_t T = s->env.size();
        std::vector<std::exception_ptr> errs(T);
        std::vector<uint64_t> macs(T, 0);
        std::vector<std::thread> pool;
        for (size_t t = 0; t < T; ++t) {
            pool.emplace_back([&, t] {
                try {
                    const uint64_t a = s->a[t], cnt = s->b[t] - s->a[t];
                    auto& alive = s->alive[t];
                    FlopCounters fc;
                    ComplexTensor temp = contract_site(s->env[t], gt, s->pol, &fc);
                    macs[t] = fc.contraction_macs;
                    std::vector<double> draws = detail::measurement_draws(s->seed, s->first + a, cnt, site);
                    std::vector<uint8_t> alive_in = alive;
                    // the reference's conditional distribution and boundary distance on this temp
                    std::vector<double> w(d);
                    for (uint64_t n = 0; n < cnt; ++n) {
                        double* mrow = marg + (a + n) * d;
                        if (near) near[a + n] = 0;
                        if (!alive_in[n] || (forced && forced[a + n] == kDeadOutcome)) {
                            for (size_t k = 0; k < d; ++k) mrow[k] = -1.0;
                            continue;
                        }
                        std::fill(w.begin(), w.end(), 0.0);
                        const cdouble* row = temp.data() + n * chir * d;
                        for (size_t r = 0; r < chir; ++r) {
                            const double l2 = lam[r] * lam[r];
                            for (size_t k = 0; k < d; ++k) w[k] += l2 * std::norm(row[r * d + k]);
                        }
                        double total = 0.0;
                        for (size_t k = 0; k < d; ++k) total += w[k];
                        double cum = 0.0;
                        bool nb = false;
                        for (size_t k = 0; k < d; ++k) {
                            mrow[k] = total == 0.0 ? -1.0 : w[k] / total;
                            cum += total == 0.0 ? 0.0 : w[k] / total;
                            if (k + 1 < d && std::fabs(draws[n] - cum) < eps) nb = true;
                        }
                        if (near) near[a + n] = nb && !forced ? 1 : 0;
                    }
                    if (!forced) {  // the reference's own measure + scaling (sampler.cpp:145-156)
                        MeasureResult mr = measure(temp, lam, draws, alive, &fc);
                        s->env[t] = std::move(mr.env);
                        scale_rows_inplace(s->env[t], s->pol.scaling, alive);
                        for (uint64_t n = 0; n < cnt; ++n) out[a + n] = mr.outcomes[n];
                    } else {        // teacher forcing along the given column
                        ComplexTensor next({cnt, chir});
                        for (uint64_t n = 0; n < cnt; ++n) {
                            const uint8_t k_f = forced[a + n];
                            out[a + n] = alive[n] ? k_f : kDeadOutcome;
                            if (!alive[n] || k_f == kDeadOutcome || marg[(a + n) * d] < 0.0) {
                                alive[n] = 0;
                                continue;
                            }
                            const cdouble* row = temp.data() + n * chir * d;
                            for (size_t r = 0; r < chir; ++r) next.at2(n, r) = row[r * d + k_f];
                        }
                        s->env[t] = std::move(next);
                        scale_rows_inplace(s->env[t], s->pol.scaling, alive);
                    }
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        }
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        for (auto m : macs) s->macs += m;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

uint64_t ref_sweep_macs(void* hs) { return static_cast<SiteSweep*>(hs)->macs; }
void ref_sweep_end(void* hs) { delete static_cast<SiteSweep*>(hs); }
}
