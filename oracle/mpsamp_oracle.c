/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 *
 * Plain-C restatement of the reference `mpsamp` sampling sweep (FastMPS, arxiv 2512.20064,
 * reference tree /root/reference/proj).  Built by oracle/Makefile into oracle/liboracle.so and
 * loaded only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  The product
 * library (paper_2512_20064_b200/libmpsg.so) never links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks every function here against golden vectors made by
 * the compiled reference itself (oracle/gen_golden.py -> tests/golden/) and, when
 * oracle/_ref/libmpsamp_ref.so is present, against the live reference on random inputs.
 *
 * Layouts follow the reference exactly:
 *   gamma_i  (chiL, chiR, d) complex row-major, d fastest      tensor.hpp:56-61, mps.hpp:10-11
 *   lambda_i length chiR                                        mps.hpp:19
 *   env      (count, chi) complex                               sampler.cpp:136
 *   rows     count x M u8, 0xFF = dead                          sampler.hpp:17
 * Complex values are interleaved (re, im) doubles (layout-compatible with std::complex<double>).
 */
#include "mpsamp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- RNG: rng.hpp:12-37 ------------------------------------------------------------------ */

uint64_t orc_mix64(uint64_t z) { /* rng.hpp:12-17 (splitmix64 finalizer) */
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t orc_key(uint64_t seed, uint64_t stream, uint64_t sample, uint64_t site) { /* :22-28 */
    uint64_t h = orc_mix64(seed ^ (stream * 0xD6E8FEB86659FD93ull));
    h = orc_mix64(h ^ (sample * 0xA5A5A5A5A5A5A5A5ull));
    h = orc_mix64(h ^ (site * 0xC2B2AE3D27D4EB4Full));
    return h;
}

double orc_to_unit(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; } /* :30-32 */

double orc_uniform(uint64_t seed, uint64_t stream, uint64_t sample, uint64_t site) {
    return orc_to_unit(orc_key(seed, stream, sample, site)); /* :34-37 */
}

/* ---- precision grids: precision.cpp:19-50 ------------------------------------------------ */

double orc_round_to_grid(double x, int mant_bits, int emin_normal, int emax) {
    if (x == 0.0 || isnan(x) || isinf(x)) return x;
    const double sign = signbit(x) ? -1.0 : 1.0;
    const double ax = fabs(x);
    int e;
    (void)frexp(ax, &e);
    const int exp_unbiased = e - 1;
    const int q_exp = (exp_unbiased > emin_normal ? exp_unbiased : emin_normal) - mant_bits;
    const double v = ldexp(ax, -q_exp);
    double n = floor(v);
    const double frac = v - n;
    if (frac > 0.5) {
        n += 1.0;
    } else if (frac == 0.5 && fmod(n, 2.0) != 0.0) {
        n += 1.0; /* ties to even */
    }
    const double r = ldexp(n, q_exp);
    const double max_normal = ldexp(2.0 - ldexp(1.0, -mant_bits), emax);
    if (r > max_normal) return sign * INFINITY;
    return sign * r;
}

double orc_round_scalar(double x, int precision) { /* precision.cpp:104-112 */
    switch (precision) {
        case ORC_F32: return orc_round_to_grid(x, 23, -126, 127);
        case ORC_TF32: return orc_round_to_grid(x, 10, -126, 127);
        case ORC_F16: return orc_round_to_grid(x, 10, -14, 15);
        default: return x;
    }
}

/* ---- contraction: contract.cpp:18-41 (f64) and :43-82 (reduced) ------------------------- */

/* out[n, r, k] = sum_{l ascending} env[n, l] * gamma[l, r, k]  (contract.cpp:31-39). */
static void contract_f64(const double* env, size_t count, size_t chil, const double* gamma,
                         size_t chir, size_t d, double* out) {
    const size_t width = chir * d;
    memset(out, 0, sizeof(double) * 2 * count * width);
    for (size_t n = 0; n < count; ++n) {
        double* dst = out + 2 * n * width;
        const double* erow = env + 2 * n * chil;
        for (size_t l = 0; l < chil; ++l) {
            const double cr = erow[2 * l], ci = erow[2 * l + 1];
            const double* g = gamma + 2 * l * width;
            for (size_t j = 0; j < width; ++j) {
                const double gr = g[2 * j], gi = g[2 * j + 1];
                dst[2 * j] += cr * gr - ci * gi;
                dst[2 * j + 1] += cr * gi + ci * gr;
            }
        }
    }
}

/* std::complex<float> product as compiled by g++ for contract.cpp:74: the inline
 * (ac - bd, ad + bc) evaluation, and when both parts are NaN the C99 Annex G recovery that
 * libgcc's __mulsc3 performs (infinite operands yield infinities, not NaN).  Only matters when
 * the F16/TF32 grids overflow to inf. */
static void cmulf_annex_g(float a, float b, float c, float d, float* re, float* im) {
    volatile float ac = a * c, bd = b * d, ad = a * d, bc = b * c;
    float x = ac - bd, y = ad + bc;
    if (isnan(x) && isnan(y)) {
        int recalc = 0;
        if (isinf(a) || isinf(b)) {
            a = copysignf(isinf(a) ? 1.0f : 0.0f, a);
            b = copysignf(isinf(b) ? 1.0f : 0.0f, b);
            if (isnan(c)) c = copysignf(0.0f, c);
            if (isnan(d)) d = copysignf(0.0f, d);
            recalc = 1;
        }
        if (isinf(c) || isinf(d)) {
            c = copysignf(isinf(c) ? 1.0f : 0.0f, c);
            d = copysignf(isinf(d) ? 1.0f : 0.0f, d);
            if (isnan(a)) a = copysignf(0.0f, a);
            if (isnan(b)) b = copysignf(0.0f, b);
            recalc = 1;
        }
        if (!recalc && (isinf(ac) || isinf(bd) || isinf(ad) || isinf(bc))) {
            if (isnan(a)) a = copysignf(0.0f, a);
            if (isnan(b)) b = copysignf(0.0f, b);
            if (isnan(c)) c = copysignf(0.0f, c);
            if (isnan(d)) d = copysignf(0.0f, d);
            recalc = 1;
        }
        if (recalc) {
            volatile float p1 = a * c, p2 = b * d, p3 = a * d, p4 = b * c;
            x = INFINITY * (p1 - p2);
            y = INFINITY * (p3 + p4);
        }
    }
    *re = x;
    *im = y;
}

/* Reduced path contract.cpp:53-81: operands RNE-rounded onto the policy grid, complex<float>
 * accumulation in ascending l. */
static void contract_reduced(const double* env, size_t count, size_t chil, const double* gamma,
                             size_t chir, size_t d, int prec, double* out) {
    const size_t width = chir * d;
    float* gb = (float*)malloc(sizeof(float) * 2 * chil * width);
    float* acc = (float*)malloc(sizeof(float) * 2 * width);
    for (size_t j = 0; j < chil * width; ++j) {
        gb[2 * j] = (float)orc_round_scalar(gamma[2 * j], prec);
        gb[2 * j + 1] = (float)orc_round_scalar(gamma[2 * j + 1], prec);
    }
    for (size_t n = 0; n < count; ++n) {
        memset(acc, 0, sizeof(float) * 2 * width);
        const double* erow = env + 2 * n * chil;
        for (size_t l = 0; l < chil; ++l) {
            const float cr = (float)orc_round_scalar(erow[2 * l], prec);
            const float ci = (float)orc_round_scalar(erow[2 * l + 1], prec);
            const float* g = gb + 2 * l * width;
            for (size_t j = 0; j < width; ++j) {
                float pr, pi;
                cmulf_annex_g(cr, ci, g[2 * j], g[2 * j + 1], &pr, &pi);
                acc[2 * j] += pr;
                acc[2 * j + 1] += pi;
            }
        }
        double* dst = out + 2 * n * width;
        for (size_t j = 0; j < 2 * width; ++j) dst[j] = (double)acc[j];
    }
    free(gb);
    free(acc);
}

int orc_contract_site(const double* env, size_t count, size_t chil, const double* gamma,
                      size_t chir, size_t d, int compute, double* out) {
    if (compute == ORC_F64) { /* non-finite check contract.cpp:117-119 */
        for (size_t j = 0; j < 2 * count * chil; ++j)
            if (!isfinite(env[j])) return ORC_ERR_NUMERIC;
        for (size_t j = 0; j < 2 * chil * chir * d; ++j)
            if (!isfinite(gamma[j])) return ORC_ERR_NUMERIC;
        contract_f64(env, count, chil, gamma, chir, d, out);
    } else {
        contract_reduced(env, count, chil, gamma, chir, d, compute, out);
    }
    return 0;
}

/* ---- measurement: sampler.cpp:60-118 ----------------------------------------------------- */

void orc_measure(const double* temp, size_t count, size_t chi, size_t d, const double* lambda,
                 const double* draws, uint8_t* alive, uint8_t* outcomes, double* env_out,
                 double* weights_out) {
    double* w = (double*)malloc(sizeof(double) * d);
    memset(env_out, 0, sizeof(double) * 2 * count * chi);
    for (size_t n = 0; n < count; ++n) {
        outcomes[n] = ORC_DEAD;
        if (weights_out)
            for (size_t k = 0; k < d; ++k) weights_out[n * d + k] = -1.0;
        if (!alive[n]) continue;
        for (size_t k = 0; k < d; ++k) w[k] = 0.0;
        const double* row = temp + 2 * n * chi * d;
        for (size_t b = 0; b < chi; ++b) { /* :84-89 */
            const double l2 = lambda[b] * lambda[b];
            const double* t = row + 2 * b * d;
            for (size_t k = 0; k < d; ++k) w[k] += l2 * (t[2 * k] * t[2 * k] + t[2 * k + 1] * t[2 * k + 1]);
        }
        double total = 0.0;
        for (size_t k = 0; k < d; ++k) total += w[k];
        if (weights_out)
            for (size_t k = 0; k < d; ++k) weights_out[n * d + k] = total == 0.0 ? -1.0 : w[k] / total;
        if (total == 0.0) { /* :94-98 */
            alive[n] = 0;
            continue;
        }
        const double draw = draws[n];
        double cum = 0.0;
        size_t outcome = 0;
        for (size_t k = 0; k < d; ++k) { /* :100-106, strict '>' and no early break */
            cum += w[k] / total;
            if (draw > cum) ++outcome;
        }
        if (outcome >= d) outcome = d - 1; /* :107 */
        outcomes[n] = (uint8_t)outcome;
        double* env_row = env_out + 2 * n * chi;
        for (size_t b = 0; b < chi; ++b) { /* :110-111 */
            env_row[2 * b] = row[2 * (b * d + outcome)];
            env_row[2 * b + 1] = row[2 * (b * d + outcome) + 1];
        }
    }
    free(w);
}

/* ---- scaling: precision.cpp:135-165 ------------------------------------------------------ */

static double component_mag(double re, double im) { /* tensor.hpp:78-82 */
    const double a = fabs(re), b = fabs(im);
    return a > b ? a : b;
}

void orc_scale_rows(double* env, size_t count, size_t row, int mode, uint8_t* alive) {
    if (mode == ORC_SCALE_NONE) return;
    if (mode == ORC_SCALE_GLOBAL) { /* :143-150 */
        double m = 0.0;
        for (size_t i = 0; i < count * row; ++i) {
            const double c = component_mag(env[2 * i], env[2 * i + 1]);
            m = (m < c) ? c : m; /* std::max(m, c): a NaN c is ignored */
        }
        if (m == 0.0) m = 1.0;
        for (size_t i = 0; i < count * row; ++i) {
            env[2 * i] /= m;
            env[2 * i + 1] /= m;
        }
        return;
    }
    for (size_t n = 0; n < count; ++n) { /* :152-163 */
        if (!alive[n]) continue;
        double* r = env + 2 * n * row;
        double m = 0.0;
        for (size_t i = 0; i < row; ++i) {
            const double c = component_mag(r[2 * i], r[2 * i + 1]);
            m = (m < c) ? c : m; /* std::max(m, c): a NaN c is ignored */
        }
        if (m == 0.0) {
            alive[n] = 0;
            continue;
        }
        /* std::complex<double> /= double divides both parts */
        for (size_t i = 0; i < row; ++i) {
            r[2 * i] /= m;
            r[2 * i + 1] /= m;
        }
    }
}

/* ---- GBS displacement (SPEC.md gbs-ops, §3.4 Eq. 6) ------------------------------
 * expm_displacement: D(mu) = exp(-|mu|^2/2) L U with L = exp(mu a^dag) lower triangular,
 * L[a][b] = mu^(a-b) sqrt(a!/b!) / (a-b)!, and U = exp(-conj(mu) a) upper triangular,
 * U[b][c] = (-conj(mu))^(c-b) sqrt(c!/b!) / (c-b)! (closed form, no iterative
 * expm; factorial ratios through lgamma).  out: n x n complex, row-major D[a][c] interleaved. */
static void cpow_int(double re, double im, int k, double* ore, double* oim) {
    double r = 1.0, i = 0.0;
    for (int j = 0; j < k; ++j) {
        const double t = r * re - i * im;
        i = r * im + i * re;
        r = t;
    }
    *ore = r;
    *oim = i;
}

void orc_displacement(double mu_re, double mu_im, size_t n, double* out) {
    const double pre = exp(-0.5 * (mu_re * mu_re + mu_im * mu_im));
    for (size_t a = 0; a < n; ++a)
        for (size_t c = 0; c < n; ++c) {
            double sr = 0.0, si = 0.0;
            const size_t bmax = a < c ? a : c;
            for (size_t b = 0; b <= bmax; ++b) {
                double lr, li, ur, ui;
                cpow_int(mu_re, mu_im, (int)(a - b), &lr, &li);
                cpow_int(-mu_re, mu_im, (int)(c - b), &ur, &ui); /* -conj(mu) */
                const double fl = exp(0.5 * (lgamma((double)a + 1) - lgamma((double)b + 1)) - lgamma((double)(a - b) + 1));
                const double fu = exp(0.5 * (lgamma((double)c + 1) - lgamma((double)b + 1)) - lgamma((double)(c - b) + 1));
                lr *= fl, li *= fl, ur *= fu, ui *= fu;
                sr += lr * ur - li * ui;
                si += lr * ui + li * ur;
            }
            out[2 * (a * n + c)] = pre * sr;
            out[2 * (a * n + c) + 1] = pre * si;
        }
}

/* apply_displacement as the reference's SiteTransform hook: temp (count, chi, d)
 * row-major, temp[n, b, :] <- D(mu[n]) temp[n, b, :] */
static void apply_displacement(double* temp, size_t count, size_t chi, size_t d, const double* mu,
                               size_t mu_stride, double* dbuf, double* v) {
    for (size_t n = 0; n < count; ++n) {
        orc_displacement(mu[2 * n * mu_stride], mu[2 * n * mu_stride + 1], d, dbuf);
        for (size_t b = 0; b < chi; ++b) {
            double* t = temp + 2 * (n * chi + b) * d;
            memcpy(v, t, sizeof(double) * 2 * d);
            for (size_t k = 0; k < d; ++k) {
                double sr = 0.0, si = 0.0;
                for (size_t q = 0; q < d; ++q) {
                    const double dr = dbuf[2 * (k * d + q)], di = dbuf[2 * (k * d + q) + 1];
                    sr += dr * v[2 * q] - di * v[2 * q + 1];
                    si += dr * v[2 * q + 1] + di * v[2 * q];
                }
                t[2 * k] = sr;
                t[2 * k + 1] = si;
            }
        }
    }
}

/* ---- the site loop: detail::sample_micro_serial sampler.cpp:129-162 ----------------------- */

int orc_sample_range(size_t m, size_t d, const size_t* bonds, const double* const* gamma,
                     const double* const* lambda, uint64_t first, size_t count, uint64_t seed,
                     int compute, int scaling, const uint8_t* forced, uint8_t* rows,
                     double* marg, uint64_t* contraction_macs) {
    return orc_sample_range_displaced(m, d, bonds, gamma, lambda, first, count, seed, compute, scaling,
                                      forced, NULL, rows, marg, contraction_macs);
}

/* Same with the GBS displacement hook (sampler.cpp:143: site_transform between contract_site and
 * the draws): mu = NULL or complex128 (count, m), mu[n][i] the displacement of sample n at site i. */
int orc_sample_range_displaced(size_t m, size_t d, const size_t* bonds, const double* const* gamma,
                               const double* const* lambda, uint64_t first, size_t count, uint64_t seed,
                               int compute, int scaling, const uint8_t* forced, const double* mu,
                               uint8_t* rows, double* marg, uint64_t* contraction_macs) {
    size_t maxchi = 1;
    for (size_t i = 0; i <= m; ++i) maxchi = bonds[i] > maxchi ? bonds[i] : maxchi;
    double* env = (double*)malloc(sizeof(double) * 2 * count * maxchi);
    double* next = (double*)malloc(sizeof(double) * 2 * count * maxchi);
    double* temp = (double*)malloc(sizeof(double) * 2 * count * maxchi * d);
    double* draws = (double*)malloc(sizeof(double) * count);
    uint8_t* alive = (uint8_t*)malloc(count);
    uint8_t* oc = (uint8_t*)malloc(count);
    double* w = marg ? (double*)malloc(sizeof(double) * count * d) : NULL;
    int rc = 0;
    double* dbuf = (double*)malloc(sizeof(double) * 2 * d * d);
    double* dvec = (double*)malloc(sizeof(double) * 2 * d);
    for (size_t n = 0; n < count; ++n) { /* :136-138 */
        env[2 * n] = 1.0;
        env[2 * n + 1] = 0.0;
        alive[n] = 1;
    }
    if (contraction_macs) *contraction_macs = 0;
    for (size_t i = 0; i < m && rc == 0; ++i) {
        const size_t cl = bonds[i], cr = bonds[i + 1];
        rc = orc_contract_site(env, count, cl, gamma[i], cr, d, compute, temp);
        if (rc) break;
        if (contraction_macs) *contraction_macs += (uint64_t)count * cl * cr * d; /* contract.cpp:97-100 */
        if (mu) apply_displacement(temp, count, cr, d, mu + 2 * i, m, dbuf, dvec); /* sampler.cpp:143 */
        for (size_t j = 0; j < count; ++j) draws[j] = orc_uniform(seed, ORC_MEASURE_STREAM, first + j, i);
        orc_measure(temp, count, cr, d, lambda[i], draws, alive, oc, next, w);
        if (forced) { /* teacher forcing: continue along the given outcome string */
            for (size_t n = 0; n < count; ++n) {
                const uint8_t kf = forced[n * m + i];
                if (kf == ORC_DEAD || !alive[n]) {
                    alive[n] = 0;
                    oc[n] = ORC_DEAD;
                    continue;
                }
                oc[n] = kf;
                for (size_t b = 0; b < cr; ++b) {
                    next[2 * (n * cr + b)] = temp[2 * ((n * cr + b) * d + kf)];
                    next[2 * (n * cr + b) + 1] = temp[2 * ((n * cr + b) * d + kf) + 1];
                }
            }
        }
        if (marg)
            for (size_t n = 0; n < count; ++n) memcpy(marg + (n * m + i) * d, w + n * d, sizeof(double) * d);
        double* t = env;
        env = next;
        next = t;
        orc_scale_rows(env, count, cr, scaling, alive);
        for (size_t n = 0; n < count; ++n) rows[n * m + i] = oc[n];
    }
    free(env);
    free(next);
    free(temp);
    free(draws);
    free(alive);
    free(oc);
    free(w);
    free(dbuf);
    free(dvec);
    return rc;
}

/* ---- bond chain: mps.cpp:78-88 ---------------------------------------------------------- */

void orc_capped_bond_dims(size_t m, size_t d, size_t chi_max, size_t* out) {
    for (size_t i = 0; i <= m; ++i) {
        const double left = pow((double)d, (double)i);
        const double right = pow((double)d, (double)(m - i));
        double cap = left < right ? left : right;
        cap = cap < (double)chi_max ? cap : (double)chi_max;
        out[i] = (size_t)cap;
    }
}

/* FNV-1a 64 of a byte buffer (mps_io.cpp:18-25; used for outcome-matrix goldens). */
uint64_t orc_fnv1a(const uint8_t* p, size_t n) {
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

/* CPU baseline probe for the port: one iteration of the site loop (sampler.cpp:140-158) at a
 * single site for `count` samples from a seeded random environment, f64 + PerSampleMax.
 * Returns the complex MACs performed (time it from the caller). */
uint64_t orc_site_step(const double* gamma, size_t chil, size_t chir, size_t d, const double* lambda,
                       size_t count, uint64_t seed) {
    double* env = (double*)malloc(sizeof(double) * 2 * count * chil);
    double* temp = (double*)malloc(sizeof(double) * 2 * count * chir * d);
    double* next = (double*)malloc(sizeof(double) * 2 * count * chir);
    double* draws = (double*)malloc(sizeof(double) * count);
    uint8_t* alive = (uint8_t*)malloc(count);
    uint8_t* oc = (uint8_t*)malloc(count);
    for (size_t j = 0; j < 2 * count * chil; ++j) env[j] = orc_uniform(99, 1, 0, j) - 0.5;
    for (size_t n = 0; n < count; ++n) {
        alive[n] = 1;
        draws[n] = orc_uniform(seed, ORC_MEASURE_STREAM, n, 0);
    }
    contract_f64(env, count, chil, gamma, chir, d, temp);
    orc_measure(temp, count, chir, d, lambda, draws, alive, oc, next, NULL);
    orc_scale_rows(next, count, chir, ORC_SCALE_PER_SAMPLE, alive);
    free(env);
    free(temp);
    free(next);
    free(draws);
    free(alive);
    free(oc);
    return (uint64_t)count * chil * chir * d;
}
