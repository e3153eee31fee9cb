/*
 * mpsg.h — C ABI of the B200-native MPS sampling sweep (FastMPS, arxiv 2512.20064).
 *
 * This is the drop-in boundary for the reference's sampling entry point.  The reference
 * (`mpsamp`, a C++20 library) has no FFI of its own; what a maintainer binds is
 *
 *   SampleBatch mpsamp::sample_batch(const MpsState&, const BatchPlan&, const SamplerOptions&,
 *                                    RunStats* = nullptr)             proj/include/mpsamp/sampler.hpp:84-85
 *   void mpsamp::detail::sample_micro_serial(const MpsState&, uint64_t first, size_t count,
 *                                            const SamplerOptions&, uint8_t* rows, RunStats&)
 *                                                                     proj/include/mpsamp/sampler.hpp:103-104
 *
 * Every entry point below replaces one of those (or one of the pieces the reference's
 * executors re-drive, sampler.hpp:98-102), takes only plain pointers and sizes, and returns an
 * error code that maps 1:1 onto the reference's exception hierarchy (errors.hpp:8-27):
 *
 *   MPSG_OK 0, MPSG_ERR_CONFIG 2 (ConfigError / DimensionError), MPSG_ERR_NUMERIC 3
 *   (NumericError), MPSG_ERR_IO 4 (IoError), MPSG_ERR_CUDA 5 (CUDA / NCCL failure),
 *   MPSG_ERR_INTERNAL 1.  mpsg_last_error() returns the thread-local message.
 *
 * Data layouts are the reference's, unchanged (tensor.hpp:56-61, mps.hpp:10-19):
 *   gamma[i]  complex128 interleaved (re, im), shape (bond[i], bond[i+1], d) row-major, d fastest
 *   lambda[i] float64, length bond[i+1], nonnegative and nonincreasing
 *   rows      uint8, count x num_sites row-major (stride num_sites), 0xFF = dead sample
 *   draws     keyed splitmix64 (rng.hpp:12-37), key(seed, 0x6d656173, global sample, site)
 *
 * The library is CUDA-only (sm_100a).  There is no CPU fallback: on a host without a B200 every
 * compute entry point returns MPSG_ERR_CUDA.
 */
#ifndef MPSG_H
#define MPSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPSG_ABI_VERSION 5  /* 2: mpsg_stats gained displacement_macs, measure_pipeline_ops; 3: mpsg_options.slice;
                               4: mpsg_stats.near_boundary_draws, mpsg_generated_*, mpsg_synthetic_site;
                               5: MPSG_MODE_GRID, block-aligned tensor-parallel shards,
                               mpsg_create_from_file_streamed */

enum {
  MPSG_OK = 0,
  MPSG_ERR_INTERNAL = 1,
  MPSG_ERR_CONFIG = 2,
  MPSG_ERR_NUMERIC = 3,
  MPSG_ERR_IO = 4,
  MPSG_ERR_CUDA = 5
};

/* Precision / ScalingMode values are the reference's enums (precision.hpp:15-17). */
enum { MPSG_F64 = 0, MPSG_F32 = 1, MPSG_TF32 = 2, MPSG_F16 = 3 };
enum { MPSG_SCALE_NONE = 0, MPSG_SCALE_GLOBAL_MAX = 1, MPSG_SCALE_PER_SAMPLE_MAX = 2 };

/* GPU contraction schemes:
 *   MPSG_MODE_SPLIT   fp16 Gamma x (hi + lo) fp16 environment, fp32 accumulate; F32-class
 *                     accuracy on the DECODED Gamma (the fp16 format moves the sampled
 *                     distribution itself by ~1e-4 relative at interior sites), 2x issued MMAs.
 *   MPSG_MODE_SINGLE  fp16 Gamma x fp16 environment, one MMA pass; F16-class accuracy.
 *   MPSG_MODE_AUTO    pick from policy.compute: TF32 / F16 -> GRID (below; else SINGLE); F64 / F32 -> PRECISE when its
 *                     state (6 fp16 planes, 12 B per complex entry) fits the device (resident) or
 *                     60% of host memory (host-streamed), else SPLIT.  mpsg_mode() reports the
 *                     choice.  Generated handles (synthetic chains) use SPLIT. */
enum { MPSG_MODE_AUTO = 0, MPSG_MODE_SPLIT = 1, MPSG_MODE_SINGLE = 2, MPSG_MODE_PRECISE = 3, MPSG_MODE_GRID = 4 };
/*   MPSG_MODE_GRID    the reference's TF32 / F16 compute policies (contract_block_reduced,
 *                     contract.cpp:43-82) on their own operand grids: Gamma and every environment
 *                     rounded component-wise exactly as round_scalar (precision.cpp:23-50) -- F16:
 *                     IEEE binary16 on the reference's own values (subnormals, overflow; a Gamma
 *                     element beyond the grid is MPSG_ERR_NUMERIC), TF32: 10-bit significands on the
 *                     f32 exponent range, realised as fp16 times power-of-two scales (exact down to
 *                     2^-28 of each column / row max) -- then one MMA pass with fp32 accumulation,
 *                     the reference's float accumulator.  4M scheme.  AUTO picks it for compute =
 *                     TF32 / F16 except on generated chains, with tensor parallelism, GlobalMax
 *                     scaling or the decay trace (there: SINGLE). */
/*   MPSG_MODE_PRECISE  SPLIT plus Gamma stored as an exact fp16 hi + lo pair per component (22-bit
 *                     mantissas instead of 11): the device samples the caller's f64 / f32 Gamma to
 *                     ~2^-23 instead of ~2^-12 per element, at 3 MMAs per K-step instead of 2 and
 *                     twice the Gamma bytes (12 B per complex entry).  3M scheme only. */
/* Complex decomposition of the contraction:
 *   MPSG_SCHEME_3M  Gauss: 3 real products (Gamma planes Gr, Gi, Gr+Gi: 6 bytes per complex entry)
 *   MPSG_SCHEME_4M  4 real products (Gamma planes Gr, Gi: 4 bytes per complex entry)
 *   MPSG_SCHEME_AUTO  3M when the 3-plane state fits (device memory when resident, host memory
 *                     when host-streamed), else 4M. */
enum { MPSG_SCHEME_AUTO = 0, MPSG_SCHEME_3M = 3, MPSG_SCHEME_4M = 4 };

#define MPSG_DEAD 0xFF

/* Mirrors mpsamp::MpsState (mps.hpp:14-22) as plain pointers into caller-owned memory. */
typedef struct mpsg_mps_view {
  uint64_t num_sites;              /* M */
  uint64_t phys_dim;               /* d */
  const uint64_t* bond_dims;       /* M + 1, boundaries 1 */
  const double* const* gamma;      /* M pointers, complex128 interleaved (chiL, chiR, d) */
  const double* const* lambda;     /* M pointers, length bond_dims[i + 1] */
} mpsg_mps_view;

/* Mirrors mpsamp::PrecisionPolicy (precision.hpp:27-33). */
typedef struct mpsg_policy {
  int compute;                     /* MPSG_F64 .. MPSG_F16 */
  int storage;                     /* MPSG_F64 / F32 / F16 (TF32 rejected, precision.cpp:98-102) */
  int scaling;                     /* MPSG_SCALE_* */
} mpsg_policy;

/* Engine options (no reference counterpart; zero-initialise for defaults). */
typedef struct mpsg_options {
  int mode;                        /* MPSG_MODE_*, default AUTO */
  uint64_t pass_samples;           /* samples per device pass (the GEMM M extent); 0 = auto */
  int record_site_times;           /* 1: fill mpsg_stats.site_seconds (one event per site);
                                      2: also time every contraction kernel (gemm_seconds) */
  int tp_size;                     /* tensor-parallel group size (0/1 = none): this handle holds
                                      column shard tp_rank of every Gamma_i (balanced_partition of
                                      chiR, collective.cpp:80-92, rounded to whole contraction K
                                      blocks: 64 columns for 3M, 32 for 4M -- so the sharded sweep
                                      accumulates the unsharded sweep's K blocks in the same order
                                      and samples bit-identically), the even-site pattern of
                                      parallel.cpp:420-443 applied at every site */
  int tp_rank;
  int host_stream_slots;           /* 0: compressed Gamma resident in HBM.  >= 2: Gamma kept in
                                      pinned host memory and streamed per site through this many
                                      device slots by a copy stream overlapping the compute
                                      (the reference's SiteStream prefetch, mps_io.cpp:294-350) */
  int record_decay_trace;          /* fill mpsg_stats.decay_trace: mean |env| per site before
                                      scaling, in the reference's own scaling (sampler.cpp:149-153,
                                      decay_probe :207-216); GlobalMax is traced as None */
  int scheme;                      /* complex decomposition of the contraction: MPSG_SCHEME_AUTO,
                                      MPSG_SCHEME_3M or MPSG_SCHEME_4M (see above) */
  int slice;                       /* how the chosen slice reaches the next environment (MPSG_SLICE_*) */
} mpsg_options;

/* MPSG_SLICE_AUTO     = MPSG_SLICE_TEMP (the faster path on every measured configuration)
 * MPSG_SLICE_TEMP     the contraction materialises all d outcomes (temp) and the selection gathers
 *                     the chosen slice
 * MPSG_SLICE_RECOMPUTE  for plain sampling calls on a 3M state without tensor parallelism (d <= 32):
 *                     the contraction emits only the Born weights, the rows are bucketed by drawn
 *                     outcome and a 1/d-size GEMM recomputes the chosen slices straight into the
 *                     next environment (no temp round trip through HBM; same arithmetic, identical
 *                     outcomes).  Measured 15-32% slower than TEMP. */
enum { MPSG_SLICE_AUTO = 0, MPSG_SLICE_TEMP = 1, MPSG_SLICE_RECOMPUTE = 2 };

/* Mirrors mpsamp::RunStats + FlopCounters (sampler.hpp:46-54, contract.hpp:12-25). */
typedef struct mpsg_stats {
  uint64_t contraction_macs;       /* sum_i count * chiL_i * chiR_i * d (contract.cpp:97-100) */
  uint64_t measure_weight_macs;    /* sum_i live_i * chiR_i * d, live samples only (sampler.cpp:81-90) */
  uint64_t dead_samples;
  double seconds;                  /* wall time of the call */
  double* site_seconds;            /* optional caller array of length M (device time per site) */
  uint64_t issued_mma_flops;       /* real flops issued to the tensor cores (incl. padding, split) */
  uint64_t h2d_bytes, d2h_bytes;
  double gemm_seconds;             /* device time of the contraction kernels (record_site_times 2) */
  uint64_t gemm_flops;             /* algorithmic flops of those launches: 8 * contraction_macs */
  uint64_t kernel_launches;        /* CUDA kernels launched by this call */
  double device_seconds;           /* device time of all passes (CUDA events; record_site_times) */
  double* decay_trace;             /* optional caller array of length M (record_decay_trace) */
  uint64_t displacement_macs;      /* count * chiR_i * d^2 per displaced site (FlopCounters field of
                                      contract.hpp:14; the apply of SPEC.md:375-381) */
  uint64_t measure_pipeline_ops;   /* d per live (sample, site) (sampler.cpp:92-93,114-115) */
  uint64_t near_boundary_draws;    /* drawn (sample, site) pairs whose uniform lies within 1e-6 of an
                                      interior CDF boundary cum_k, k < d - 1 (sampler.cpp:100-106):
                                      the only draws whose outcome may differ from the reference's
                                      under rounding; counted on the device */
} mpsg_stats;

typedef struct mpsg_handle_s* mpsg_handle;

/* ---- library -------------------------------------------------------------------------- */
int mpsg_abi_version(void);
const char* mpsg_last_error(void);
/* Number of visible sm_100 devices (0 when none; never an error). */
int mpsg_device_count(void);

/* ---- state ----------------------------------------------------------------------------- */
/* Validates like MpsState::validate (mps.cpp:12-38) and PrecisionPolicy::validate
 * (precision.cpp:98-102), rejects non-finite Gamma like contract_site at F64
 * (contract.cpp:117-119), compresses every site to the device format (fp16 planes with
 * power-of-two row/column scales) and keeps it resident on each listed device (data-parallel
 * replicas).  devices == NULL / ndev == 0 means device 0. */
int mpsg_create(const mpsg_mps_view* mps, const mpsg_policy* policy, const mpsg_options* opts,
                const int* devices, int ndev, mpsg_handle* out);

/* Incremental builder for states too large for host memory (e.g. generated on the device).
 * gamma may be a host pointer or a device pointer on the first listed device; dtype is
 * MPSG_F64 (complex128) or MPSG_F32 (complex64). */
int mpsg_builder_begin(uint64_t num_sites, uint64_t phys_dim, const uint64_t* bond_dims,
                       const mpsg_policy* policy, const mpsg_options* opts, const int* devices,
                       int ndev, mpsg_handle* out);
int mpsg_builder_set_site(mpsg_handle h, uint64_t site, const void* gamma, int gamma_is_device,
                          int dtype, const double* lambda);
int mpsg_builder_finish(mpsg_handle h);

void mpsg_destroy(mpsg_handle h);

/* Bytes of the compressed state held per device: in HBM, or for a host-streamed handle in pinned
 * host memory (there the 3M sum planes are re-formed on the device after each copy, so a 3M
 * host-streamed state holds 2/3 of the resident state's bytes, as does a compact-3M state in HBM);
 * for a generated handle the bytes of its base isometries in HBM. */
uint64_t mpsg_state_bytes(mpsg_handle h);
/* The contraction scheme the handle runs: MPSG_SCHEME_3M or MPSG_SCHEME_4M (0 for a null handle). */
int mpsg_scheme(mpsg_handle h);
/* The precision mode the handle runs: MPSG_MODE_SPLIT, _SINGLE or _PRECISE (0 for a null handle). */
int mpsg_mode(mpsg_handle h);
/* Where the handle's compressed Gamma lives (0 for a null handle):
 *   MPSG_STORE_RESIDENT  all planes in HBM
 *   MPSG_STORE_COMPACT   3M with only [Gr, Gi] in HBM; each site is copied into a ring of device slots
 *                        and its Gs plane re-formed there (AUTO when only the 2-plane state fits)
 *   MPSG_STORE_HOST      pinned host memory, streamed per site (host_stream_slots)
 *   MPSG_STORE_GENERATED regenerated on the device every pass (mpsg_generated_*)
 *   MPSG_STORE_FILE      re-read from an MPSB file every pass (mpsg_create_from_file_streamed) */
#define MPSG_STORE_RESIDENT 1
#define MPSG_STORE_COMPACT 2
#define MPSG_STORE_HOST 3
#define MPSG_STORE_GENERATED 4
#define MPSG_STORE_FILE 5
int mpsg_gamma_store(mpsg_handle h);

/* The Gamma values the GPU actually samples (decoded compressed format), reference layout:
 * complex128 interleaved (chiL, chiR, d).  The CPU oracle consumes these.  A tensor-parallel
 * handle writes only its own column shard (other entries are left untouched). */
int mpsg_decoded_gamma(mpsg_handle h, uint64_t site, double* out);

/* ---- synthetic chains regenerated on the device ------------------------------------------
 * For chains whose compressed Gamma exceeds device and host memory (c4: M = 8176, chi = 1e4,
 * d = 4 is 13-20 TB), a handle can hold a random right-canonical chain of the random_mps form
 * (mps.cpp:148-175) as its generators instead of its tensors:
 *   Gamma_i[l, r, k] = B_b(i)[l, r*d + k] * phase_i[r*d + k] * Lambda_{i-1}[l] / Lambda_i[r]
 * B_b a base isometry registered once (complex64 (rows >= bond[i], cols >= bond[i+1] * d) with
 * orthonormal rows; a site uses its leading bond[i] x bond[i+1]*d block), phase_i[j] = exp(2 pi i u)
 * with u the reference's keyed uniform (rng.hpp:22-37) of (seed, 0x70686173, site i, column j),
 * and the products rounded in fp32 in that order.  Every pass regenerates and compresses each site
 * on the device into a ring of host_stream_slots (default 3) device slots, on a side stream that
 * overlaps the previous sites' contractions -- the paper's double-buffered site stream
 * (SiteStream, mps_io.cpp:294-350) with the device as the source.  Bond scales,
 * validation and compression are those of mpsg_builder_set_site, so a state built from the
 * materialised sites (mpsg_synthetic_site + mpsg_builder_set_site) samples identically. */
int mpsg_generated_begin(uint64_t num_sites, uint64_t phys_dim, const uint64_t* bond_dims,
                         const mpsg_policy* policy, const mpsg_options* opts, const int* devices,
                         int ndev, uint64_t seed, mpsg_handle* out);
/* Registers a base isometry (complex64 interleaved, rows x cols row-major; a device pointer on the
 * first listed device, or host memory); the handle keeps its own copy on every device. */
int mpsg_generated_add_base(mpsg_handle h, const void* base, int base_is_device, uint64_t rows,
                            uint64_t cols, int* base_id);
/* Site `site` (in increasing order) regenerates from base `base_id` with Lambda_site = lambda
 * (length bond[site + 1]; validated like MpsState::validate).  Finish with mpsg_builder_finish. */
int mpsg_generated_set_site(mpsg_handle h, uint64_t site, int base_id, const double* lambda);
/* The generator formula evaluated into `out` (complex64 rows x cols, device memory on the calling
 * thread's current device): base (row stride ld) as above, lambda_prev (rows; NULL = ones) and
 * lambda (cols / phys_dim) the site's bond spectra. */
int mpsg_synthetic_site(const void* base, uint64_t ld, uint64_t rows, uint64_t cols, uint64_t phys_dim,
                        const double* lambda_prev, const double* lambda, uint64_t seed, uint64_t site,
                        void* out);
/* The ORIGINAL values of site `site` of a generated handle -- the generator itself, before the
 * device compression (mpsg_decoded_gamma returns what the device samples) -- as complex128 (chiL,
 * chiR, d) in host memory: the chain a caller of the reference would hold (parity against the
 * caller's MPS, e.g. MPSG_MODE_PRECISE at the c3 / c4 shapes that exceed host memory as complex128). */
int mpsg_generated_site_values(mpsg_handle h, uint64_t site, double* out);

/* ---- MPSB files (the reference's on-disk format, mps_io.hpp:17-24) ----------------------- */
/* Read an MPSB file (any storage precision, checksums verified -> MPSG_ERR_IO) and build the
 * device state, streaming sites through a one-slot prefetch thread (SiteStream,
 * mps_io.cpp:294-350).  The file-based executors run_serial / run_data_parallel
 * (parallel.hpp:24-52) become mpsg_create_from_file + mpsg_sample. */
int mpsg_create_from_file(const char* path, const mpsg_policy* policy, const mpsg_options* opts,
                          const int* devices, int ndev, mpsg_handle* out);
/* The same file, streamed from storage on every pass instead of held: for chains larger than device
 * and host memory (c4: 13-26 TB).  Only the header and the Lambda vectors are read here; each pass a
 * reader thread preads the site payloads in chain order into pinned staging buffers and verifies
 * their checksums (the reference's SiteStream, mps_io.cpp:294-350, checksum as mps_io.cpp:120-146),
 * the copy stream uploads the raw Gamma scalars (f64 / f32 / f16 storage) and the compression
 * kernels pack them into the ring of host_stream_slots device slots (default 3) the sweep consumes.
 * Samples and marginals equal those of mpsg_create_from_file on the same file bit for bit.  A payload
 * whose checksum fails surfaces as MPSG_ERR_IO from the sampling call (the handle is then unusable).
 * mpsg_state_bytes reports the Gamma bytes read per pass. */
int mpsg_create_from_file_streamed(const char* path, const mpsg_policy* policy, const mpsg_options* opts,
                                   const int* devices, int ndev, mpsg_handle* out);
/* Write the state as an MPSB file (save_mps, mps_io.cpp:167-210): the decoded Gamma values at
 * `storage` precision (MPSG_F64 / F32 / F16) and the Lambda vectors. */
int mpsg_save_file(mpsg_handle h, const char* path, int storage);

/* ---- tensor parallelism ------------------------------------------------------------------ */
/* Per site every rank contracts its Gamma column shard with the full environment, the per-
 * (sample, outcome) (weight, max) partials are all-gathered and summed in rank order (so every
 * rank draws the same outcome), and the environment shards are all-gathered for the next site.
 * All ranks call mpsg_sample with the same range and obtain identical rows. */
/* 128-byte NCCL unique id, created on one rank and shared with the others out of band. */
int mpsg_nccl_unique_id(uint8_t id[128]);
/* Join the NCCL communicator of tp_size ranks (one process or thread per rank and device). */
int mpsg_tp_connect_nccl(mpsg_handle h, const uint8_t id[128]);
/* Group n handles of one process (ranks 0..n-1, any devices, possibly the same one) with an
 * in-process exchange instead of NCCL; each rank's mpsg_sample must run on its own thread. */
int mpsg_tp_connect_local(mpsg_handle* handles, int n);

/* ---- sampling: replaces sample_batch / sample_micro_serial ------------------------------ */
/* Samples global indices [first, first + count) with measurement seed `seed` and writes
 * rows (count x M, host memory).  Equivalent to detail::sample_micro_serial over that range
 * (sampler.cpp:129-162); with first = 0, count = N it is sample_batch (sampler.cpp:164-205)
 * for any BatchPlan, since outcomes are keyed by global sample index.  Work is split across
 * the handle's devices (one host thread each). */
int mpsg_sample(mpsg_handle h, uint64_t seed, uint64_t first, uint64_t count, uint8_t* rows,
                mpsg_stats* stats);

/* Same, writing into device memory on the first listed device (no D2H). */
int mpsg_sample_device(mpsg_handle h, uint64_t seed, uint64_t first, uint64_t count,
                       uint8_t* rows_dev, mpsg_stats* stats);

/* Teacher-forced per-site marginals: walks the GPU sweep along the given outcome strings
 * (count x M, 0xFF = dead) and writes p[n, i, k] = w[n,k] / sum_k w[n,k] (sampler.cpp:83-100)
 * as float64 count x M x d (-1 for dead).  Used for the 1e-4 marginal parity check. */
int mpsg_marginals(mpsg_handle h, uint64_t first, uint64_t count, const uint8_t* forced,
                   double* marg);

/* ---- GBS displacement: the SiteTransform hook (sampler.hpp:71-79, applied at sampler.cpp:143)
 * specialised to the paper's displacement operators (SPEC.md gbs-ops, §3.4).  mu is
 * complex128 (count, M) row-major: sample n of the range is displaced by D(mu[n][i]) at site i,
 * temp[n, b, :] <- D temp[n, b, :] between the contraction and the measurement; D(mu) =
 * exp(-|mu|^2/2) exp(mu a^dag) exp(-conj(mu) a) in closed form (exact Fock-basis elements).
 * phys_dim <= 16.  The reference's src/gbs.cpp is absent; parity is against the oracle's
 * restatement of SPEC.md:366-381 (oracle/mpsamp_oracle.c orc_displacement). */
int mpsg_sample_displaced(mpsg_handle h, uint64_t seed, uint64_t first, uint64_t count,
                          const double* mu, uint8_t* rows, mpsg_stats* stats);
int mpsg_marginals_displaced(mpsg_handle h, uint64_t first, uint64_t count, const uint8_t* forced,
                             const double* mu, double* marg);
/* expm_displacement on the device: D(mu), n x n complex128 row-major (n <= 64). */
int mpsg_displacement_matrix(double mu_re, double mu_im, uint64_t n, double* out);

/* The device RNG: draws[j] = uniform(seed, 0x6d656173, first + j, site) computed by the GPU
 * (detail::measurement_draws, sampler.cpp:120-127). */
int mpsg_device_draws(uint64_t seed, uint64_t first, uint64_t count, uint64_t site, double* out);

/* One contraction through the tcgen05 GEMM (contract_site, contract.cpp:109-121): env is
 * complex128 (count, chiL) in the reference scaling; temp receives complex128
 * (count, chiR, d) in the same scaling.  Exposed for numerics tests. */
int mpsg_contract_site(mpsg_handle h, uint64_t site, const double* env, uint64_t count,
                       double* temp);

#ifdef __cplusplus
}
#endif
#endif /* MPSG_H */
