// Kernel interface of the per-site sweep step (host engine <-> device kernels).
//
// Device data layout:
//   G    fp16  [gplanes][Np][Kp]   compressed site tensor, planes [Gr, Gi] (4M) or
//              [Gr, Gi, Gs = Gr + Gi] (3M, Gs exact by construction), K-major (l contiguous);
//              output column j = k * chirp + r  (k-major so a 128-column tile is one outcome k)
//   cinfo float2 [Np]  (column scale cs_j, weight factor wl_r = (Lambda_r / gamma_r)^2)
//   env  fp16  [2 * C planes][cap rows][Kp]   internal environment, C = 2 components (re, im) for
//              4M or 3 (re, im, re + im) for 3M; planes [hi.c0 .. hi.cC-1, lo.c0 .. lo.cC-1]
//   temp float2 [rows][d][chirp]  contracted site, internal scaling, complex fp32
//   pstat float2 [rows][ntiles]   per (sample, 128-column tile): (sum wl*|t|^2, max |t| comp.)
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

namespace mpsg {

// One-time setup per (call site, device).  The dynamic-shared-memory opt-in
// (cudaFuncSetAttribute), occupancy queries and __constant__ tables are properties of a device's
// context, and a multi-device handle drives its devices from concurrent host threads, so every
// such cache is keyed by the current device and guarded by a mutex.
constexpr int kMaxDevices = 64;
struct PerDevice {
  std::mutex mu;
  int value[kMaxDevices] = {};
  bool set[kMaxDevices] = {};
  template <typename F>
  int get(F&& init) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = kMaxDevices - 1;
    std::lock_guard<std::mutex> lk(mu);
    if (!set[dev]) {
      value[dev] = init();
      set[dev] = true;
    }
    return value[dev];
  }
};
// Raises the engine's MPSG_ERR_CUDA error when a launch (or a launch attribute) failed.
void check_launch(cudaError_t e, const char* what);

constexpr int kBM = 128;  // samples per tile (UMMA M)
constexpr int kBN = 128;  // complex output columns per tile (UMMA N per real plane)
constexpr int kBK = 32;   // K elements per pipeline stage (64 B rows, SWIZZLE_64B)
constexpr int kBK3 = 64;  // 3M kernel: K elements per stage (128 B rows, SWIZZLE_128B)
constexpr int kGemmThreads = 256;
constexpr int kPlaneRe = 0;  // Gamma planes: Gr, Gi (, Gs)
constexpr int kPlaneIm = 1;
constexpr uint64_t kMeasureStream = 0x6d656173ull;  // rng.hpp:19
// The next environment is renormalised (power of two) to a max component in [2^13, 2^14): the hi/lo
// fp16 split then keeps the lo part out of the fp16 subnormal range for components down to ~1e-5 of
// the max (with a max in [0.5, 1) every component below 0.25 had a subnormal, i.e. imprecise, lo
// part).  Products stay far from fp32 overflow (|t| <= 2^14 * K).
constexpr int kEnvExp = 14;
constexpr uint8_t kDead = 0xFF;                      // sampler.hpp:17
// Parity rule: a draw within this distance of an interior CDF boundary cum_k (k < d - 1) may flip
// outcome under any rounding difference; such draws are counted on the device (mpsg_stats).
constexpr double kBoundaryEps = 1e-6;

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

#ifdef __CUDACC__
// Environment split of one renormalised entry (re, im): hi / lo fp16 parts per component, and the
// 3M sum component formed from the split parts, s = (hi_re + lo_re) + (hi_im + lo_im) rounded once in
// fp32, then split the same way.  Every writer of environment planes (selection, slice GEMM, host
// contract_site) uses it, so a tensor-parallel rank can re-form the s planes from the re / im planes
// it receives (the environment exchange ships 4 of the 3M's 6 planes) and obtain the same bits.
__host__ __device__ __forceinline__ void env_split(float re, float im, __half* hv, __half* lv) {
  hv[0] = __float2half_rn(re);
  lv[0] = __float2half_rn(re - __half2float(hv[0]));  // exact difference
  hv[1] = __float2half_rn(im);
  lv[1] = __float2half_rn(im - __half2float(hv[1]));
  const float a = __half2float(hv[0]) + __half2float(lv[0]);  // exact: 22 significant bits (adds only:
                                                             // no contraction, same bits on host and device)
  const float b = __half2float(hv[1]) + __half2float(lv[1]);
  const float sv = a + b;
  hv[2] = __float2half_rn(sv);
  lv[2] = __float2half_rn(sv - __half2float(hv[2]));
}
#endif

struct SiteGemmArgs {
  int m_tiles;       // rows / 128
  int n_tiles;       // Np / 128 (even)
  int k_blocks;      // total K blocks = shards * kshard_blocks
  int kshard_blocks; // K blocks per env shard (Kshard / 32); env TMA map is 3-D (k, row, shard)
  int plane_rows_a;  // row offset between env planes (= env capacity rows)
  int np;            // Np (row offset between G planes)
  int chirp;         // padded local chiR (multiple of 128)
  int d;
  int group_n;       // N-tile pairs per raster group
  const float2* cinfo;
  float2* temp;
  float2* pstat;
};

// 3M kernel (site_gemm_3m_kernel): D[j, n] = sum_l Gamma[j, l] E[n, l] with Gamma as the A
// operand (a CTA pair covers 256 output columns, 128 per SM) and the environment as B
// (128 samples per unit, 64 rows per SM).  Products P_c = E_c x G_c for c = re, im, s; then
// Re = P_re - P_im and Im = P_s - P_re - P_im.
struct Gemm3MArgs {
  int g_tiles;       // Np / 256 (Gamma column tiles of the pair)
  int s_tiles;       // rows / 128 (sample tiles)
  int k_blocks, kshard_blocks;
  int env_cap;       // row offset between env planes
  int np;            // row offset between Gamma planes
  int chirp, d;
  int nt;            // Np / 128: pstat row stride
  int group;         // Gamma tiles per raster group
  int flags;         // diagnostics (0 in production): 32 = clock64 timing probes (g_prof3m)
  int raster;        // unit order: 1 = snake over sample tiles, 2 = groups last-to-first (site_gemm_3m.cu)
  const float2* cinfo;
  float2* temp;      // null: weights-only contraction (slice-recompute path, no temp stores)
  float2* pstat;
  // slice GEMM (slice-recompute path): the environment rows are bucketed by outcome (rows
  // [off_k, off_k+1) drew outcome k, off = prefix sums of bcount[0..d]); only the units whose
  // sample tile meets the bucket of their Gamma columns' outcome run, and the epilogue writes the
  // next environment's hi / lo planes (row scale `scale`) instead of temp / pstat
  const int* bcount;
  const float* scale;
  __half* env_next;  // [2 * 3][env_cap][kp_next]
  int kp_next;
  int pdl;           // launched as a programmatic dependent of the previous kernel in the stream
};

// Slice-recompute path: rows of the environment scattered into outcome buckets (bucket d = dead
// from the next site), carrying their sample index, outcome, renormalisation scale and liveness.
struct PermuteArgs {
  int rows, d, planes, kp, env_cap;
  const uint8_t* rowk;
  const float* scale;
  const int* perm;
  const __half* env;
  const int* bcount;
  int* bfill;
  uint8_t* rowk2;
  float* scale2;
  int* perm2;
  uint8_t* alive2;
  __half* env2;
};

// Per-(sample, outcome) partials read by the select kernel: element (part, n, k) lives at
// part_base[part * part_stride + n * row_stride + k * k_stride]; parts are summed in order.
// Reference operand grids (MPSG_MODE_GRID): the reduced compute policies' round_scalar
// (precision.cpp:23-50) applied to Gamma and to every environment, component-wise.
//   kGridF16:  IEEE binary16 (10-bit significand, normal exponents from -14, subnormals, overflow to
//              inf) on the reference's own values -- no bond, column or per-sample scaling
//   kGridTF32: 10-bit significand, f32 exponent range -- scale-invariant, so Gamma keeps its
//              power-of-two bond / column scales (column max in [2^14, 2^15)) and the environment its
//              per-sample power of two; the rounding sees the reference's value times a power of two
constexpr int kGridNone = 0, kGridF16 = 1, kGridTF32 = 2;

struct SelectArgs {
  int site, num_sites, d;
  int chir_loc;             // live local columns of the slice (this rank's shard width)
  int chirp;                // padded local chiR (temp row stride per outcome)
  int parts;                // number of partials per (n, k)
  long long part_stride, row_stride, k_stride;
  int rows;                 // samples handled this pass (multiple of 128 >= count)
  int count;                // live samples this pass
  int kp_next;              // width of this rank's next-env shard (0 on the last site)
  int env_cap;              // env plane stride in rows
  int env_comp;             // env components per precision half: 2 (re, im) or 3 (re, im, re+im)
  int slice_max;            // 1: the renormalisation max comes from the chosen slice, not the partials
  uint64_t seed, first;
  const float2* temp;
  const float2* part_base;
  uint8_t* alive;
  uint8_t* rows_out;        // [count][num_sites] (device)
  __half* env_next;         // this rank's shard of the next env: [4][env_cap][kp_next]
  const uint8_t* forced;    // optional [count][num_sites] teacher forcing
  double* marg;             // optional [count][num_sites][d]
  // decay trace (sampler.cpp:149-153): optional.  logscale[n] = ln(E_int / (env_ref * gamma)) per
  // sample; inv_gamma[r] = 1 / gamma_i[r] (local columns); trace accumulates sum |env_ref|.
  double* logscale;
  const double* inv_gamma;
  double* trace;
  int scaling;              // reference ScalingMode for the logscale update (precision.cpp:135-165)
  int grid;                 // kGrid*: round the next environment onto the reference policy's grid
  // GBS displacement fused into the selection (tp == 1, no decay trace): the weights, the draw and
  // the gathered slice use D(mu[n]) temp[n, :, r] computed on the fly from the d stored outcomes
  const double2* mu;        // [rows][num_sites] or null
  const float2* cinfo;      // site column info (wl_r = cinfo[r].y) for the displaced weights
  unsigned long long* live; // optional: += number of live samples measured at this site (RunStats)
  unsigned long long* near; // optional: += number of draws within kBoundaryEps of an interior CDF
                            // boundary at this site (the north star's "counted and reported" rule)
  // slice-recompute path: row n holds sample perm[n] of the pass (null: identity); with rowk set the
  // kernel records (outcome or d = dead next, scale) per row and counts the buckets instead of
  // writing the next environment (the slice GEMM does)
  const int* perm;
  uint8_t* rowk;
  float* scale_out;
  int* bcount;              // [d + 1]
  int pdl;                  // launched as a programmatic dependent (select4_kernel only)
};

// GBS displacement site transform (SPEC.md gbs-ops; the hook of sampler.cpp:143): for every live
// sample n and local column r, temp[n, :, r] <- D(mu[n]) temp[n, :, r], then the per-(sample, tile)
// Born-weight partials and max are recomputed into pstat.
constexpr int kMaxDisplacedDim = 16;
struct DisplaceArgs {
  int d, chirp, chir_loc, nt, tpk;  // tpk = chirp / 128 tiles per outcome
  int rows, count;
  int site, num_sites;
  const double2* mu;                // [rows][num_sites] displacement amplitudes of this pass
  const uint8_t* alive;
  const float2* cinfo;              // site column info: wl_r = cinfo[r].y
  float2* temp;
  float2* pstat;
};

// host launchers (sweep_kernels.cu)
void launch_displace(const DisplaceArgs& a, cudaStream_t s);
// D(mu) (n x n, f64, row-major complex) computed by the device generator.
void launch_displacement_matrix(double mu_re, double mu_im, int n, double2* out, cudaStream_t s);
void launch_site_gemm(bool split, const CUtensorMap& tma_env, const CUtensorMap& tma_g,
                      const SiteGemmArgs& a, int grid, cudaStream_t s);
// CTA-pair variant (cta_group::2, M = 256 per unit; a.m_tiles counts 256-row tiles; the Gamma map
// has a 64-row box).
void launch_site_gemm_pair(bool split, const CUtensorMap& tma_env, const CUtensorMap& tma_g64,
                           const SiteGemmArgs& a, int grid, cudaStream_t s);
int gemm_pair_smem_bytes(bool split);
// 3M kernel: tma_g has a 64 x 128-row box over [3][Np][Kp], tma_env a 64 x 64-row box over the
// 6-plane env, both SWIZZLE_128B; Kp and the env shard width are multiples of 64.
// with_max: also the per-(sample, tile) max component in pstat.y (tensor parallelism); otherwise
// pstat.y is 0 and the select kernel computes the chosen slice's max (SelectArgs::slice_max).
// epi_warps: 4 or 8 epilogue warps (one or two per TMEM lane quarter).
// quad: 4-CTA clusters sharing the environment tiles by multicast (see site_gemm_3m.cu).
// glo: Gamma lo planes present (MPSG_MODE_PRECISE, split only).
// slice = true: the slice GEMM of the slice-recompute path (Gemm3MArgs::bcount / scale / env_next)
// tma_temp: a 3-D map of temp ({chirp, d, rows} float2, box 32 x 1 x 8) -> the epilogue stores temp
// with TMA tensor stores (8-warp SPLIT / SINGLE K1); null -> per-thread global stores
void launch_site_gemm_3m(bool split, bool with_max, int epi_warps, bool quad, bool glo,
                         const CUtensorMap& tma_env64, const CUtensorMap& tma_g, const Gemm3MArgs& a,
                         int grid, cudaStream_t s, bool slice = false, const CUtensorMap* tma_temp = nullptr);
int gemm_3m_smem_bytes(bool split);
void launch_select(const SelectArgs& a, cudaStream_t s);
// env [shards][6][env_cap][kshard] (3M): planes 2, 5 (s = re + im, hi / lo) of rows [0, rows) of every
// shard re-formed from planes 0, 1, 3, 4 exactly as env_split forms them (kshard % 8 == 0)
void launch_env_reform_s(__half* env, int env_cap, int kshard, int shards, int rows, cudaStream_t s);
void launch_permute_rows(const PermuteArgs& a, cudaStream_t s);
// zeroes rows [sum(bcount[0..d)), rows) of the next environment (the samples dead from there on)
void launch_zero_dead(__half* env, int planes, int env_cap, int kp, int rows, const int* bcount, int d,
                      cudaStream_t s);
// pstat [rows][nt] -> out [rows][d]: (sum of weights, max) over the tiles of each outcome
void launch_reduce_tiles(const float2* pstat, int nt, int tiles_per_k, int d, int rows,
                         float2* out, cudaStream_t s);
// Site-0 env in the shard-major layout [shards][2C][cap][kshard]: E[n][0] = 1 (shard 0) in the
// hi.re plane and, for C = 3, the hi.s plane.
void launch_init_env(__half* env, int env_comp, int env_cap, int kshard0, int shards, int rows,
                     int count, uint8_t* alive, cudaStream_t s, double* logscale = nullptr,
                     int* perm = nullptr);
void launch_draws(uint64_t seed, uint64_t first, uint64_t count, uint64_t site, double* out,
                  cudaStream_t s);
// Compression of one site's column shard [b0, b0 + width) of chiR: src complex (chiL, chiR, d)
// f64 or f32 interleaved on device; row l goes to padded K position lpos[l].
// g[2 pe + j] = g[j] + g[pe + j]: re-forms the 3M sum plane Gs = Gr + Gi of a host-streamed site
// (exact: quantize_pair puts Gr, Gi and their sum on one fp16 grid).  pe % 8 == 0.
void launch_sum_plane(__half* g, size_t pe, cudaStream_t s);
// colmax: [width * d] zero-initialised scratch (left zeroed).  src_prec: the source scalars, complex
// interleaved -- kSrcF64 / kSrcF32 / kSrcF16 (the MPSB storage precisions, mps_io.cpp:167-199).
constexpr int kSrcF64 = 0, kSrcF32 = 1, kSrcF16 = 3;  // = MPSG_F64, MPSG_F32, MPSG_F16
void launch_compress_site(const void* src, int src_prec, int chil, int chir, int d, int b0,
                          int width, int kp, int chirp, const int* lpos, const double* gl,
                          const double* gr, const double* wl, int gplanes, __half* g_out,
                          float2* cinfo_out, double* cs_out, unsigned long long* colmax, int* err,
                          cudaStream_t s, int grid = kGridNone);

// Synthetic chains regenerated on the device (mpsg_generated_*, mpsg_synthetic_site): the random_mps
// form (mps.cpp:148-175) Gamma_i[l, r*d + k] = B[l, r*d + k] * phase_i[r*d + k] *
// lambda_{i-1}[l] / lambda_i[r] with B a base isometry (rows orthonormal) and unit phases keyed by
// (seed, kPhaseStream, site, column) with the reference's counter-based key chain (rng.hpp:22-37).
constexpr uint64_t kPhaseStream = 0x70686173ull;  // "phas"
struct SynthSite {
  const float2* base;     // B, complex64 (>= chil rows, row stride ld)
  long long ld;           // row stride of B (complex elements)
  long long cols;         // chir * d
  const float2* phase;    // [cols] this site's phases (launch_synth_phase)
  const float* lam_prev;  // [chil] fp32 lambda_{i-1} (ones(1) at site 0)
  const float* inv_lam;   // [chir] fp32 1 / lambda_i (rounded on the host)
  int d;
};
void launch_synth_phase(uint64_t seed, uint64_t site, int cols, float2* phase, cudaStream_t s);
// out: complex64 (rows, cols) row-major = the site's Gamma
void launch_synth_values(const SynthSite& g, int rows, float2* out, cudaStream_t s);
// compression of a regenerated site's column shard, straight from the generator (no Gamma buffer)
void launch_compress_synth(const SynthSite& g, int chil, int d, int b0, int width, int kp, int chirp,
                           const int* lpos, const double* gl, const double* gr, const double* wl, int gplanes,
                           __half* g_out, float2* cinfo_out, double* cs_out, unsigned long long* colmax,
                           int* err, cudaStream_t s);
int gemm_smem_bytes(bool split);

}  // namespace mpsg
