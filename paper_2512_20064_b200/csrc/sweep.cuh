// Kernel interface of the per-site sweep step (host engine <-> device kernels).
//
// Device data layout:
//   G    fp16  [kGPlanes][Np][Kp]   compressed site tensor ([-Gi, Gr, Gi]), K-major (l contiguous);
//              output column j = k * chirp + r  (k-major so a 128-column tile is one outcome k)
//   cinfo float2 [Np]  (column scale cs_j, weight factor wl_r = (Lambda_r / gamma_r)^2)
//   env  fp16  [4 planes (hi.re, hi.im, lo.re, lo.im)][cap rows][Kp]   internal environment
//   temp float2 [rows][d][chirp]  contracted site, internal scaling, complex fp32
//   pstat float2 [rows][ntiles]   per (sample, 128-column tile): (sum wl*|t|^2, max |t| comp.)
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mpsg {

constexpr int kBM = 128;  // samples per tile (UMMA M)
constexpr int kBN = 128;  // complex output columns per tile (UMMA N per real plane)
constexpr int kBK = 32;   // K elements per pipeline stage (64 B rows, SWIZZLE_64B)
constexpr int kGemmThreads = 256;
// Compressed Gamma planes: 3 = [-Gi | Gr | Gi] (two N=256 UMMAs per K-step and env pair:
// Er x [Gr;Gi] and Ei x [-Gi;Gr]); 2 = [Gr | Gi] (four N=128 UMMAs).
#ifndef MPSG_GPLANES
#define MPSG_GPLANES 2
#endif
constexpr int kGPlanes = MPSG_GPLANES;
constexpr int kPlaneRe = kGPlanes == 3 ? 1 : 0;
constexpr int kPlaneIm = kGPlanes == 3 ? 2 : 1;
constexpr uint64_t kMeasureStream = 0x6d656173ull;  // rng.hpp:19
constexpr uint8_t kDead = 0xFF;                      // sampler.hpp:17

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

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

// Per-(sample, outcome) partials read by the select kernel: element (part, n, k) lives at
// part_base[part * part_stride + n * row_stride + k * k_stride]; parts are summed in order.
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
};

// host launchers (sweep_kernels.cu)
void launch_site_gemm(bool split, const CUtensorMap& tma_env, const CUtensorMap& tma_g,
                      const SiteGemmArgs& a, int grid, cudaStream_t s);
// CTA-pair variant (cta_group::2, M = 256 per unit; a.m_tiles counts 256-row tiles; the Gamma map
// has a 64-row box).
void launch_site_gemm_pair(bool split, const CUtensorMap& tma_env, const CUtensorMap& tma_g64,
                           const SiteGemmArgs& a, int grid, cudaStream_t s);
int gemm_pair_smem_bytes(bool split);
void launch_select(const SelectArgs& a, cudaStream_t s);
// pstat [rows][nt] -> out [rows][d]: (sum of weights, max) over the tiles of each outcome
void launch_reduce_tiles(const float2* pstat, int nt, int tiles_per_k, int d, int rows,
                         float2* out, cudaStream_t s);
// Site-0 env in the shard-major layout [shards][4][cap][kshard]: E[n][0] = 1 (shard 0).
void launch_init_env(__half* env, int env_cap, int kshard0, int shards, int rows, int count,
                     uint8_t* alive, cudaStream_t s, double* logscale = nullptr);
void launch_draws(uint64_t seed, uint64_t first, uint64_t count, uint64_t site, double* out,
                  cudaStream_t s);
// Compression of one site's column shard [b0, b0 + width) of chiR: src complex (chiL, chiR, d)
// f64 or f32 interleaved on device; row l goes to padded K position lpos[l].
void launch_compress_site(const void* src, bool src_f64, int chil, int chir, int d, int b0,
                          int width, int kp, int chirp, const int* lpos, const double* gl,
                          const double* gr, const double* wl, __half* g_out, float2* cinfo_out,
                          double* cs_out, int* err, cudaStream_t s);
int gemm_smem_bytes(bool split);

}  // namespace mpsg
