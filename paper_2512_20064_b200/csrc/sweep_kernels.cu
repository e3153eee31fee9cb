// Per-site sweep kernels for sm_100a.
//
//   K1 site_gemm_kernel   temp = env x Gamma_i on tcgen05 (TMA -> smem -> UMMA -> TMEM), complex
//                         4M decomposition with the sign folded into the instruction descriptor,
//                         fused measurement epilogue: per (sample, 128-column tile) partial Born
//                         weight sum wl_r |t|^2 and max component, temp stored k-major.
//                         Reference: contract_site (contract.cpp:18-41,109-121) + the weight loop
//                         of measure (sampler.cpp:83-90) + partial_measure_stats (parallel.cpp:90-114).
//   K2 select_kernel      per sample: reduce partials (f64), keyed draw (rng.hpp:22-37), f64 CDF
//                         search with strict '>' and clamp (sampler.cpp:92-107), dead handling,
//                         gather of the chosen slice (sampler.cpp:110-111), power-of-two
//                         renormalisation (precision.cpp:152-163) and hi/lo fp16 split into the
//                         next site's GEMM operand.
//   init / draws / compress helpers.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <type_traits>

#include "ptx.cuh"


#include "sweep.cuh"

namespace mpsg {

// ============================================================================================
// RNG (rng.hpp:12-37), bit-exact with the reference.
// ============================================================================================
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double keyed_uniform(uint64_t seed, uint64_t stream, uint64_t sample,
                                                uint64_t site) {
  uint64_t h = mix64(seed ^ (stream * 0xD6E8FEB86659FD93ull));
  h = mix64(h ^ (sample * 0xA5A5A5A5A5A5A5A5ull));
  h = mix64(h ^ (site * 0xC2B2AE3D27D4EB4Full));
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

// ============================================================================================
// K1: tcgen05 complex GEMM + fused measurement epilogue
// ============================================================================================
template <bool kSplit>
struct GemmCfg {
  static constexpr int kAPlanes = kSplit ? 4 : 2;  // env planes: hi.re hi.im [lo.re lo.im]
  static constexpr int kTile = kBM * kBK * 2;      // 8 KiB: 128 rows x 64 B (A and B alike)
  static constexpr int kStageBytes = (kAPlanes + 2) * kTile;
  static constexpr int kStages = kSplit ? 4 : 6;
  static constexpr int kBarrierBytes = 256;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + kBarrierBytes;
  static_assert(kBM == 128 && kBN == 128 && kBK == 32, "tile shape baked into descriptors");
};

int gemm_smem_bytes(bool split) { return split ? GemmCfg<true>::kSmem : GemmCfg<false>::kSmem; }

// Work unit = (M tile, pair of N tiles); the two CTAs of a cluster share the unit's env (A) tiles
// through TMA multicast and each computes one of the two N tiles.  Units are rastered in groups
// of `group_n` N-tile pairs so concurrently running clusters reuse Gamma tiles from L2.
__device__ __forceinline__ void unit_coords(int u, const SiteGemmArgs& a, int& m, int& np) {
  const int pairs = a.n_tiles >> 1;
  const int per_group = a.group_n * a.m_tiles;
  const int g = u / per_group;
  const int n0 = g * a.group_n;
  const int gw = min(a.group_n, pairs - n0);
  const int r = u - g * per_group;
  m = r / gw;
  np = n0 + (r - m * gw);
}

template <bool kSplit>
__global__ void __launch_bounds__(kGemmThreads, 1)
    site_gemm_kernel(const __grid_constant__ CUtensorMap tma_env,
                     const __grid_constant__ CUtensorMap tma_g, const SiteGemmArgs a) {
  using C = GemmCfg<kSplit>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = static_cast<int>(ptx::cluster_ctarank());  // 0 / 1 within the CTA pair
  const int cluster = blockIdx.x >> 1;
  const int num_clusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);   // own producer's expect_tx; bytes arrive from both CTAs
      ptx::mbar_init(&empty[s], 2);  // released by the MMA commits of both CTAs
    }
    for (int j = 0; j < 2; ++j) {
      ptx::mbar_init(&tfull[j], 1);
      ptx::mbar_init(&tempty[j], 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tma_env);
    ptx::tma_prefetch_desc(&tma_g);
  }
  if (warp == 2) {
    ptx::tmem_alloc(tmem_slot, 512);  // 2 accumulator stages x (re 128 + im 128) fp32 columns
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // peer barriers initialised before any multicast / remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int units = a.m_tiles * (a.n_tiles >> 1);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol_env = ptx::l2_policy_evict_normal();  // re-read by every N pair of the group
      const uint64_t pol_g = ptx::l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cluster; u < units; u += num_clusters) {
        int m, np;
        unit_coords(u, a, m, np);
        const int n = 2 * np + rank;
        int shard = 0, kin = 0;  // K block kb = shard * kshard_blocks + kin
        for (int kb = 0; kb < a.k_blocks; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);  // free in both CTAs
          uint8_t* st = smem + stage * C::kStageBytes;
          ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
#pragma unroll
          for (int q = rank; q < C::kAPlanes; q += 2)  // this CTA's half of the env planes
            ptx::tma_load_3d_mc(&tma_env, &full[stage], st + q * C::kTile, kin * kBK,
                                q * a.plane_rows_a + m * kBM, shard, 0x3, pol_env);
#pragma unroll
          for (int p = 0; p < 2; ++p)
            ptx::tma_load_2d(&tma_g, &full[stage], st + (C::kAPlanes + p) * C::kTile, kb * kBK,
                             p * a.np + n * kBN, pol_g);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
          if (++kin == a.kshard_blocks) {
            kin = 0;
            ++shard;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread) ----------------
    if (lane == 0) {
      constexpr uint32_t kId = ptx::idesc_f16_f32(kBM, kBN, false);
      constexpr uint32_t kIdNeg = ptx::idesc_f16_f32(kBM, kBN, true);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cluster; u < units; u += num_clusters) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_re = tmem_base + acc * 256;
        const uint32_t d_im = d_re + 128;
        for (int kb = 0; kb < a.k_blocks; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t st = ptx::smem_u32(smem + stage * C::kStageBytes);
#pragma unroll
          for (int ks = 0; ks < kBK / 16; ++ks) {
            const uint32_t off = ks * 32;  // 16 fp16 along K
            const uint32_t accum = (kb | ks) ? 1u : 0u;
            const uint64_t br = ptx::sdesc_kmajor_sw64(st + (C::kAPlanes + 0) * C::kTile + off);
            const uint64_t bi = ptx::sdesc_kmajor_sw64(st + (C::kAPlanes + 1) * C::kTile + off);
            // Re += Er.Gr - Ei.Gi ; Im += Er.Gi + Ei.Gr.  The Er tile feeds two consecutive MMAs
            // through the A collector; no collector for the Ei pair (reuse combined with an operand
            // negation gives wrong results).
#pragma unroll
            for (int h = 0; h < (kSplit ? 2 : 1); ++h) {
              const uint32_t acc0 = h ? 1u : accum;
              const uint64_t ar = ptx::sdesc_kmajor_sw64(st + (2 * h + 0) * C::kTile + off);
              const uint64_t ai = ptx::sdesc_kmajor_sw64(st + (2 * h + 1) * C::kTile + off);
              ptx::umma_f16_ss_afill(d_re, ar, br, kId, acc0);
              ptx::umma_f16_ss_alast(d_im, ar, bi, kId, acc0);
              ptx::umma_f16_ss(d_re, ai, bi, kIdNeg, 1u);
              ptx::umma_f16_ss(d_im, ai, br, kId, 1u);
            }
          }
          ptx::umma_commit_mc(&empty[stage], 0x3);  // slot free in both CTAs once MMAs retire
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> (weights, max, temp) ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = cluster; u < units; u += num_clusters) {
      int m, np;
      unit_coords(u, a, m, np);
      const int n = 2 * np + rank;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int row = m * kBM + q * 32 + lane;
      const int col0 = n * kBN;
      const int k = col0 / a.chirp;
      if (k < a.d) {  // the N padding tile (odd tile count) has nothing to store
        const int r0 = col0 - k * a.chirp;
        float2* dst = a.temp + (static_cast<size_t>(row) * a.d + k) * a.chirp + r0;
        const float2* ci = a.cinfo + col0;
        const uint32_t tb = tmem_base + acc * 256 + (static_cast<uint32_t>(q * 32) << 16);
        float w = 0.f, mx = 0.f;
#pragma unroll 1
        for (int c = 0; c < kBN / 32; ++c) {
          float re[32], im[32];
          ptx::tmem_ld_32x32b_x32(tb + c * 32, re);
          ptx::tmem_ld_32x32b_x32(tb + 128 + c * 32, im);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float4 cc = *reinterpret_cast<const float4*>(ci + c * 32 + j);  // (cs0, wl0, cs1, wl1)
            const float tr0 = re[j] * cc.x, ti0 = im[j] * cc.x;
            const float tr1 = re[j + 1] * cc.z, ti1 = im[j + 1] * cc.z;
            w = fmaf(cc.y, fmaf(tr0, tr0, ti0 * ti0), w);
            w = fmaf(cc.w, fmaf(tr1, tr1, ti1 * ti1), w);
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(tr0), fabsf(ti0)), fmaxf(fabsf(tr1), fabsf(ti1))));
            *reinterpret_cast<float4*>(dst + c * 32 + j) = make_float4(tr0, ti0, tr1, ti1);
          }
        }
        a.pstat[static_cast<size_t>(row) * a.n_tiles + n] = make_float2(w, mx);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // no remote arrive / multicast may target an exited peer
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, 512);
  }
}

template <bool kSplit>
static void launch_gemm_t(const CUtensorMap& tma_env, const CUtensorMap& tma_g,
                          const SiteGemmArgs& a, int grid, cudaStream_t s) {
  static PerDevice attr;
  attr.get([] {
    check_launch(cudaFuncSetAttribute(site_gemm_kernel<kSplit>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      GemmCfg<kSplit>::kSmem), "site_gemm_kernel smem opt-in");
    return 1;
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = GemmCfg<kSplit>::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  check_launch(cudaLaunchKernelEx(&cfg, site_gemm_kernel<kSplit>, tma_env, tma_g, a), "site_gemm_kernel");
}

void launch_site_gemm(bool split, const CUtensorMap& tma_env, const CUtensorMap& tma_g,
                      const SiteGemmArgs& a, int grid, cudaStream_t s) {
  grid = (grid + 1) & ~1;  // whole CTA pairs
  if (split)
    launch_gemm_t<true>(tma_env, tma_g, a, grid, s);
  else
    launch_gemm_t<false>(tma_env, tma_g, a, grid, s);
}

// --------------------------------------------------------------------------------------------
// K1 (pair): the CTA pair issues one M=256 UMMA (cta_group::2): each SM stores and reads its own
// 128 env rows and half (64 rows) of the Gamma tile, halving the per-SM shared-memory traffic of
// the B operand.  Unit = (256-row M tile, 128-column N tile).
// --------------------------------------------------------------------------------------------
template <bool kSplit>
struct PairCfg {
  static constexpr int kAPlanes = kSplit ? 4 : 2;
  static constexpr int kATile = kBM * kBK * 2;         // 8 KiB: 128 rows x 64 B
  static constexpr int kBTile = (kBN / 2) * kBK * 2;   // 4 KiB: this CTA's 64 of the 128 B rows
  static constexpr int kStageBytes = kAPlanes * kATile + 2 * kBTile;
  static constexpr int kStages = kSplit ? 5 : 8;
  static constexpr int kCinfoBytes = 2 * kBN * 8;  // double-buffered column info of the tile
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256 + kCinfoBytes;
};

int gemm_pair_smem_bytes(bool split) { return split ? PairCfg<true>::kSmem : PairCfg<false>::kSmem; }

__device__ __forceinline__ void unit_coords_pair(int u, const SiteGemmArgs& a, int& m, int& n) {
  const int per_group = a.group_n * a.m_tiles;
  const int g = u / per_group;
  const int n0 = g * a.group_n;
  const int gw = min(a.group_n, a.n_tiles - n0);
  const int r = u - g * per_group;
  m = r / gw;
  n = n0 + (r - m * gw);
}

// a.m_tiles counts 256-row tiles here.
template <bool kSplit>
__global__ void __launch_bounds__(kGemmThreads, 1)
    site_gemm_pair_kernel(const __grid_constant__ CUtensorMap tma_env,
                          const __grid_constant__ CUtensorMap tma_g64, const SiteGemmArgs a) {
  using C = PairCfg<kSplit>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float2* s_cinfo = reinterpret_cast<float2*>(smem + C::kStages * C::kStageBytes + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = static_cast<int>(ptx::cluster_ctarank());
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int num_clusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);   // leader: own expect_tx, bytes from both CTAs
      ptx::mbar_init(&empty[s], 1);  // the leader's multicast commit
    }
    for (int j = 0; j < 2; ++j) {
      ptx::mbar_init(&tfull[j], 1);
      ptx::mbar_init(&tempty[j], 8);  // leader: one arrival per epilogue warp of both CTAs
    }
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tma_env);
    ptx::tma_prefetch_desc(&tma_g64);
  }
  if (warp == 2) {
    ptx::tmem_alloc_pair(tmem_slot, 512);
    ptx::tmem_relinquish_pair();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int units = a.m_tiles * a.n_tiles;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; bytes counted on the leader's barrier) ----------
    if (lane == 0) {
      const uint64_t pol_env = ptx::l2_policy_evict_normal();
      const uint64_t pol_g = ptx::l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cluster; u < units; u += num_clusters) {
        int m, n;
        unit_coords_pair(u, a, m, n);
        int shard = 0, kin = 0;
        for (int kb = 0; kb < a.k_blocks; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * C::kStageBytes;
          const uint32_t lbar = ptx::leader_bar(&full[stage]);
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
#pragma unroll
          for (int q = 0; q < C::kAPlanes; ++q)
            ptx::tma_load_3d_pair(&tma_env, lbar, st + q * C::kATile, kin * kBK,
                                  q * a.plane_rows_a + m * 2 * kBM + rank * kBM, shard, pol_env);
#pragma unroll
          for (int p = 0; p < 2; ++p)
            ptx::tma_load_2d_pair(&tma_g64, lbar, st + C::kAPlanes * C::kATile + p * C::kBTile,
                                  kb * kBK, p * a.np + n * kBN + rank * (kBN / 2), pol_g);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
          if (++kin == a.kshard_blocks) {
            kin = 0;
            ++shard;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the leader CTA's warp 1 drives both SMs ----------------
    // The whole warp runs the loop with warp-uniform operands; one elected lane issues (no per-MMA
    // R2UR waterfall, as in the 3M kernel).
    if (leader) {
      constexpr uint32_t kId = ptx::idesc_f16_f32(2 * kBM, kBN, false);
      constexpr uint32_t kIdNeg = ptx::idesc_f16_f32(2 * kBM, kBN, true);
      const uint64_t desc0 = ptx::sdesc_kmajor_sw64(ptx::smem_u32(smem));
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cluster; u < units; u += num_clusters) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_re = tmem_base + acc * 256;
        const uint32_t d_im = d_re + 128;
        for (int kb = 0; kb < a.k_blocks; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint64_t st = desc0 + ((stage * C::kStageBytes) >> 4);  // 16 B units
#pragma unroll
          for (int ks = 0; ks < kBK / 16; ++ks) {
            const uint64_t off = 2 * ks;  // 32 B per K16 step inside the 64 B swizzle row
            const uint64_t br = st + ((C::kAPlanes * C::kATile) >> 4) + off;
            const uint64_t bi = br + (C::kBTile >> 4);
            const uint32_t accum = (kb | ks) ? 1u : 0u;
#pragma unroll
            for (int h = 0; h < (kSplit ? 2 : 1); ++h) {
              const uint32_t acc0 = h ? 1u : accum;
              const uint64_t ar = st + (((2 * h + 0) * C::kATile) >> 4) + off;
              const uint64_t ai = st + (((2 * h + 1) * C::kATile) >> 4) + off;
              ptx::umma_pair_elect(d_re, ar, br, kId, acc0, true, false);
              ptx::umma_pair_elect(d_im, ar, bi, kId, acc0, false, true);
              ptx::umma_pair_elect(d_re, ai, bi, kIdNeg, 1u, false, false);
              ptx::umma_pair_elect(d_im, ai, br, kId, 1u, false, false);
            }
          }
          ptx::umma_commit_pair_mc_elect(&empty[stage], 0x3);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma_commit_pair_mc_elect(&tfull[acc], 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs, each on its own 128 rows) ----------------
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    const int et = threadIdx.x - 128;  // epilogue thread 0..127
    for (int u = cluster; u < units; u += num_clusters) {
      int m, n;
      unit_coords_pair(u, a, m, n);
      const int col0 = n * kBN;
      // stage this tile's (cs, wl) column info in shared memory before the accumulator is ready
      float2* ci = s_cinfo + acc * kBN;
      ci[et] = a.cinfo[col0 + et];
      asm volatile("bar.sync 1, 128;" ::: "memory");
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int row = m * 2 * kBM + rank * kBM + q * 32 + lane;
      const int k = col0 / a.chirp;
      if (k < a.d) {
        const int r0 = col0 - k * a.chirp;
        float2* dst = a.temp + (static_cast<size_t>(row) * a.d + k) * a.chirp + r0;
        const uint32_t tb = tmem_base + acc * 256 + (static_cast<uint32_t>(q * 32) << 16);
        float w = 0.f, mx = 0.f;
#pragma unroll 1
        for (int c = 0; c < kBN / 32; ++c) {
          float re[32], im[32];
          ptx::tmem_ld_32x32b_x32(tb + c * 32, re);
          ptx::tmem_ld_32x32b_x32(tb + 128 + c * 32, im);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float4 cc = *reinterpret_cast<const float4*>(ci + c * 32 + j);
            const float tr0 = re[j] * cc.x, ti0 = im[j] * cc.x;
            const float tr1 = re[j + 1] * cc.z, ti1 = im[j + 1] * cc.z;
            w = fmaf(cc.y, fmaf(tr0, tr0, ti0 * ti0), w);
            w = fmaf(cc.w, fmaf(tr1, tr1, ti1 * ti1), w);
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(tr0), fabsf(ti0)), fmaxf(fabsf(tr1), fabsf(ti1))));
            *reinterpret_cast<float4*>(dst + c * 32 + j) = make_float4(tr0, ti0, tr1, ti1);
          }
        }
        a.pstat[static_cast<size_t>(row) * a.n_tiles + n] = make_float2(w, mx);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_remote_relaxed(&tempty[acc], 0);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair(tmem_base, 512);
  }
}

template <bool kSplit>
static void launch_gemm_pair_t(const CUtensorMap& tma_env, const CUtensorMap& tma_g64,
                               const SiteGemmArgs& a, int grid, cudaStream_t s) {
  static PerDevice attr;
  attr.get([] {
    check_launch(cudaFuncSetAttribute(site_gemm_pair_kernel<kSplit>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      PairCfg<kSplit>::kSmem), "site_gemm_pair_kernel smem opt-in");
    return 1;
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = PairCfg<kSplit>::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  check_launch(cudaLaunchKernelEx(&cfg, site_gemm_pair_kernel<kSplit>, tma_env, tma_g64, a), "site_gemm_pair_kernel");
}

void launch_site_gemm_pair(bool split, const CUtensorMap& tma_env, const CUtensorMap& tma_g64,
                           const SiteGemmArgs& a, int grid, cudaStream_t s) {
  grid = (grid + 1) & ~1;
  if (split)
    launch_gemm_pair_t<true>(tma_env, tma_g64, a, grid, s);
  else
    launch_gemm_pair_t<false>(tma_env, tma_g64, a, grid, s);
}

// ============================================================================================
// GBS displacement (§3.4 Eq. 6): D(mu) = exp(-|mu|^2/2) L U with the
// closed-form triangular factors L = exp(mu a^dag), U = exp(-conj(mu) a); applied per sample to the
// d outcome components of every column of temp (the reference's SiteTransform hook position,
// sampler.cpp:143).  The closed form gives the exact Fock-basis elements of D(mu) (no truncation
// of the generator).
// ============================================================================================
// c_fact[a][b] = sqrt(a! / b!) / (a - b)! for b <= a <= 64 (the closed-form factors of L and U)
// (a __constant__ symbol exists once per device: the table is uploaded to every device it runs on)
__constant__ double c_fact[65][65];
static void ensure_fact_table() {
  static PerDevice ready;
  ready.get([] {
    static double h[65][65];
    for (int a = 0; a <= 64; ++a)
      for (int b = 0; b <= 64; ++b)
        h[a][b] = b <= a ? std::exp(0.5 * (std::lgamma(a + 1.0) - std::lgamma(b + 1.0)) - std::lgamma(a - b + 1.0)) : 0.0;
    check_launch(cudaMemcpyToSymbol(c_fact, h, sizeof(h)), "displacement factorial table upload");
    return 1;
  });
}

__device__ __forceinline__ double2 displacement_element(double mr, double mi, int a, int c) {
  // D[a][c] = exp(-|mu|^2/2) sum_{b <= min(a, c)} L[a][b] U[b][c]
  const double pre = exp(-0.5 * (mr * mr + mi * mi));
  double sr = 0.0, si = 0.0;
  const int bmax = min(a, c);
  for (int b = 0; b <= bmax; ++b) {
    double lr = 1.0, li = 0.0, ur = 1.0, ui = 0.0;
    for (int j = 0; j < a - b; ++j) {  // mu^(a-b)
      const double t = lr * mr - li * mi;
      li = lr * mi + li * mr;
      lr = t;
    }
    for (int j = 0; j < c - b; ++j) {  // (-conj(mu))^(c-b) = (-mr + i mi)^(c-b)
      const double t = -ur * mr - ui * mi;
      ui = ur * mi - ui * mr;
      ur = t;
    }
    const double fl = c_fact[a][b];
    const double fu = c_fact[c][b];
    lr *= fl, li *= fl, ur *= fu, ui *= fu;
    sr += lr * ur - li * ui;
    si += lr * ui + li * ur;
  }
  return make_double2(pre * sr, pre * si);
}

__global__ void displacement_matrix_kernel(double mr, double mi, int n, double2* out) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) out[e] = displacement_element(mr, mi, e / n, e % n);
}

void launch_displacement_matrix(double mu_re, double mu_im, int n, double2* out, cudaStream_t s) {
  ensure_fact_table();
  displacement_matrix_kernel<<<1, 256, 0, s>>>(mu_re, mu_im, n, out);
}

// One warp per sample: D(mu_n) into shared memory (f64 generation, fp32 apply), then per 128-column
// tile the transformed components, their Born-weight partials and max (fixed-order warp trees).
template <int MAXD>
__global__ void __launch_bounds__(256) displace_kernel(const DisplaceArgs a) {
  __shared__ float2 sD[8][MAXD * MAXD];
  const int wib = threadIdx.x >> 5;
  const int n = blockIdx.x * 8 + wib;
  const int lane = threadIdx.x & 31;
  if (n >= a.count || !a.alive[n]) return;  // warp-uniform
  const int d = a.d;
  const double2 mu = a.mu[static_cast<size_t>(n) * a.num_sites + a.site];
  for (int e = lane; e < d * d; e += 32) {
    const double2 v = displacement_element(mu.x, mu.y, e / d, e % d);
    sD[wib][e] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
  }
  __syncwarp();
  const float2* D = sD[wib];
  float2* row = a.temp + static_cast<size_t>(n) * d * a.chirp;  // [d][chirp]
  for (int t = 0; t < a.tpk; ++t) {
    float w[MAXD], mx[MAXD];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) w[k] = 0.f, mx[k] = 0.f;
    for (int j = 0; j < 4; ++j) {
      const int r = t * 128 + j * 32 + lane;
      if (r >= a.chir_loc) continue;
      float2 v[MAXD];
#pragma unroll
      for (int k = 0; k < MAXD; ++k)
        if (k < d) v[k] = row[static_cast<size_t>(k) * a.chirp + r];
      const float wl = a.cinfo[r].y;
#pragma unroll
      for (int k = 0; k < MAXD; ++k) {
        if (k >= d) break;
        float orr = 0.f, oi = 0.f;
#pragma unroll
        for (int q = 0; q < MAXD; ++q) {
          if (q >= d) break;
          const float2 dk = D[k * d + q];
          orr = fmaf(dk.x, v[q].x, fmaf(-dk.y, v[q].y, orr));
          oi = fmaf(dk.x, v[q].y, fmaf(dk.y, v[q].x, oi));
        }
        row[static_cast<size_t>(k) * a.chirp + r] = make_float2(orr, oi);
        w[k] = fmaf(wl, fmaf(orr, orr, oi * oi), w[k]);
        mx[k] = fmaxf(mx[k], fmaxf(fabsf(orr), fabsf(oi)));
      }
    }
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
      if (k >= d) break;
      float ws = w[k], ms = mx[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ws += __shfl_xor_sync(0xffffffffu, ws, o);
        ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
      }
      if (lane == 0) a.pstat[static_cast<size_t>(n) * a.nt + k * a.tpk + t] = make_float2(ws, ms);
    }
  }
}

void launch_displace(const DisplaceArgs& a, cudaStream_t s) {
  ensure_fact_table();
  if (a.d <= 8)
    displace_kernel<8><<<(a.count + 7) / 8, 256, 0, s>>>(a);
  else
    displace_kernel<kMaxDisplacedDim><<<(a.count + 7) / 8, 256, 0, s>>>(a);
}

// ============================================================================================
// K2: measurement select + gather + renormalise + split (one warp per sample)
// ============================================================================================
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Born weight of outcome k for sample n: fixed-order f64 reduction of its partials.
__device__ __forceinline__ double outcome_weight(const SelectArgs& a, int n, int k, int lane) {
  const float2* base = a.part_base + n * a.row_stride + k * a.k_stride;
  double s = 0.0;
  for (int t = lane; t < a.parts; t += 32) s += static_cast<double>(base[t * a.part_stride].x);
  return warp_sum(s);
}
__device__ __forceinline__ float outcome_max(const SelectArgs& a, int n, int k, int lane) {
  const float2* base = a.part_base + n * a.row_stride + k * a.k_stride;
  float m = 0.f;
  for (int t = lane; t < a.parts; t += 32) m = fmaxf(m, base[t * a.part_stride].y);
  return warp_max(m);
}

// max component of the chosen (contiguous) temp slice of sample n, outcome k
__device__ __forceinline__ float slice_max(const SelectArgs& a, int n, int k, int lane) {
  const float2* src = a.temp + (static_cast<size_t>(n) * a.d + k) * a.chirp;
  float m = 0.f;
  for (int r = lane * 2; r < a.chir_loc; r += 64) {  // chirp is even: the 16 B load stays in the row
    const float4 v = *reinterpret_cast<const float4*>(src + r);
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    if (r + 1 < a.chir_loc) m = fmaxf(m, fmaxf(fabsf(v.z), fabsf(v.w)));
  }
  return warp_max(m);
}

// Max component of the chosen slice in the reference's scaling (env_ref = temp_int / gamma_r up to
// the per-sample power of two): the PerSampleMax divisor of the grid modes (precision.cpp:155-160).
__device__ __forceinline__ double slice_max_ref(const SelectArgs& a, int n, int k, int lane) {
  const float2* src = a.temp + (static_cast<size_t>(n) * a.d + k) * a.chirp;
  double m = 0.0;
  for (int r = lane; r < a.chir_loc; r += 32) {
    const float2 v = src[r];
    m = fmax(m, static_cast<double>(fmaxf(fabsf(v.x), fabsf(v.y))) * a.inv_gamma[r]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;
}

// Displaced selection (SelectArgs::mu): D(mu_n) in shared memory, then one pass over the d stored
// outcomes of every column computes the transformed Born weights and maxima (f64 per lane, fixed-
// order warp trees); returns the chosen outcome (or kDead) exactly like the undisplaced path.
template <int MAXD>
__device__ int select_displaced(const SelectArgs& a, int n, int lane, const float2* D, float& mx_out) {
  const int d = a.d;
  double ws[MAXD];
  float ms[MAXD];
#pragma unroll
  for (int k = 0; k < MAXD; ++k) ws[k] = 0.0, ms[k] = 0.f;
  // lane handles 2 consecutive columns per step (one 16 B load per outcome; the padding columns
  // of temp and cinfo are zero, so the even-rounded tail is harmless)
  const int lim = (a.chir_loc + 1) & ~1;
  for (int r = lane * 2; r < lim; r += 64) {
    float4 v[MAXD];
#pragma unroll
    for (int q = 0; q < MAXD; ++q)
      if (q < d) v[q] = *reinterpret_cast<const float4*>(a.temp + (static_cast<size_t>(n) * d + q) * a.chirp + r);
    const float4 wl2 = *reinterpret_cast<const float4*>(a.cinfo + r);  // (cs0, wl0, cs1, wl1)
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
      if (k >= d) break;
      float o0r = 0.f, o0i = 0.f, o1r = 0.f, o1i = 0.f;
#pragma unroll
      for (int q = 0; q < MAXD; ++q) {
        if (q >= d) break;
        const float2 dk = D[k * d + q];
        o0r = fmaf(dk.x, v[q].x, fmaf(-dk.y, v[q].y, o0r));
        o0i = fmaf(dk.x, v[q].y, fmaf(dk.y, v[q].x, o0i));
        o1r = fmaf(dk.x, v[q].z, fmaf(-dk.y, v[q].w, o1r));
        o1i = fmaf(dk.x, v[q].w, fmaf(dk.y, v[q].z, o1i));
      }
      ws[k] += static_cast<double>(wl2.y) * (static_cast<double>(o0r) * o0r + static_cast<double>(o0i) * o0i) +
               static_cast<double>(wl2.w) * (static_cast<double>(o1r) * o1r + static_cast<double>(o1i) * o1i);
      ms[k] = fmaxf(ms[k], fmaxf(fmaxf(fabsf(o0r), fabsf(o0i)), fmaxf(fabsf(o1r), fabsf(o1i))));
    }
  }
  double total = 0.0;  // sampler.cpp:92-93, ascending k
#pragma unroll
  for (int k = 0; k < MAXD; ++k) {
    if (k >= d) break;
    ws[k] = warp_sum(ws[k]);
    ms[k] = warp_max(ms[k]);
    total += ws[k];
  }
  if (a.marg != nullptr) {
    double* mrow = a.marg + (static_cast<size_t>(n) * a.num_sites + a.site) * d;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
      if (k < d && lane == k) mrow[k] = total == 0.0 ? -1.0 : ws[k] / total;
  }
  if (total == 0.0) return kDead;  // sampler.cpp:94-98
  int kk;
  if (a.forced != nullptr) {
    kk = a.forced[static_cast<size_t>(n) * a.num_sites + a.site];
    if (kk == kDead) return kDead;
  } else {
    const double draw = keyed_uniform(a.seed, kMeasureStream, a.first + n, a.site);
    double cum = 0.0;
    kk = 0;
    bool near = false;
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {  // sampler.cpp:100-106
      if (k >= d) break;
      cum += ws[k] / total;
      if (draw > cum) ++kk;
      near |= k + 1 < d && fabs(draw - cum) < kBoundaryEps;
    }
    if (kk >= d) kk = d - 1;  // :107
    if (near && a.near != nullptr && lane == 0) atomicAdd(a.near, 1ull);
  }
  float mx = 0.f;
#pragma unroll
  for (int k = 0; k < MAXD; ++k)
    if (k == kk) mx = ms[k];
  mx_out = mx;
  return kk;
}

template <bool kDisp, int MAXD = 1>
__global__ void __launch_bounds__(256) select_kernel(const SelectArgs a) {
  __shared__ float2 sD[kDisp ? 8 : 1][MAXD * MAXD];
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const bool in_range = n < a.rows;
  const int sidx = !in_range ? 0 : a.perm != nullptr ? a.perm[n] : n;  // sample of this row within the pass
  const bool live_in = in_range && sidx < a.count && a.alive[n];
  // measure's live counter (RunStats), aggregated per block: one warp per sample made it one
  // same-address atomic per sample, which serialised in L2 (~60 us per 65536-row site)
  if (a.live != nullptr) {
    const int c = __syncthreads_count(live_in && lane == 0);
    if (threadIdx.x == 0 && c > 0) atomicAdd(a.live, static_cast<unsigned long long>(c));
  }
  if (!in_range) return;
  int outcome = kDead;   // recorded at this site
  bool live_out = false; // carries into the next site
  float scale = 0.f;
  double gdiv = 1.0, gmul = 1.0;  // grid modes: next env = RN((temp / gdiv) * gmul)
  const float2* D = sD[kDisp ? wib : 0];
  if (kDisp && live_in) {
    const double2 mu = a.mu[static_cast<size_t>(n) * a.num_sites + a.site];
    for (int e = lane; e < a.d * a.d; e += 32) {
      const double2 v = displacement_element(mu.x, mu.y, e / a.d, e % a.d);
      sD[wib][e] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
    }
    __syncwarp();
    float mx = 0.f;
    const int kk = select_displaced<MAXD>(a, n, lane, D, mx);
    if (kk != kDead) {
      outcome = kk;
      if (mx > 0.f) {
        int e;
        frexpf(mx, &e);
        scale = ldexpf(1.0f, kEnvExp - e);
        live_out = true;
      }
    }
  } else if (live_in) {
    // Born weights of the outcomes (sampler.cpp:83-90): for d <= 32 lane k owns outcome k and sums
    // its tile partials sequentially in f64 (fixed order); the totals and the CDF walk broadcast the
    // per-lane weights in ascending k, exactly the reference's accumulation order over k.
    const bool by_lane = a.d <= 32;
    double wk = 0.0;
    float mk = 0.f;
    if (by_lane && lane < a.d) {
      const float2* base = a.part_base + n * a.row_stride + lane * a.k_stride;
      for (int t = 0; t < a.parts; ++t) {
        const float2 v = base[t * a.part_stride];
        wk += static_cast<double>(v.x);
        mk = fmaxf(mk, v.y);
      }
    }
    auto weight = [&](int k) -> double {
      return by_lane ? __shfl_sync(0xffffffffu, wk, k) : outcome_weight(a, n, k, lane);
    };
    double total = 0.0;  // sampler.cpp:92-93, ascending k
    for (int k = 0; k < a.d; ++k) total += weight(k);
    if (a.marg != nullptr) {
      double* mrow = a.marg + (static_cast<size_t>(n) * a.num_sites + a.site) * a.d;
      if (by_lane) {
        if (lane < a.d) mrow[lane] = total == 0.0 ? -1.0 : wk / total;
      } else {
        for (int k = 0; k < a.d; ++k) {
          const double w = outcome_weight(a, n, k, lane);
          if (lane == 0) mrow[k] = total == 0.0 ? -1.0 : w / total;
        }
      }
    }
    if (total != 0.0) {  // total == 0 -> dead (sampler.cpp:94-98)
      int kk;
      if (a.forced != nullptr) {
        kk = a.forced[static_cast<size_t>(n) * a.num_sites + a.site];
      } else {
        const double draw = keyed_uniform(a.seed, kMeasureStream, a.first + sidx, a.site);
        double cum = 0.0;
        kk = 0;
        bool near = false;  // the draw lies within kBoundaryEps of an interior CDF boundary
        for (int k = 0; k < a.d; ++k) {  // sampler.cpp:100-106: strict '>', no early break
          cum += weight(k) / total;
          if (draw > cum) ++kk;
          near |= k + 1 < a.d && fabs(draw - cum) < kBoundaryEps;
        }
        if (kk >= a.d) kk = a.d - 1;  // :107
        if (near && a.near != nullptr && lane == 0) atomicAdd(a.near, 1ull);
      }
      if (kk != kDead) {
        outcome = kk;
        // per-sample max of the chosen slice (precision.cpp:155-160); 0 -> dead from here on
        float mx;
        if (a.slice_max)
          mx = slice_max(a, n, kk, lane);
        else
          mx = by_lane ? __shfl_sync(0xffffffffu, mk, kk) : outcome_max(a, n, kk, lane);
        if (mx > 0.f) {
          int e;
          frexpf(mx, &e);  // mx = f * 2^e, f in [0.5, 1): the env max lands in [2^13, 2^14)
          scale = ldexpf(1.0f, kEnvExp - e);
          live_out = true;
          if (a.grid != kGridNone) {
            // the reference divides the gathered row by its max component (PerSampleMax) before the
            // next contraction rounds it (precision.cpp:151-160, contract.cpp:66-68); F16 keeps the
            // reference's absolute values, TF32 a power of two of them (its grid is scale-invariant)
            if (a.scaling == 2) gdiv = a.grid == kGridTF32 ? slice_max_ref(a, n, kk, lane) : static_cast<double>(mx);
            if (a.grid == kGridTF32) {
              int eg;
              frexp(static_cast<double>(mx) / gdiv, &eg);
              gmul = ldexp(1.0, kEnvExp - eg);
            }
          }
        }
      }
    }
  }
  if (!live_in && a.marg != nullptr && lane == 0 && n < a.count) {
    double* mrow = a.marg + (static_cast<size_t>(n) * a.num_sites + a.site) * a.d;
    for (int k = 0; k < a.d; ++k) mrow[k] = -1.0;
  }
  if (lane == 0 && sidx < a.count) {
    a.rows_out[static_cast<size_t>(sidx) * a.num_sites + a.site] = static_cast<uint8_t>(outcome);
    a.alive[n] = live_out ? 1 : 0;
  }
  if (a.rowk != nullptr) {  // slice-recompute path: bucket the row; the slice GEMM writes its env
    if (lane == 0) {
      const int b = live_out ? outcome : a.d;
      a.rowk[n] = static_cast<uint8_t>(b);
      a.scale_out[n] = scale;
      atomicAdd(a.bcount + b, 1);
    }
    return;
  }
  if (a.trace != nullptr && outcome != kDead) {
    // reference-scale |env| of the gathered slice: |temp_int| / gamma_r * exp(-logscale)
    const float2* src = a.temp + (static_cast<size_t>(n) * a.d + outcome) * a.chirp;
    double acc = 0.0, mref = 0.0;
    for (int r = lane; r < a.chir_loc; r += 32) {
      const float2 v = src[r];
      const double ig = a.inv_gamma[r];
      acc += hypot(static_cast<double>(v.x), static_cast<double>(v.y)) * ig;
      mref = fmax(mref, fmax(fabs(static_cast<double>(v.x)), fabs(static_cast<double>(v.y))) * ig);
    }
    acc = warp_sum(acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mref = fmax(mref, __shfl_xor_sync(0xffffffffu, mref, o));
    if (lane == 0) {
      const double ls = a.logscale[n];
      atomicAdd(a.trace, acc * exp(-ls));
      // next site: E_next = temp_int * scale  ->  logscale' = logscale + ln(scale) (+ ln m for
      // PerSampleMax, whose reference env is divided by its max component m = mref * exp(-ls))
      double nl = ls + log(static_cast<double>(scale));
      if (a.scaling == 2 && mref > 0.0) nl += log(mref) - ls;
      a.logscale[n] = live_out ? nl : 0.0;
    }
  }
  if (a.kp_next > 0) {
    // next env row: E[n, r] = temp[n, k, r] * 2^-e, split hi/lo fp16 (zeros for dead / pad), per
    // component re, im (and re + im for the 3M contraction, rounded once in fp32 then split).
    // Each lane handles 4 consecutive columns: two 16 B loads, one 8 B store per plane.
    const size_t plane = static_cast<size_t>(a.env_cap) * a.kp_next;
    __half* e0 = a.env_next + static_cast<size_t>(n) * a.kp_next;
    const float2* src = a.temp + (static_cast<size_t>(n) * a.d + (live_out ? outcome : 0)) * a.chirp;
    const int live_cols = live_out ? a.chir_loc : 0;
    const int C = a.env_comp;
    if constexpr (!kDisp) {
      if (a.grid != kGridNone) {
        // single precision half on the policy's grid (round_scalar, IEEE RNE from the f64 quotient
        // exactly as the reference's double row / max); the lo planes stay zero
        for (int r = lane; r < a.kp_next; r += 32) {
          const float2 v = r < live_cols ? src[r] : make_float2(0.f, 0.f);
          e0[r] = __double2half(static_cast<double>(v.x) / gdiv * gmul);
          e0[plane + r] = __double2half(static_cast<double>(v.y) / gdiv * gmul);
          e0[2 * plane + r] = __float2half_rn(0.f);
          e0[3 * plane + r] = __float2half_rn(0.f);
        }
        return;
      }
      // 8 consecutive columns per lane: four 16 B loads, one 16 B store per plane
      for (int r = lane * 8; r < a.kp_next; r += 256) {  // kp_next is a multiple of 32
        float re[8], im[8];
        if (r + 7 < live_cols) {  // chirp is a multiple of 128: these loads stay inside the row
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 v = *reinterpret_cast<const float4*>(src + r + 2 * j);
            re[2 * j] = v.x, im[2 * j] = v.y, re[2 * j + 1] = v.z, im[2 * j + 1] = v.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float2 v = r + j < live_cols ? src[r + j] : make_float2(0.f, 0.f);
            re[j] = v.x, im[j] = v.y;
          }
        }
        __align__(16) __half hv[3][8], lv[3][8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          __half h3[3], l3[3];
          env_split(re[j] * scale, im[j] * scale, h3, l3);
#pragma unroll
          for (int c = 0; c < 3; ++c) hv[c][j] = h3[c], lv[c][j] = l3[c];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (c >= C) break;
          *reinterpret_cast<uint4*>(e0 + c * plane + r) = *reinterpret_cast<const uint4*>(hv[c]);
          *reinterpret_cast<uint4*>(e0 + (C + c) * plane + r) = *reinterpret_cast<const uint4*>(lv[c]);
        }
      }
      return;
    }
    if constexpr (kDisp) {  // (the undisplaced path returned above)
      for (int r = lane * 4; r < a.kp_next; r += 128) {  // kp_next is a multiple of 32
        float4 v01 = make_float4(0.f, 0.f, 0.f, 0.f), v23 = v01;
        if (kDisp && r < live_cols) {  // displaced: row `outcome` of D applied on the fly
          float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          for (int q = 0; q < a.d; ++q) {  // chirp is a multiple of 128: the 4 columns stay in the row
            const float2 dk = D[outcome * a.d + q];
            const float2* src_q = a.temp + (static_cast<size_t>(n) * a.d + q) * a.chirp + r;
            const float4 x01 = *reinterpret_cast<const float4*>(src_q);
            const float4 x23 = *reinterpret_cast<const float4*>(src_q + 2);
            const float xs[8] = {x01.x, x01.y, x01.z, x01.w, x23.x, x23.y, x23.z, x23.w};
  #pragma unroll
            for (int j = 0; j < 4; ++j) {
              o[2 * j] = fmaf(dk.x, xs[2 * j], fmaf(-dk.y, xs[2 * j + 1], o[2 * j]));
              o[2 * j + 1] = fmaf(dk.x, xs[2 * j + 1], fmaf(dk.y, xs[2 * j], o[2 * j + 1]));
            }
          }
  #pragma unroll
          for (int j = 0; j < 4; ++j)
            if (r + j >= live_cols) o[2 * j] = o[2 * j + 1] = 0.f;
          v01 = make_float4(o[0], o[1], o[2], o[3]);
          v23 = make_float4(o[4], o[5], o[6], o[7]);
        } else if (r + 3 < live_cols) {  // chirp is a multiple of 128: these loads stay inside the row
          v01 = *reinterpret_cast<const float4*>(src + r);
          v23 = *reinterpret_cast<const float4*>(src + r + 2);
        } else if (r < live_cols) {
          const float2 z = make_float2(0.f, 0.f);
          const float2 c0 = src[r];
          const float2 c1 = r + 1 < live_cols ? src[r + 1] : z;
          const float2 c2 = r + 2 < live_cols ? src[r + 2] : z;
          v01 = make_float4(c0.x, c0.y, c1.x, c1.y);
          v23 = make_float4(c2.x, c2.y, 0.f, 0.f);
        }
        const float cre[4] = {v01.x * scale, v01.z * scale, v23.x * scale, v23.z * scale};
        const float cim[4] = {v01.y * scale, v01.w * scale, v23.y * scale, v23.w * scale};
        __align__(8) __half hv[3][4], lv[3][4];
  #pragma unroll
        for (int j = 0; j < 4; ++j) {
          __half h3[3], l3[3];
          env_split(cre[j], cim[j], h3, l3);
  #pragma unroll
          for (int c = 0; c < 3; ++c) hv[c][j] = h3[c], lv[c][j] = l3[c];
        }
  #pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (c >= C) break;
          *reinterpret_cast<uint2*>(e0 + c * plane + r) = *reinterpret_cast<const uint2*>(hv[c]);
          *reinterpret_cast<uint2*>(e0 + (C + c) * plane + r) = *reinterpret_cast<const uint2*>(lv[c]);
        }
      }
    }
  }
}

// pstat [rows][nt] -> out [rows][d]: per outcome k the sum of its tiles' weights (fixed-order f64
// reduction, rounded to fp32 for the exchange) and the max; one warp per sample.
__global__ void reduce_tiles_kernel(const float2* pstat, int nt, int tpk, int d, int rows,
                                    float2* out) {
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (n >= rows) return;
  for (int k = 0; k < d; ++k) {
    double s = 0.0;
    float m = 0.f;
    for (int t = lane; t < tpk; t += 32) {
      const float2 v = pstat[static_cast<size_t>(n) * nt + k * tpk + t];
      s += static_cast<double>(v.x);
      m = fmaxf(m, v.y);
    }
    s = warp_sum(s);
    m = warp_max(m);
    if (lane == 0) out[static_cast<size_t>(n) * d + k] = make_float2(static_cast<float>(s), m);
  }
}

void launch_reduce_tiles(const float2* pstat, int nt, int tiles_per_k, int d, int rows,
                         float2* out, cudaStream_t s) {
  const int threads = 256;
  reduce_tiles_kernel<<<(rows * 32 + threads - 1) / threads, threads, 0, s>>>(pstat, nt, tiles_per_k,
                                                                             d, rows, out);
}

// Tensor-parallel environment exchange: the 3M s planes (hi 2, lo 5) of every shard re-formed from
// the received re / im planes (hi 0, 1; lo 3, 4) with env_split's arithmetic, 8 columns per thread.
__global__ void env_reform_s_kernel(__half* env, int env_cap, int kshard, int shards, int rows) {
  const size_t plane = static_cast<size_t>(env_cap) * kshard;
  const int per_row = kshard / 8;
  const size_t total = static_cast<size_t>(shards) * rows * per_row;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(e / (static_cast<size_t>(rows) * per_row));
    const size_t rem = e - static_cast<size_t>(q) * rows * per_row;
    const int n = static_cast<int>(rem / per_row), c8 = static_cast<int>(rem - static_cast<size_t>(n) * per_row);
    __half* base = env + static_cast<size_t>(q) * 6 * plane + static_cast<size_t>(n) * kshard + 8 * c8;
    const uint4 hr = *reinterpret_cast<const uint4*>(base);
    const uint4 hi = *reinterpret_cast<const uint4*>(base + plane);
    const uint4 lr = *reinterpret_cast<const uint4*>(base + 3 * plane);
    const uint4 li = *reinterpret_cast<const uint4*>(base + 4 * plane);
    const __half* phr = reinterpret_cast<const __half*>(&hr);
    const __half* phi = reinterpret_cast<const __half*>(&hi);
    const __half* plr = reinterpret_cast<const __half*>(&lr);
    const __half* pli = reinterpret_cast<const __half*>(&li);
    __align__(16) __half hs[8], ls[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float a = __half2float(phr[j]) + __half2float(plr[j]);
      const float b = __half2float(phi[j]) + __half2float(pli[j]);
      const float sv = a + b;
      hs[j] = __float2half_rn(sv);
      ls[j] = __float2half_rn(sv - __half2float(hs[j]));
    }
    *reinterpret_cast<uint4*>(base + 2 * plane) = *reinterpret_cast<const uint4*>(hs);
    *reinterpret_cast<uint4*>(base + 5 * plane) = *reinterpret_cast<const uint4*>(ls);
  }
}

void launch_env_reform_s(__half* env, int env_cap, int kshard, int shards, int rows, cudaStream_t s) {
  const size_t total = static_cast<size_t>(shards) * rows * (kshard / 8);
  if (total == 0) return;
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 4 * 148));
  env_reform_s_kernel<<<blocks, 256, 0, s>>>(env, env_cap, kshard, shards, rows);
}

// K2 fast path for short rows (chi <= 512): R rows per warp, each row's chosen slice held in
// registers.  select_kernel's one-warp-per-row chain (alive -> partials -> draw -> slice max -> env
// stores, the max pass and the split pass each a round trip per 64 columns) is latency-bound when a
// row is only 2-4 KB: ~14 waves of 32 resident warps per SM over a 65536-row pass.  Here a warp runs
// the weights / CDF / draw of R rows at once (32/R lanes per row, lane k of a group owns outcome k),
// then issues all loads of the R chosen slices together (CH chunks of 256 columns per row, 8 columns
// per lane: 4 * R * CH 16 B loads in flight per lane), takes the max and splits from registers.
// The arithmetic is select_kernel's operation for operation (fixed-order f64 partial sums per
// outcome, ascending-k totals and CDF, max of the chosen slice, env_split), so outcomes and
// environments are bit-identical to it (tests/test_gpu_parity.py::test_select_fast_path_identical).
// Covers the plain sampling pass: no displacement, no GRID rounding, no decay trace, no slice-
// recompute bucketing, d <= 32 / R.
template <int R, int CH>
__global__ void __launch_bounds__(256) select_rows_kernel(const SelectArgs a) {
  constexpr unsigned kFull = 0xffffffffu;
  constexpr int kG = 32 / R;  // lanes per row in the draw phase
  const int lane = threadIdx.x & 31;
  const int grp = lane / kG, k = lane % kG, g0 = grp * kG;
  const unsigned gmask = (kG == 32 ? kFull : ((1u << kG) - 1u)) << g0;
  const int wrow0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * R;
  ptx::grid_dep_wait();  // (programmatic dependent launch) the contraction's temp / partials are complete
  ptx::grid_dep_launch();
  // ---- phase 1: lane group grp = row wrow0 + grp ----
  const int n = wrow0 + grp;
  const bool in_range = n < a.rows;
  const int sidx = !in_range ? 0 : a.perm != nullptr ? a.perm[n] : n;
  const bool live_in = in_range && sidx < a.count && a.alive[n];
  if (a.live != nullptr) {
    const int c = __syncthreads_count(live_in && k == 0);
    if (threadIdx.x == 0 && c > 0) atomicAdd(a.live, static_cast<unsigned long long>(c));
  }
  if (wrow0 >= a.rows) return;  // whole warp out of range (rows is a multiple of 128)
  double wk = 0.0;
  float mk = 0.f;
  if (live_in && k < a.d) {  // sampler.cpp:83-90: outcome k's tile partials in order, f64
    const float2* base = a.part_base + n * a.row_stride + k * a.k_stride;
    for (int t = 0; t < a.parts; ++t) {
      const float2 v = base[t * a.part_stride];
      wk += static_cast<double>(v.x);
      mk = fmaxf(mk, v.y);
    }
  }
  double total = 0.0;  // sampler.cpp:92-93, ascending k
  for (int q = 0; q < a.d; ++q) total += __shfl_sync(kFull, wk, g0 + q);
  if (a.marg != nullptr && k < a.d) {
    if (live_in)
      a.marg[(static_cast<size_t>(n) * a.num_sites + a.site) * a.d + k] = total == 0.0 ? -1.0 : wk / total;
    else if (in_range && n < a.count)
      a.marg[(static_cast<size_t>(n) * a.num_sites + a.site) * a.d + k] = -1.0;
  }
  int kk = kDead;
  if (live_in && total != 0.0) {  // total == 0 -> dead (sampler.cpp:94-98); group-uniform branch
    if (a.forced != nullptr) {
      kk = a.forced[static_cast<size_t>(n) * a.num_sites + a.site];
    } else {
      const double draw = keyed_uniform(a.seed, kMeasureStream, a.first + sidx, a.site);
      double cum = 0.0;
      kk = 0;
      bool near = false;
      for (int q = 0; q < a.d; ++q) {  // sampler.cpp:100-106: strict '>', no early break
        cum += __shfl_sync(gmask, wk, g0 + q) / total;
        if (draw > cum) ++kk;
        near |= q + 1 < a.d && fabs(draw - cum) < kBoundaryEps;
      }
      if (kk >= a.d) kk = a.d - 1;  // :107
      if (near && a.near != nullptr && k == 0) atomicAdd(a.near, 1ull);
    }
  }
  // the partials' max of the chosen outcome (used when slice_max == 0: TP / long-K epilogues)
  const float mk_sel = __shfl_sync(kFull, mk, g0 + ((kk != kDead && kk < kG) ? kk : 0));
  // ---- phase 2: the warp loads the R chosen slices (all loads in flight), max, split, store ----
  int out_r[R];
  float mx_r[R];
  float2 v[R][CH][8];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    out_r[r] = __shfl_sync(kFull, kk, r * kG);
    mx_r[r] = __shfl_sync(kFull, mk_sel, r * kG);
    const int live_cols = out_r[r] != kDead ? a.chir_loc : 0;
    const float2* src = a.temp + (static_cast<size_t>(wrow0 + r) * a.d + (out_r[r] != kDead ? out_r[r] : 0)) * a.chirp;
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) {
      const int c = ch * 256 + lane * 8;
      if (c + 7 < live_cols) {  // chirp is a multiple of 128: these loads stay inside the row
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 x = *reinterpret_cast<const float4*>(src + c + 2 * j);
          v[r][ch][2 * j] = make_float2(x.x, x.y);
          v[r][ch][2 * j + 1] = make_float2(x.z, x.w);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[r][ch][j] = c + j < live_cols ? src[c + j] : make_float2(0.f, 0.f);
      }
    }
  }
  if (a.slice_max) {  // precision.cpp:155-160: max component of the chosen slice (zeros beyond it)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float m = 0.f;
#pragma unroll
      for (int ch = 0; ch < CH; ++ch)
#pragma unroll
        for (int j = 0; j < 8; ++j) m = fmaxf(m, fmaxf(fabsf(v[r][ch][j].x), fabsf(v[r][ch][j].y)));
      mx_r[r] = warp_max(m);
    }
  }
  float scale_r[R];
  bool live_r[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    scale_r[r] = 0.f;
    live_r[r] = false;
    if (out_r[r] != kDead && mx_r[r] > 0.f) {
      int e;
      frexpf(mx_r[r], &e);  // the env max lands in [2^13, 2^14)
      scale_r[r] = ldexpf(1.0f, kEnvExp - e);
      live_r[r] = true;
    }
  }
  if (lane < R) {
    int o = kDead;
    bool lv = false;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r == lane) o = out_r[r], lv = live_r[r];
    const int nr = wrow0 + lane;
    const int sr = a.perm != nullptr ? a.perm[nr] : nr;
    if (sr < a.count) {
      a.rows_out[static_cast<size_t>(sr) * a.num_sites + a.site] = static_cast<uint8_t>(o);
      a.alive[nr] = lv ? 1 : 0;
    }
  }
  if (a.kp_next <= 0) return;
  // next env rows (select_kernel's split; zeros for dead rows and beyond the slice): one 16 B store
  // per plane and 8 columns
  const size_t plane = static_cast<size_t>(a.env_cap) * a.kp_next;
  const int C = a.env_comp;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const float sc = live_r[r] ? scale_r[r] : 0.f;
    __half* e0 = a.env_next + static_cast<size_t>(wrow0 + r) * a.kp_next;
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) {
      const int c = ch * 256 + lane * 8;
      if (c >= a.kp_next) break;
      __align__(16) __half hv[3][8], lv[3][8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        __half h3[3], l3[3];
        // dead rows: select_kernel splits zeros (it reads nothing); the loads above gave zeros too
        env_split(live_r[r] ? v[r][ch][j].x * sc : 0.f, live_r[r] ? v[r][ch][j].y * sc : 0.f, h3, l3);
#pragma unroll
        for (int q = 0; q < 3; ++q) hv[q][j] = h3[q], lv[q][j] = l3[q];
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (q >= C) break;
        *reinterpret_cast<uint4*>(e0 + q * plane + c) = *reinterpret_cast<const uint4*>(hv[q]);
        *reinterpret_cast<uint4*>(e0 + (C + q) * plane + c) = *reinterpret_cast<const uint4*>(lv[q]);
      }
    }
  }
}

template <int R, int CH>
static void launch_select_rows(const SelectArgs& a, cudaStream_t s) {
  const int threads = 256;
  const int warps = a.rows / R;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((warps * 32 + threads - 1) / threads);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.pdl ? 1 : 0;
  check_launch(cudaLaunchKernelEx(&cfg, select_rows_kernel<R, CH>, a), "select_rows_kernel");
}

void launch_select(const SelectArgs& a, cudaStream_t s) {
  const int threads = 256;
  const int blocks = (a.rows * 32 + threads - 1) / threads;
  static const bool legacy = [] {
    const char* v = std::getenv("MPSG_SELECT_LEGACY");
    return v != nullptr && std::atoi(v) != 0;
  }();
  const bool plain = !legacy && a.mu == nullptr && a.grid == kGridNone && a.trace == nullptr && a.rowk == nullptr;
  if (plain && a.d <= 8 && a.chir_loc <= 256 && a.kp_next <= 256 && a.rows % 4 == 0) {
    launch_select_rows<4, 1>(a, s);
    return;
  }
  if (plain && a.d <= 16 && a.chir_loc <= 512 && a.kp_next <= 512 && a.rows % 2 == 0) {
    launch_select_rows<2, 2>(a, s);
    return;
  }
  if (a.mu != nullptr) {
    ensure_fact_table();
    if (a.d <= 8)
      select_kernel<true, 8><<<blocks, threads, 0, s>>>(a);
    else
      select_kernel<true, kMaxDisplacedDim><<<blocks, threads, 0, s>>>(a);
  } else {
    select_kernel<false><<<blocks, threads, 0, s>>>(a);
  }
}

// ============================================================================================
// site-0 environment (sampler.cpp:136-138: env = ones(count, 1), all alive)
// ============================================================================================
__global__ void init_env_kernel(__half* env, int env_comp, int env_cap, int kshard0, int shards,
                                int rows, int count, uint8_t* alive, double* logscale, int* perm) {
  const int planes = 2 * env_comp;
  const size_t plane = static_cast<size_t>(env_cap) * kshard0;
  const size_t total = static_cast<size_t>(shards) * planes * plane;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t p = i / plane, rem = i - p * plane;  // p = shard * planes + plane
    const size_t n = rem / kshard0, c = rem - n * kshard0;
    // E = 1 + 0i: hi.re = 1 and, for the 3M layout, hi.(re + im) = 1
    const bool one = (p == 0 || (env_comp == 3 && p == 2)) && c == 0 && n < static_cast<size_t>(count);
    env[i] = __float2half_rn(one ? 1.0f : 0.0f);
  }
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < rows; n += gridDim.x * blockDim.x) {
    alive[n] = n < count ? 1 : 0;
    if (logscale) logscale[n] = 0.0;
    if (perm) perm[n] = n;
  }
}

void launch_init_env(__half* env, int env_comp, int env_cap, int kshard0, int shards, int rows,
                     int count, uint8_t* alive, cudaStream_t s, double* logscale, int* perm) {
  init_env_kernel<<<296, 256, 0, s>>>(env, env_comp, env_cap, kshard0, shards, rows, count, alive,
                                      logscale, perm);
}

// ============================================================================================
// Slice-recompute path: bucket scatter of the environment rows by drawn outcome (one warp per
// row; the order inside a bucket is the atomic arrival order -- every row's arithmetic is
// independent of its position, so the sampled values are not) and zeroing of the dead rows
// ============================================================================================
__device__ __forceinline__ int bucket_offset(const int* bcount, int k) {
  int o = 0;
  for (int q = 0; q < k; ++q) o += bcount[q];
  return o;
}

__global__ void __launch_bounds__(256) permute_rows_kernel(const PermuteArgs a) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= a.rows) return;
  const int k = a.rowk[j];
  int dst = 0;
  if (lane == 0) dst = bucket_offset(a.bcount, k) + atomicAdd(a.bfill + k, 1);
  dst = __shfl_sync(0xffffffffu, dst, 0);
  const size_t plane = static_cast<size_t>(a.env_cap) * a.kp;
  const int v8 = a.kp / 8;  // kp is a multiple of 64
  for (int p = 0; p < a.planes; ++p) {
    const uint4* src = reinterpret_cast<const uint4*>(a.env + p * plane + static_cast<size_t>(j) * a.kp);
    uint4* out = reinterpret_cast<uint4*>(a.env2 + p * plane + static_cast<size_t>(dst) * a.kp);
    for (int c = lane; c < v8; c += 32) out[c] = src[c];
  }
  if (lane == 0) {
    a.perm2[dst] = a.perm[j];
    if (a.rowk2 != nullptr) a.rowk2[dst] = static_cast<uint8_t>(k);
    a.scale2[dst] = a.scale[j];
    a.alive2[dst] = k < a.d ? 1 : 0;
  }
}

void launch_permute_rows(const PermuteArgs& a, cudaStream_t s) {
  const int blocks = (a.rows * 32 + 255) / 256;
  permute_rows_kernel<<<blocks, 256, 0, s>>>(a);
}

__global__ void zero_dead_kernel(__half* env, int planes, int env_cap, int kp, int rows, const int* bcount,
                                 int d) {
  __shared__ int r0;
  if (threadIdx.x == 0) r0 = bucket_offset(bcount, d);
  __syncthreads();
  const size_t plane = static_cast<size_t>(env_cap) * kp;
  const size_t per_plane = static_cast<size_t>(rows - r0) * kp / 8;  // uint4 per plane
  const size_t total = per_plane * planes;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t p = i / per_plane, rem = i - p * per_plane;
    reinterpret_cast<uint4*>(env + p * plane + static_cast<size_t>(r0) * kp)[rem] = make_uint4(0, 0, 0, 0);
  }
}

void launch_zero_dead(__half* env, int planes, int env_cap, int kp, int rows, const int* bcount, int d,
                      cudaStream_t s) {
  zero_dead_kernel<<<148, 256, 0, s>>>(env, planes, env_cap, kp, rows, bcount, d);
}

__global__ void draws_kernel(uint64_t seed, uint64_t first, uint64_t count, uint64_t site,
                             double* out) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < count;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[j] = keyed_uniform(seed, kMeasureStream, first + j, site);
}

void launch_draws(uint64_t seed, uint64_t first, uint64_t count, uint64_t site, double* out,
                  cudaStream_t s) {
  draws_kernel<<<148, 256, 0, s>>>(seed, first, count, site, out);
}

// ============================================================================================
// Compression: Gamma (chiL, chiR, d) -> fp16 planes [2][Np][Kp] with power-of-two scales
//   Ghat[l, r, k] = Gamma[l, r, k] * gr[r] / gl[l] / cs[r, k],  |Ghat| <= 1
// The source is either a complex array (f64 / f32, the caller's Gamma) or the synthetic-chain
// generator below (regenerated on the device every pass for chains beyond HBM and host memory).
// ============================================================================================
template <typename T>
struct ArraySrc {  // complex T interleaved, (chiL, chiR * d) row-major
  // fp32 / fp16 sources: every scaled value is an exact float (see quantize_pair_f32)
  static constexpr bool kExactF32 = !std::is_same<T, double>::value;
  const T* p;
  size_t stride;
  __device__ __forceinline__ static double wide(double x) { return x; }
  __device__ __forceinline__ static double wide(float x) { return static_cast<double>(x); }
  __device__ __forceinline__ static double wide(__half x) { return static_cast<double>(__half2float(x)); }
  struct Col {};  // nothing per column
  __device__ __forceinline__ Col col(size_t) const { return {}; }
  __device__ __forceinline__ void load(int l, size_t j, const Col&, double& re, double& im) const {
    const T* q = p + 2 * (static_cast<size_t>(l) * stride + j);
    re = wide(q[0]);
    im = wide(q[1]);
  }
};

// Synthetic random right-canonical chain of the random_mps form (mps.cpp:148-175):
//   Gamma_i[l, j] = B[l, j] * phase_i[j] * (lambda_{i-1}[l] * (1 / lambda_i[r])),  j = r * d + k
// with explicitly rounded fp32 operations, so every kernel that evaluates it (the compression of a
// regenerated site, mpsg_synthetic_site) produces the same bits.
// (ph = phase_i[j], il = 1 / lambda_i[r]: per column, hoisted out of the compression kernels' row loops)
// (b = B[l, j] and lp = lambda_{i-1}[l] already loaded: the compression kernels batch these loads)
__device__ __forceinline__ float2 synth_from_base(float2 b, float2 ph, float lp, float il) {
  const float tr = __fsub_rn(__fmul_rn(b.x, ph.x), __fmul_rn(b.y, ph.y));
  const float ti = __fadd_rn(__fmul_rn(b.x, ph.y), __fmul_rn(b.y, ph.x));
  const float sc = __fmul_rn(lp, il);
  return make_float2(__fmul_rn(tr, sc), __fmul_rn(ti, sc));
}
__device__ __forceinline__ float2 synth_value_c(const SynthSite& g, int l, size_t j, float2 ph, float il) {
  return synth_from_base(g.base[static_cast<size_t>(l) * g.ld + j], ph, g.lam_prev[l], il);
}
__device__ __forceinline__ float2 synth_value(const SynthSite& g, int l, size_t j) {
  return synth_value_c(g, l, j, g.phase[j], g.inv_lam[j / g.d]);
}
struct SynthSrc {
  static constexpr bool kExactF32 = true;  // fp32 generator values
  SynthSite g;
  struct Col {
    float2 ph;
    float il;
  };
  __device__ __forceinline__ Col col(size_t j) const { return {g.phase[j], g.inv_lam[j / g.d]}; }
  __device__ __forceinline__ void load(int l, size_t j, const Col& c, double& re, double& im) const {
    const float2 v = synth_value_c(g, l, j, c.ph, c.il);
    re = static_cast<double>(v.x);
    im = static_cast<double>(v.y);
  }
};

// phase_i[j] = exp(2 pi i u), u = keyed uniform of (seed, kPhaseStream, site, j) (rng.hpp:22-37)
__global__ void synth_phase_kernel(uint64_t seed, uint64_t site, int cols, float2* phase) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x) {
    const double u = keyed_uniform(seed, kPhaseStream, site, static_cast<uint64_t>(j));
    double sn, cs;
    sincospi(2.0 * u, &sn, &cs);
    phase[j] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
  }
}

__global__ void synth_values_kernel(const SynthSite g, int rows, float2* out) {
  const size_t n = static_cast<size_t>(rows) * g.cols;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int l = static_cast<int>(e / g.cols);
    out[e] = synth_value(g, l, e - static_cast<size_t>(l) * g.cols);
  }
}

void launch_synth_phase(uint64_t seed, uint64_t site, int cols, float2* phase, cudaStream_t s) {
  synth_phase_kernel<<<std::max(1, std::min((cols + 255) / 256, 592)), 256, 0, s>>>(seed, site, cols, phase);
}
void launch_synth_values(const SynthSite& g, int rows, float2* out, cudaStream_t s) {
  synth_values_kernel<<<1184, 256, 0, s>>>(g, rows, out);
}

// 1 / x for a power of two x (the bond and column scales): exact, and a few integer ops instead of an
// f64 division (the divisions made the compression kernels FP64-bound: pack 1.5 ms per chi = 8192
// site, the regenerated supply's main overhead).
// Fast path on the exponent bits (2^-floor(log2 x) for a positive normal x whose reciprocal power is
// normal -- every scale the engine forms); ilogb / ldexp otherwise.  Bit-identical to the original
// (the library calls made the compression kernels issue-bound: ~200 instructions per element).
__device__ __forceinline__ double inv_pow2(double x) {
  const long long b = __double_as_longlong(x);
  const int e = static_cast<int>((b >> 52) & 0x7ff);
  if (b > 0 && e >= 1 && e <= 2045) return __longlong_as_double(static_cast<long long>(2046 - e) << 52);
  return ldexp(1.0, -ilogb(x));
}

// Per local column jl = r_loc * d + k: max over l of max(|re|, |im|) * gr[r] / gl[l] (f64), as an
// order-independent atomic max of the nonnegative doubles' bit patterns.  A 2-D grid (64-row chunks
// x 128 columns) keeps enough loads in flight to stream the source at HBM rate.
template <typename Src>
__global__ void colmax_kernel(const Src src, int chil, int d, int b0, int width, const double* gl,
                              const double* gr, unsigned long long* colmax, int* err) {
  const int jl = blockIdx.x * blockDim.x + threadIdx.x;
  if (jl >= width * d) return;
  const int rl = jl / d, k = jl - rl * d;
  const int r = b0 + rl;
  const size_t j = static_cast<size_t>(r) * d + k;
  const int l0 = blockIdx.y * 64, l1 = min(chil, l0 + 64);
  double mx = 0.0;
  bool finite = true;
  // per-column operands loaded once per thread (the row loop is load-instruction bound otherwise)
  const typename Src::Col cj = src.col(j);
  const double grr = gr[r];
  if constexpr (std::is_same<Src, SynthSrc>::value) {
    // max(|re f|, |im f|) = max(|re|, |im|) f: f > 0 and both f64 products are exact; rows in groups
    // of 8 with their loads issued together
    for (int lb = l0; lb < l1; lb += 8) {
      float2 bv[8];
      float lp[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int l = lb + i;
        bv[i] = l < l1 ? src.g.base[static_cast<size_t>(l) * src.g.ld + j] : make_float2(0.f, 0.f);
        lp[i] = l < l1 ? src.g.lam_prev[l] : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int l = lb + i;
        if (l >= l1) break;
        const float2 v = synth_from_base(bv[i], cj.ph, lp[i], cj.il);
        if (!isfinite(v.x) || !isfinite(v.y)) finite = false;
        mx = fmax(mx, static_cast<double>(fmaxf(fabsf(v.x), fabsf(v.y))) * (grr * inv_pow2(gl[l])));
      }
    }
  }
  for (int l = l0; l < l1 && !std::is_same<Src, SynthSrc>::value; ++l) {
    double re, im;
    src.load(l, j, cj, re, im);
    if (!isfinite(re) || !isfinite(im)) finite = false;
    const double f = grr * inv_pow2(gl[l]);
    mx = fmax(mx, fmax(fabs(re * f), fabs(im * f)));
  }
  if (!finite) atomicExch(err, 3);  // NumericError: non-finite Gamma (contract.cpp:117-119)
  if (mx > 0.0) atomicMax(colmax + jl, static_cast<unsigned long long>(__double_as_longlong(mx)));
}

// Column scales from the maxima: cs = 2^e with mx = f 2^e, f in [0.5, 1); clears colmax for reuse.
// Grid modes: F16 keeps cs = 1 (the policy's absolute grid); TF32 puts the column max in
// [2^14, 2^15), so fp16 normals cover 2^-28 of it on the 11-bit grid.
__global__ void colfinish_kernel(int d, int b0, int width, int chirp, const double* wl,
                                 unsigned long long* colmax, float2* cinfo, double* cs_out, int* err,
                                 int grid) {
  const int jl = blockIdx.x * blockDim.x + threadIdx.x;
  if (jl >= width * d) return;
  const int rl = jl / d, k = jl - rl * d;
  const double mx = __longlong_as_double(static_cast<long long>(colmax[jl]));
  colmax[jl] = 0ull;
  double cs = 1.0;
  if (mx > 0.0 && grid != kGridF16) {
    int e;
    frexp(mx, &e);
    if (e > 120) {
      atomicExch(err, 3);  // outside the compressed format's range
      e = 120;
    }
    if (e < -120) e = -120;
    cs = ldexp(1.0, grid == kGridTF32 ? e - 15 : e);
  }
  cs_out[jl] = cs;
  cinfo[k * chirp + rl] = make_float2(static_cast<float>(cs), static_cast<float>(wl[b0 + rl]));
}

// Rounds (a, b) onto the fp16 grid of the binade of max(|a|, |b|, |a + b|), so that a, b and
// a + b are all exactly representable in fp16 (the 3M contraction stores Gs = Gr + Gi and must
// sample exactly the decoded Gamma).  |a|, |b| < 1 after column scaling.
__device__ __forceinline__ void quantize_pair(double a, double b, __half& ha, __half& hb, __half& hs) {
  const double m = fmax(fmax(fabs(a), fabs(b)), fabs(a + b));
  if (m == 0.0) {
    ha = hb = hs = __float2half_rn(0.f);
    return;
  }
  int e;
  frexp(m, &e);  // m in [2^(e-1), 2^e): fp16 spacing there is 2^(e-11)
  const double u = ldexp(1.0, max(e - 11, -24));
  const double iu = ldexp(1.0, -max(e - 11, -24));
  const double qa = rint(a * iu) * u, qb = rint(b * iu) * u;  // RNE; |qa + qb| <= 2^e
  ha = __double2half(qa);
  hb = __double2half(qb);
  hs = __double2half(qa + qb);
}

// quantize_pair for fp32-exact inputs, in fp32 / integer arithmetic with the same result bit for bit:
// the binade of max(|a|, |b|, |a + b|) is taken from the round-toward-zero fp32 sum (RZ never crosses
// a power of two upward, and a power of two is representable, so the exponent equals the exact sum's),
// a * 2^-k, rint and the re-scaling are exact, and qa + qb (a multiple of u below 2^(e+1)) is exact.
// The f64 original is FP64-bound (pack took 1.3 ms per chi = 8192 regenerated site).
__device__ __forceinline__ void quantize_pair_f32(float a, float b, __half& ha, __half& hb, __half& hs) {
  const float m = fmaxf(fmaxf(fabsf(a), fabsf(b)), fabsf(__fadd_rz(a, b)));
  if (m == 0.f) {
    ha = hb = hs = __float2half_rn(0.f);
    return;
  }
  // frexpf's exponent from the bits (m = f 2^e, f in [0.5, 1)); a subnormal m has e <= -126, so
  // ue = -24 for it either way; u = 2^ue and 1/u are built from their exponent fields
  const int eb = (__float_as_int(m) >> 23) & 0xff;
  const int ue = eb == 0 ? -24 : max(eb - 126 - 11, -24);
  const float u = __int_as_float((ue + 127) << 23), iu = __int_as_float((127 - ue) << 23);
  const float qa = rintf(a * iu) * u, qb = rintf(b * iu) * u;
  ha = __float2half_rn(qa);
  hb = __float2half_rn(qb);
  hs = __float2half_rn(qa + qb);
}

template <typename Src>
__global__ void pack_kernel(const Src src, int chil, int d, int b0, int width, int kp,
                            int chirp, const int* lpos, const double* gl, const double* gr,
                            const double* cs, int gplanes, __half* g_out, int np, int grid, int* err) {
  // planes: [Gr, Gi (, Gs)] and, for gplanes = 6 (MPSG_MODE_PRECISE), [Gr_lo, Gi_lo, Gs_lo] -- the
  // residual of the hi grid, itself rounded by quantize_pair, so every plane (and Gs = Gr + Gi per
  // precision half) is an exact fp16 number.  Tile: 64 rows l x 32 columns j; read along j
  // (coalesced source rows), written along l as half2 (the K-major planes, 128 B per warp store).
  __shared__ __half tp[6][64][33];
  const int wcols = width * d;
  const int j0 = blockIdx.x * 32, l0 = blockIdx.y * 64;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  // this thread's column: its per-column operands are loaded once, outside the row loop
  const int jc = j0 + tx;
  const bool col_ok = jc < wcols;
  const int rc = col_ok ? jc / d : 0, kc = col_ok ? jc - rc * d : 0;
  const size_t jsrc = static_cast<size_t>(b0 + rc) * d + kc;
  typename Src::Col cj{};
  double grr = 0.0, ics = 0.0;
  if (col_ok) {
    cj = src.col(jsrc);
    grr = gr[b0 + rc];
    ics = inv_pow2(cs[jc]);
  }
  bool done = false;
  if constexpr (std::is_same<Src, SynthSrc>::value) {
    if (grid == kGridNone) {
      // generator source: the thread's 8 rows' operands are loaded up front (8 base loads in flight per
      // thread -- one at a time left the kernel waiting on DRAM latency), then each value is scaled by
      // its power of two in fp32 when that is a normal float: v * f in fp32 is one rounding of the
      // same exact product as float(double(v) * f), i.e. the generic path's bits without f64 work
      float2 bv[8];
      float lp[8];
      double ig[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int l = l0 + ty + 8 * i;
        const bool ok = l < chil && col_ok;
        bv[i] = ok ? src.g.base[static_cast<size_t>(l) * src.g.ld + jsrc] : make_float2(0.f, 0.f);
        lp[i] = ok ? src.g.lam_prev[l] : 0.f;
        ig[i] = ok ? inv_pow2(gl[l]) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int yy = ty + 8 * i, l = l0 + yy;
        __half h[6];
#pragma unroll
        for (int p = 0; p < 6; ++p) h[p] = __float2half_rn(0.f);
        if (l < chil && col_ok) {
          const double f = grr * ig[i] * ics;
          const float2 v = synth_from_base(bv[i], cj.ph, lp[i], cj.il);
          float a, b;
          if (f >= 0x1p-126 && f <= 0x1p127) {
            const float ff = static_cast<float>(f);
            a = __fmul_rn(v.x, ff);
            b = __fmul_rn(v.y, ff);
          } else {
            a = static_cast<float>(static_cast<double>(v.x) * f);
            b = static_cast<float>(static_cast<double>(v.y) * f);
          }
          quantize_pair_f32(a, b, h[0], h[1], h[2]);
          if (gplanes == 6)
            quantize_pair_f32(a - __half2float(h[0]), b - __half2float(h[1]), h[3], h[4], h[5]);
        }
#pragma unroll
        for (int p = 0; p < 6; ++p)
          if (p < gplanes) tp[p][yy][tx] = h[p];
      }
      done = true;
    }
  }
  for (int yy = ty; yy < 64 && !done; yy += 8) {
    const int l = l0 + yy;
    __half h[6];
#pragma unroll
    for (int p = 0; p < 6; ++p) h[p] = __float2half_rn(0.f);
    if (l < chil && col_ok) {
      const double f = grr * inv_pow2(gl[l]) * ics;
      double re, im;
      src.load(l, jsrc, cj, re, im);
      if (grid != kGridNone) {  // round_scalar per component (precision.cpp:23-50): IEEE RNE
        h[0] = __double2half(re * f);
        h[1] = __double2half(im * f);
        if (__hisinf(h[0]) || __hisinf(h[1])) atomicExch(err, 3);  // beyond the F16 grid
      } else if constexpr (Src::kExactF32) {
        const float a = static_cast<float>(re * f), b = static_cast<float>(im * f);  // exact
        quantize_pair_f32(a, b, h[0], h[1], h[2]);
        if (gplanes == 6)  // residuals of the hi grid: exact in fp32 (below half a grid step)
          quantize_pair_f32(a - __half2float(h[0]), b - __half2float(h[1]), h[3], h[4], h[5]);
      } else {
        quantize_pair(re * f, im * f, h[0], h[1], h[2]);
        if (gplanes == 6)
          quantize_pair(re * f - static_cast<double>(__half2float(h[0])),
                        im * f - static_cast<double>(__half2float(h[1])), h[3], h[4], h[5]);
      }
    }
#pragma unroll
    for (int p = 0; p < 6; ++p)
      if (p < gplanes) tp[p][yy][tx] = h[p];
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {
    const int jl = j0 + yy, l = l0 + 2 * tx;
    if (jl >= wcols || l >= chil) continue;
    const int rl = jl / d, k = jl - rl * d;
    const size_t row = static_cast<size_t>(k) * chirp + rl;
    const int c0 = lpos[l];
    const bool pair = l + 1 < chil && lpos[l + 1] == c0 + 1 && (c0 & 1) == 0;
    for (int p = 0; p < gplanes; ++p) {
      __half* dst = g_out + (static_cast<size_t>(p) * np + row) * kp;
      if (pair) {
        *reinterpret_cast<__half2*>(dst + c0) = __halves2half2(tp[p][2 * tx][yy], tp[p][2 * tx + 1][yy]);
      } else {
        dst[c0] = tp[p][2 * tx][yy];
        if (l + 1 < chil) dst[lpos[l + 1]] = tp[p][2 * tx + 1][yy];
      }
    }
  }
}

__global__ void __launch_bounds__(256) sum_plane_kernel(__half* g, size_t n8, size_t pe) {
  const uint4* a = reinterpret_cast<const uint4*>(g);
  const uint4* b = reinterpret_cast<const uint4*>(g + pe);
  uint4* c = reinterpret_cast<uint4*>(g + 2 * pe);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint4 x = a[i], y = b[i];
    uint4 z;
    const __half2* xh = reinterpret_cast<const __half2*>(&x);
    const __half2* yh = reinterpret_cast<const __half2*>(&y);
    __half2* zh = reinterpret_cast<__half2*>(&z);
#pragma unroll
    for (int q = 0; q < 4; ++q) zh[q] = __hadd2(xh[q], yh[q]);
    c[i] = z;
  }
}

void launch_sum_plane(__half* g, size_t pe, cudaStream_t s) {
  const size_t n8 = pe / 8;
  if (n8 == 0) return;
  // two CTAs per SM at most: the kernel shares the GPU with the persistent contraction
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n8 + 255) / 256, 2 * 148));
  sum_plane_kernel<<<blocks, 256, 0, s>>>(g, n8, pe);
}

template <typename Src>
static void compress_from(const Src& src, int chil, int d, int b0, int width, int kp, int chirp,
                          const int* lpos, const double* gl, const double* gr, const double* wl, int gplanes,
                          __half* g_out, float2* cinfo_out, double* cs_out, unsigned long long* colmax, int* err,
                          cudaStream_t s, int grid = kGridNone) {
  if (width <= 0) return;
  const int wcols = width * d;
  const int np = round_up(d * chirp, 2 * kBN);
  colmax_kernel<Src><<<dim3((wcols + 127) / 128, (chil + 63) / 64), 128, 0, s>>>(src, chil, d, b0, width, gl, gr,
                                                                                 colmax, err);
  colfinish_kernel<<<(wcols + 127) / 128, 128, 0, s>>>(d, b0, width, chirp, wl, colmax, cinfo_out, cs_out, err,
                                                       grid);
  pack_kernel<Src><<<dim3((wcols + 31) / 32, (chil + 63) / 64), dim3(32, 8), 0, s>>>(
      src, chil, d, b0, width, kp, chirp, lpos, gl, gr, cs_out, gplanes, g_out, np, grid, err);
}

void launch_compress_site(const void* src, int src_prec, int chil, int chir, int d, int b0,
                          int width, int kp, int chirp, const int* lpos, const double* gl,
                          const double* gr, const double* wl, int gplanes, __half* g_out,
                          float2* cinfo_out, double* cs_out, unsigned long long* colmax, int* err,
                          cudaStream_t s, int grid) {
  const size_t stride = static_cast<size_t>(chir) * d;
  if (src_prec == kSrcF64)
    compress_from(ArraySrc<double>{static_cast<const double*>(src), stride}, chil, d, b0, width, kp, chirp, lpos,
                  gl, gr, wl, gplanes, g_out, cinfo_out, cs_out, colmax, err, s, grid);
  else if (src_prec == kSrcF32)
    compress_from(ArraySrc<float>{static_cast<const float*>(src), stride}, chil, d, b0, width, kp, chirp, lpos,
                  gl, gr, wl, gplanes, g_out, cinfo_out, cs_out, colmax, err, s, grid);
  else  // IEEE binary16 bits (MPSB f16 storage): exact in f64
    compress_from(ArraySrc<__half>{static_cast<const __half*>(src), stride}, chil, d, b0, width, kp, chirp, lpos,
                  gl, gr, wl, gplanes, g_out, cinfo_out, cs_out, colmax, err, s, grid);
}

void launch_compress_synth(const SynthSite& g, int chil, int d, int b0, int width, int kp, int chirp,
                           const int* lpos, const double* gl, const double* gr, const double* wl, int gplanes,
                           __half* g_out, float2* cinfo_out, double* cs_out, unsigned long long* colmax,
                           int* err, cudaStream_t s) {
  compress_from(SynthSrc{g}, chil, d, b0, width, kp, chirp, lpos, gl, gr, wl, gplanes, g_out, cinfo_out, cs_out,
                colmax, err, s);
}

}  // namespace mpsg
