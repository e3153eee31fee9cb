// K1 (3M): the site contraction temp = env x Gamma_i as three real products on tcgen05.
//
//   P_re = E_re . G_re,   P_im = E_im . G_im,   P_s = E_s . G_s     (E_s = E_re + E_im, G_s = G_re + G_im)
//   Re = P_re - P_im,     Im = P_s - P_re - P_im
//
// Gauss's 3-multiplication complex product: 6 instead of 8 issued UMMAs per K-step in SPLIT mode
// (hi + lo environment), 3 instead of 4 in SINGLE mode.  G_s is exact in fp16 by construction
// (quantize_pair in sweep_kernels.cu), E_s is rounded once in fp32 by the select kernel before
// its hi/lo split, so the contraction keeps the F32-class accuracy of the 4M kernel.
//
// Orientation: Gamma is the A operand (M = 256 output columns per CTA pair, 128 per SM) and the
// environment is B (N = 128 samples per unit, each SM stores 64 of them), so one Gamma tile in the
// A collector feeds both the hi and the lo environment MMA.  The three products of a unit run as
// three sequential K loops, each into its own 128-column TMEM slot of a 4-slot ring: while the
// epilogue drains unit t (slots s, s+1, s+2) the MMAs of unit t+1 already fill slot s+3.
//
// Epilogue (4 warps per SM, thread = output column j): Re/Im for 32 samples per TMEM load,
// column scale cs_j, Born weight wl_j |t|^2 and max component per (sample, column); the per-sample
// sums over the warp's 32 columns come from a register transpose-reduction (31 shuffles per 32
// values), then over the 4 warps through shared memory in a fixed order -> pstat[n][tile];
// temp[n][k][r] stores are 256 B contiguous per sample.
//
// Reference: contract_site (contract.cpp:18-41,109-121) + the weight loop of measure
// (sampler.cpp:83-90) + partial_measure_stats (parallel.cpp:90-114).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ptx.cuh"
#include "sweep.cuh"

namespace mpsg {

// kGlo (MPSG_MODE_PRECISE): Gamma carries a lo plane per component too; stage = [A_hi | A_lo | B_hi |
// B_lo] and three MMAs per K16 step (A_hi x B_hi, A_hi x B_lo through the A collector, A_lo x B_hi).
// kTma: temp leaves through TMA tensor stores from a per-warp double-buffered staging area (8 samples
// x 32 columns of float2 per buffer) instead of per-thread 8 B global stores -- the store instructions
// cost ~40% of the epilogue at chi <= 512 (clock64 probes with the stores removed: 7.0k -> 4.1k cycles
// per unit, profiles/r2_prof3m/); one operand stage is given up for the staging area.
template <bool kSplit, bool kGlo = false, bool kTma = false>
struct Cfg3M {
  static constexpr int kHalves = kSplit ? 2 : 1;
  static constexpr int kAHalves = kGlo ? 2 : 1;
  static constexpr int kATile = kBM * kBK3 * 2;        // 16 KiB: 128 Gamma rows x 128 B
  static constexpr int kBTile = (kBM / 2) * kBK3 * 2;  // 8 KiB: this SM's 64 sample rows
  static constexpr int kBOff = kAHalves * kATile;      // B tiles after the A tile(s)
  static constexpr int kStageBytes = kAHalves * kATile + kHalves * kBTile;
  static constexpr int kStages = kGlo ? 4 : (kSplit ? (kTma ? 5 : 6) : (kTma ? 7 : 8));
  static constexpr int kRedBytes = 4 * kBM * 8;        // [4 lane quarters][128 samples] float2
  static constexpr int kBarBytes = 512;
  static constexpr int kOffBytes = 256;                // slice GEMM: bucket offsets
  static constexpr int kTmaBufFloat2 = 8 * 32;         // one staging buffer: 8 samples x 32 columns
  static constexpr int kTmaBytes = kTma ? 8 * 2 * kTmaBufFloat2 * 8 : 0;  // 8 epilogue warps x 2 buffers
  static constexpr int kSmem = kStages * kStageBytes + 1024 + kBarBytes + kRedBytes + kOffBytes + kTmaBytes;
};

int gemm_3m_smem_bytes(bool split) { return split ? Cfg3M<true>::kSmem : Cfg3M<false>::kSmem; }

// Unit u -> (Gamma tile m, sample tile t).  Groups of `group` Gamma tiles are swept over all sample
// tiles (Gamma index fastest), so the group's Gamma planes stay in L2 while each environment tile
// is fetched from DRAM once per group.
// raster & 1 (snake): every other group sweeps the sample tiles in reverse, so it starts on the tiles
// the previous group touched last -- still in L2 -- instead of re-fetching them from DRAM.
// raster & 2 (reversed groups, whole groups only): the groups run last-to-first, so the second
// pipeline lane's launch starts on the Gamma group the first lane's launch left in L2.
__device__ __forceinline__ void unit_coords_3m(int u, const Gemm3MArgs& a, int g_tiles, int& m, int& t) {
  const int per_group = a.group * a.s_tiles;
  const int gi = u / per_group;  // processing order
  const int g = ((a.raster & 2) && g_tiles % a.group == 0) ? (g_tiles / a.group - 1 - gi) : gi;
  const int m0 = g * a.group;
  const int gw = min(a.group, g_tiles - m0);
  const int r = u - gi * per_group;
  t = r / gw;
  m = m0 + (r - t * gw);
  if ((a.raster & 1) && (gi & 1)) t = a.s_tiles - 1 - t;
}

// warps 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4.. epilogue (kEpiWarps = 4 or 8)
constexpr int kEpiSamples = 16;  // samples per epilogue TMEM load (x16)

// v[i] (i = 0..15, one value per sample) summed / maxed over the 32 lanes: afterwards lanes L and
// L ^ 16 hold the reduction for sample L & 15.  Each round halves the vector, exchanging the half
// the partner keeps; the last round folds the two 16-lane halves.
template <bool kMax>
__device__ __forceinline__ float transpose_reduce16(float (&v)[16], int lane) {
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float send = up ? v[i] : v[i + o];
      const float keep = up ? v[i + o] : v[i];
      const float recv = __shfl_xor_sync(0xffffffffu, send, o);
      v[i] = kMax ? fmaxf(keep, recv) : keep + recv;
    }
  }
  const float other = __shfl_xor_sync(0xffffffffu, v[0], 16);
  return kMax ? fmaxf(v[0], other) : v[0] + other;
}

// Timing probes (flags & 32; flags & 64 additionally skips the temp stores -- a timing experiment,
// the results are then wrong): [0] epilogue cycles waiting for the accumulators, [1] epilogue busy
// cycles, [2] MMA cycles waiting for a free TMEM slot, [3] MMA cycles waiting for operands,
// [4] units, [5] epilogue cycles from accumulator-ready to slot release.
__device__ unsigned long long g_prof3m[8];

// kMax: also the per-(sample, tile) max component (tensor-parallel handles exchange it; otherwise
// the select kernel takes the max of the chosen slice itself).
// kQuad: 4-CTA clusters = two CTA pairs working on the same sample tile and adjacent Gamma tiles;
// the pairs share every environment tile through TMA multicast (pair 0 fetches the hi plane, pair 1
// the lo plane, each for both pairs), cutting the L2 -> SM traffic per MMA by a quarter.  A stage
// is refilled only when both pairs have consumed it (commits multicast to all four CTAs).
// kSlice: the slice GEMM of the slice-recompute path (Gemm3MArgs::bcount): units whose sample tile
// misses the bucket of their outcome are skipped by every role alike, and the epilogue writes the
// next environment's hi / lo planes exactly as the select kernel would from temp.
template <bool kSplit, bool kMax, int kEpiWarps, bool kQuad, bool kGlo = false, bool kSlice = false,
          bool kTma = false>
__global__ void __launch_bounds__(128 + 32 * kEpiWarps, 1)
    site_gemm_3m_kernel(const __grid_constant__ CUtensorMap tma_env64,
                        const __grid_constant__ CUtensorMap tma_g, const Gemm3MArgs a,
                        const __grid_constant__ CUtensorMap tma_temp) {
  static_assert(!kTma || (kEpiWarps == 8 && !kGlo && !kSlice && !kQuad), "TMA temp stores: 8-warp K1 only");
  using C = Cfg3M<kSplit, kGlo, kTma>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;  // [2] per unit parity
  uint64_t* tempty = tfull + 2;          // [4] per TMEM slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  float2* red = reinterpret_cast<float2*>(smem + C::kStages * C::kStageBytes + C::kBarBytes);
  int* boff = reinterpret_cast<int*>(smem + C::kStages * C::kStageBytes + C::kBarBytes + C::kRedBytes);
  float2* tbuf = reinterpret_cast<float2*>(smem + C::kStages * C::kStageBytes + C::kBarBytes + C::kRedBytes +
                                           C::kOffBytes);  // 128 B aligned (kTma staging)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int kCl = kQuad ? 4 : 2;
  const int crank = static_cast<int>(ptx::cluster_ctarank());
  const int rank = crank & 1;  // rank within the CTA pair
  const int pair = crank >> 1;
  const bool leader = rank == 0;
  const int cluster = blockIdx.x / kCl;
  const int num_clusters = gridDim.x / kCl;
  const int g_units = kQuad ? (a.g_tiles + 1) >> 1 : a.g_tiles;  // Gamma tile (pairs) per unit row

  if constexpr (kSlice) ptx::grid_dep_wait();  // the prologue reads the selection's bucket counts
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);   // leader: own expect_tx, bytes from both CTAs
      ptx::mbar_init(&empty[s], kQuad ? 2 : 1);  // the leaders' multicast commits
    }
    for (int j = 0; j < 2; ++j) ptx::mbar_init(&tfull[j], 1);
    for (int j = 0; j < 4; ++j) ptx::mbar_init(&tempty[j], 2 * kEpiWarps);  // epilogue warps x 2 CTAs
    ptx::fence_mbar_init();
    if constexpr (kSlice) {  // bucket k = rows [boff[k], boff[k + 1])
      int o = 0;
      for (int k = 0; k <= a.d; ++k) {
        boff[k] = o;
        o += a.bcount[k];
      }
      boff[a.d + 1] = o;
    }
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tma_env64);
    ptx::tma_prefetch_desc(&tma_g);
  }
  if (warp == 2) {
    ptx::tmem_alloc_pair(tmem_slot, 512);  // 4 slots x 128 fp32 columns
    ptx::tmem_relinquish_pair();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: the prologue above overlapped the previous kernel's tail; from
  // here on the previous selection's environment writes / temp reads must be complete.
  ptx::grid_dep_wait();
  ptx::grid_dep_launch();
  const int units = g_units * a.s_tiles;
  // slice GEMM: does Gamma tile pair m (outcome of either SM's 128 columns) meet sample tile t's rows?
  auto unit_on = [&](int m, int t) -> bool {
    if constexpr (!kSlice) {
      return true;
    } else {
      const int r0 = t * kBM, r1 = r0 + kBM;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int k = (m * 2 * kBM + hh * kBM) / a.chirp;
        if (k < a.d && boff[k] < r1 && boff[k + 1] > r0) return true;
      }
      return false;
    }
  };

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; bytes counted on the leader's barrier) ----------
    if (lane == 0) {
      const uint64_t pol_env = ptx::l2_policy_evict_normal();
      const uint64_t pol_g = ptx::l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cluster; u < units; u += num_clusters) {
        int m, t;
        unit_coords_3m(u, a, g_units, m, t);
        if (kQuad) m = 2 * m + pair;
        if (!unit_on(m, t)) continue;
        const int grow = m * 2 * kBM + rank * kBM;     // this SM's Gamma rows
        const int erow = t * kBM + rank * (kBM / 2);   // this SM's sample rows
#pragma unroll 1
        for (int c = 0; c < 3; ++c) {
          int shard = 0, kin = 0;
          for (int kb = 0; kb < a.k_blocks; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + stage * C::kStageBytes;
            const uint32_t lbar = ptx::leader_bar(&full[stage]);
            if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
            ptx::tma_load_2d_pair(&tma_g, lbar, st, kb * kBK3, c * a.np + grow, pol_g);
            if constexpr (kGlo)  // the component's lo plane (planes 3..5)
              ptx::tma_load_2d_pair(&tma_g, lbar, st + C::kATile, kb * kBK3, (3 + c) * a.np + grow, pol_g);
            if constexpr (kQuad) {  // env plane h = pair for both pairs (same rows: same rank)
              if (pair < C::kHalves)
                ptx::tma_load_3d_pair_mc(&tma_env64, lbar, st + C::kBOff + pair * C::kBTile, kin * kBK3,
                                         (3 * pair + c) * a.env_cap + erow, shard,
                                         static_cast<uint16_t>((1u << rank) | (1u << (rank + 2))), pol_env);
            } else {
#pragma unroll
              for (int h = 0; h < C::kHalves; ++h)
                ptx::tma_load_3d_pair(&tma_env64, lbar, st + C::kBOff + h * C::kBTile, kin * kBK3,
                                      (3 * h + c) * a.env_cap + erow, shard, pol_env);
            }
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
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the leader CTA's warp 1 drives both SMs ----------------
    // The whole warp runs the loop (uniform control flow and operands); one elected lane issues.
    if (leader) {
      constexpr uint32_t kId = ptx::idesc_f16_f32(2 * kBM, kBM, false);
      const uint64_t desc0 = ptx::sdesc_kmajor_sw128(ptx::smem_u32(smem));
      long long w_slot = 0, w_full = 0;
      int stage = 0;
      uint32_t phase = 0;
      uint32_t gp = 0;  // running product index: TMEM slot gp % 4
      int unit = 0;
      for (int u = cluster; u < units; u += num_clusters) {
        if constexpr (kSlice) {
          int m, t;
          unit_coords_3m(u, a, g_units, m, t);
          if (!unit_on(m, t)) continue;
        }
#pragma unroll 1
        for (int c = 0; c < 3; ++c, ++gp) {
          const uint32_t slot = gp & 3;
          long long t0 = (a.flags & 32) ? clock64() : 0;
          ptx::mbar_wait(&tempty[slot], ((gp >> 2) & 1) ^ 1);
          if (a.flags & 32) w_slot += clock64() - t0;
          ptx::tc_fence_after();
          const uint32_t d = tmem_base + slot * 128;
          for (int kb = 0; kb < a.k_blocks; ++kb) {
            if (a.flags & 32) t0 = clock64();
            ptx::mbar_wait(&full[stage], phase);
            if (a.flags & 32) w_full += clock64() - t0;
            ptx::tc_fence_after();
            // descriptor start addresses are in 16 B units: +32 B per K16 step inside the atom
            const uint64_t ad = desc0 + ((stage * C::kStageBytes) >> 4);
            const uint64_t bd = ad + (C::kBOff >> 4);
#pragma unroll
            for (int ks = 0; ks < kBK3 / 16; ++ks) {
              const uint32_t accum = (kb | ks) ? 1u : 0u;
              if constexpr (kSplit) {
                ptx::umma_pair_elect(d, ad + 2 * ks, bd + 2 * ks, kId, accum, true, false);
                ptx::umma_pair_elect(d, ad + 2 * ks, bd + (C::kBTile >> 4) + 2 * ks, kId, 1u, false, true);
                if constexpr (kGlo)  // Gamma lo x env hi
                  ptx::umma_pair_elect(d, ad + (C::kATile >> 4) + 2 * ks, bd + 2 * ks, kId, 1u, false, false);
              } else {
                ptx::umma_pair_elect(d, ad + 2 * ks, bd + 2 * ks, kId, accum, false, false);
              }
            }
            ptx::umma_commit_pair_mc_elect(&empty[stage], kQuad ? 0xF : 0x3);
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        // all three products of the unit done -> this pair's epilogues
        ptx::umma_commit_pair_mc_elect(&tfull[unit & 1], static_cast<uint16_t>(0x3u << (2 * pair)));
        ++unit;
      }
      if ((a.flags & 32) && lane == 0) {
        atomicAdd(&g_prof3m[2], static_cast<unsigned long long>(w_slot));
        atomicAdd(&g_prof3m[3], static_cast<unsigned long long>(w_full));
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs): kEpiWarps / 4 warps per TMEM lane quarter; thread = one
    // of this SM's 128 output columns, warp part h covers samples [kSpan h, kSpan h + kSpan) -----
    constexpr int kSpan = kBM * 4 / kEpiWarps;  // samples per epilogue warp and unit
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;
    const int ec = q * 32 + lane;  // column within the SM's 128
    uint32_t gp = 0;
    int unit = 0;
    int tst = 0;  // kTma: this warp's staging-buffer sequence number
    const uint64_t pol_temp = kTma ? ptx::l2_policy_evict_first() : 0;
    for (int u = cluster; u < units; u += num_clusters) {
      int m, t;
      unit_coords_3m(u, a, g_units, m, t);
      if (kQuad) m = 2 * m + pair;
      if (!unit_on(m, t)) continue;
      const int col0 = m * 2 * kBM + rank * kBM;  // first of this SM's 128 columns (one outcome)
      const int k = col0 / a.chirp;
      // the pair-padding tile (and a quad's phantom odd Gamma tile) has nothing to store
      const bool valid = k < a.d && m < a.g_tiles;
      const int r = col0 - k * a.chirp + ec;
      const float2 ci = valid ? a.cinfo[col0 + ec] : make_float2(0.f, 0.f);
      const long long e0 = (a.flags & 32) ? clock64() : 0;
      ptx::mbar_wait(&tfull[unit & 1], (unit >> 1) & 1);
      const long long e1 = (a.flags & 32) ? clock64() : 0;
      long long e2 = 0;
      ptx::tc_fence_after();
      const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
      const uint32_t c0 = h * kSpan;
      const uint32_t t_re = tmem_base + lanes + ((gp + 0) & 3) * 128 + c0;
      const uint32_t t_im = tmem_base + lanes + ((gp + 1) & 3) * 128 + c0;
      const uint32_t t_s = tmem_base + lanes + ((gp + 2) & 3) * 128 + c0;
      const size_t row_stride = static_cast<size_t>(a.d) * a.chirp;
      // (flags & 128: diagnostic -- every sample tile stores into the first 8 tiles' rows, an L2-resident
      // region, to time the epilogue when the temp stream never reaches DRAM; results are then wrong)
      const int tt = (a.flags & 128) ? (t & 7) : t;
      float2* dst = a.temp == nullptr ? nullptr
                    : a.temp + (static_cast<size_t>(tt) * kBM + c0) * row_stride + static_cast<size_t>(k) * a.chirp + r;
#pragma unroll 1
      for (int ch = 0; ch < kSpan / kEpiSamples; ++ch) {
        float pr[kEpiSamples], pi[kEpiSamples], ps[kEpiSamples];
        ptx::tmem_ld_32x32b_x16(t_re + ch * kEpiSamples, pr);
        ptx::tmem_ld_32x32b_x16(t_im + ch * kEpiSamples, pi);
        ptx::tmem_ld_32x32b_x16(t_s + ch * kEpiSamples, ps);
        ptx::tmem_wait_ld();
        if (ch == kSpan / kEpiSamples - 1) {  // this warp's part of the unit's three slots is read
          ptx::tc_fence_before();
          __syncwarp();
          if (a.flags & 32) e2 = clock64();
          if (lane == 0) {
            ptx::mbar_arrive_remote_relaxed(&tempty[(gp + 0) & 3], 2 * pair);
            ptx::mbar_arrive_remote_relaxed(&tempty[(gp + 1) & 3], 2 * pair);
            ptx::mbar_arrive_remote_relaxed(&tempty[(gp + 2) & 3], 2 * pair);
          }
        }
        if constexpr (kSlice) {
          // next environment rows of this SM's outcome bucket: E = temp * scale split hi / lo per
          // component re, im, re + im (env_split, the select kernel's arithmetic)
          if (valid && r < a.kp_next) {
            const int j0 = t * kBM + c0 + ch * kEpiSamples;
            const int lo = boff[k], hi = boff[k + 1];
            const size_t plane = static_cast<size_t>(a.env_cap) * a.kp_next;
#pragma unroll
            for (int i = 0; i < kEpiSamples; ++i) {
              const int j = j0 + i;
              if (j < lo || j >= hi) continue;
              const float re = (pr[i] - pi[i]) * ci.x;
              const float im = (ps[i] - pr[i] - pi[i]) * ci.x;
              const float sc = a.scale[j];
              __half hv[3], lv[3];
              env_split(re * sc, im * sc, hv, lv);
              __half* e0 = a.env_next + static_cast<size_t>(j) * a.kp_next + r;
#pragma unroll
              for (int cc = 0; cc < 3; ++cc) {
                e0[cc * plane] = hv[cc];
                e0[(3 + cc) * plane] = lv[cc];
              }
            }
          }
        } else if (valid) {
          if constexpr (kTma) {
            // two 8-sample halves through this warp's double-buffered staging area: lane = column,
            // one 8 x 32 float2 TMA tensor store per half (256 B contiguous per sample in temp)
            float2* wbuf = tbuf + (warp - 4) * 2 * C::kTmaBufFloat2;
#pragma unroll
            for (int hf = 0; hf < kEpiSamples / 8; ++hf) {
              float2* buf = wbuf + (tst & 1) * C::kTmaBufFloat2;
              if (tst >= 2 && lane == 0) ptx::bulk_wait_group_read<1>();  // this buffer's last store read it
              __syncwarp();
#pragma unroll
              for (int i8 = 0; i8 < 8; ++i8) {
                const int i = hf * 8 + i8;
                const float re = (pr[i] - pi[i]) * ci.x;
                const float im = (ps[i] - pr[i] - pi[i]) * ci.x;
                buf[i8 * 32 + lane] = make_float2(re, im);
                pr[i] = ci.y * fmaf(re, re, im * im);
                if constexpr (kMax) pi[i] = fmaxf(fabsf(re), fabsf(im));
              }
              ptx::fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                ptx::tma_store_3d(&tma_temp, buf, col0 - k * a.chirp + q * 32, k,
                                  t * kBM + static_cast<int>(c0) + ch * kEpiSamples + hf * 8, pol_temp);
                ptx::bulk_commit_group();
              }
              ++tst;
            }
          } else {
#pragma unroll
            for (int i = 0; i < kEpiSamples; ++i) {
              const float re = (pr[i] - pi[i]) * ci.x;
              const float im = (ps[i] - pr[i] - pi[i]) * ci.x;
              // streaming store: temp (1.6 GB per c3 site) must not evict the Gamma group from L2;
              // no temp at all on the slice-recompute path (weights only)
              // (flags & 64: diagnostic -- skip the stores, to time the epilogue without them)
              if (a.temp != nullptr && !(a.flags & 64))
                __stcs(dst + (ch * kEpiSamples + i) * row_stride, make_float2(re, im));
              pr[i] = ci.y * fmaf(re, re, im * im);
              if constexpr (kMax) pi[i] = fmaxf(fabsf(re), fabsf(im));
            }
          }
          const float w = transpose_reduce16<false>(pr, lane);
          float mx = 0.f;
          if constexpr (kMax) mx = transpose_reduce16<true>(pi, lane);
          if (lane < 16) red[q * kBM + c0 + ch * kEpiSamples + lane] = make_float2(w, mx);
        }
      }
      if (valid && !kSlice) {
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        if (h == 0) {  // thread ec reduces sample ec of the unit over the 4 lane quarters, in order
          float2 v = red[ec];
#pragma unroll
          for (int w = 1; w < 4; ++w) {
            const float2 o = red[w * kBM + ec];
            v.x += o.x;
            v.y = fmaxf(v.y, o.y);
          }
          a.pstat[(static_cast<size_t>(t) * kBM + ec) * a.nt + col0 / kBM] = v;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");  // red is rewritten next unit
      }
      if ((a.flags & 32) && threadIdx.x == 128) {
        const long long e3 = clock64();
        atomicAdd(&g_prof3m[0], static_cast<unsigned long long>(e1 - e0));
        atomicAdd(&g_prof3m[1], static_cast<unsigned long long>(e3 - e1));
        atomicAdd(&g_prof3m[5], static_cast<unsigned long long>(e2 - e1));
        atomicAdd(&g_prof3m[4], 1ull);
      }
      ++unit;
      gp += 3;
    }
    if constexpr (kTma) {
      if (lane == 0) ptx::bulk_wait_group<0>();  // this warp's temp stores performed
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

template <bool kSplit, bool kMax, int kEpiWarps, bool kQuad, bool kGlo = false, bool kSlice = false,
          bool kTma = false>
static void launch_3m_t(const CUtensorMap& tma_env64, const CUtensorMap& tma_g, const Gemm3MArgs& a,
                        int grid, cudaStream_t s, const CUtensorMap* tma_temp = nullptr) {
  auto kern = site_gemm_3m_kernel<kSplit, kMax, kEpiWarps, kQuad, kGlo, kSlice, kTma>;
  using Cf = Cfg3M<kSplit, kGlo, kTma>;
  constexpr int kCl = kQuad ? 4 : 2;
  static PerDevice clusters;  // per device: smem opt-in + occupancy query
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(128 + 32 * kEpiWarps);
  cfg.dynamicSmemBytes = Cf::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int max_clusters = clusters.get([&] {
    check_launch(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmem),
                 "site_gemm_3m_kernel smem opt-in");
    cudaLaunchConfig_t q = cfg;
    q.gridDim = dim3(kCl);
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &q) != cudaSuccess || mc < 1) {
      cudaGetLastError();
      mc = 148 / kCl;  // 4-CTA clusters: 33 on a B200 (132 SMs)
    }
    return mc;
  });
  cfg.gridDim = dim3(kCl * std::max(1, std::min(max_clusters, grid / kCl)));
  if (a.pdl) cfg.numAttrs = 2;
  // kernels without TMA temp stores never read the map: pass any valid one
  check_launch(cudaLaunchKernelEx(&cfg, kern, tma_env64, tma_g, a, tma_temp ? *tma_temp : tma_g),
               "site_gemm_3m_kernel");
}

template <bool kSplit, bool kMax>
static void launch_3m_w(int epi_warps, bool quad, bool glo, const CUtensorMap& e, const CUtensorMap& g,
                        const Gemm3MArgs& a, int grid, cudaStream_t s, const CUtensorMap* tma_temp) {
  if constexpr (kSplit) {
    if (glo) {
      launch_3m_t<kSplit, kMax, 8, false, true>(e, g, a, grid, s);
      return;
    }
  }
  if (tma_temp && !quad && epi_warps == 8) {
    launch_3m_t<kSplit, kMax, 8, false, false, false, true>(e, g, a, grid, s, tma_temp);
    return;
  }
  if (quad)
    launch_3m_t<kSplit, kMax, 8, true>(e, g, a, grid, s);
  else if (epi_warps == 4)
    launch_3m_t<kSplit, kMax, 4, false>(e, g, a, grid, s);
  else if (epi_warps == 16)
    launch_3m_t<kSplit, kMax, 16, false>(e, g, a, grid, s);
  else
    launch_3m_t<kSplit, kMax, 8, false>(e, g, a, grid, s);
}

void launch_site_gemm_3m(bool split, bool with_max, int epi_warps, bool quad, bool glo,
                         const CUtensorMap& tma_env64, const CUtensorMap& tma_g, const Gemm3MArgs& a,
                         int grid, cudaStream_t s, bool slice, const CUtensorMap* tma_temp) {
  if (slice) {  // slice GEMM: 8 epilogue warps, CTA pairs
    if (split)
      glo ? launch_3m_t<true, false, 8, false, true, true>(tma_env64, tma_g, a, grid, s)
          : launch_3m_t<true, false, 8, false, false, true>(tma_env64, tma_g, a, grid, s);
    else
      launch_3m_t<false, false, 8, false, false, true>(tma_env64, tma_g, a, grid, s);
    return;
  }
  if (a.temp == nullptr) tma_temp = nullptr;  // weights only: nothing to store
  if (split)
    with_max ? launch_3m_w<true, true>(epi_warps, quad, glo, tma_env64, tma_g, a, grid, s, tma_temp)
             : launch_3m_w<true, false>(epi_warps, quad, glo, tma_env64, tma_g, a, grid, s, tma_temp);
  else
    with_max ? launch_3m_w<false, true>(epi_warps, quad, glo, tma_env64, tma_g, a, grid, s, tma_temp)
             : launch_3m_w<false, false>(epi_warps, quad, glo, tma_env64, tma_g, a, grid, s, tma_temp);
}

}  // namespace mpsg

// diagnostics (not part of include/mpsg.h): read and reset the 3M kernel's timing probes
extern "C" __attribute__((visibility("default"))) int mpsg_debug_prof3m(unsigned long long* out, int n) {
  unsigned long long h[8] = {0};
  if (cudaMemcpyFromSymbol(h, mpsg::g_prof3m, sizeof(h)) != cudaSuccess) return 5;
  const unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(mpsg::g_prof3m, z, sizeof(z));
  for (int i = 0; i < n && i < 8; ++i) out[i] = h[i];
  return 0;
}
