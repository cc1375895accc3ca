// TMA-pipelined fused gate sweep for sm_100a (the hot loop of SURVEY §8(a) a3/a4).
//
// One persistent CTA per SM (544 threads).  Warp 16 is the producer: it streams each
// 64 KB tile (2^T amplitudes gathered from 2^(7-m) contiguous runs) into a shared-memory
// stage — one cp.async.bulk per run when runs are >= 2 KB, else per-lane 16-byte cp.async
// (one warp instruction per 512-byte row) — completing on a "full" mbarrier.  Warps 0-15
// are two ping-pong consumer groups of 8 warps taking alternate tiles.  A group runs up
// to 3 register passes over its tile; in each pass a thread holds 16 slots x 16 bytes
// (4 hi bits in registers, the lane / vector bits are the row's low bits, 3 hi bits are
// warp bits) and executes the pass's op list: butterflies of the factored X^1/2 / Y^1/2
// on register slots, the vector bit or lane bits (warp shuffles), and fused diagonals
// (§2.4 Eqs. 3-6) applied through the host-computed DiagSplit decomposition
// (one add, one table lookup, one complex multiply per amplitude).  Passes are separated
// by a shared-memory remap; the stage is released right after the last pass's shared
// reads, and results are stored straight to HBM.  Several consecutive layers run in one
// launch whenever their high targets fit the tile (one HBM pass instead of several).
#include "sweep_common.cuh"

namespace qsim {

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Fused diagonal through the DiagSplit decomposition (kernels.h).  The phase table
// holds w^k * scale at byte offset 8k (float2) / 16k (double2); the cross terms of
// register bits with their B-side CZ partners are a per-tile parity mask over the slots.
template <typename R, int NV>
__device__ __forceinline__ void apply_split(typename Cx2<R>::T (&v)[16][NV], const uint32_t B, const DiagDev &d,
                                            const DiagSplit &sp, const typename Cx2<R>::T *tab) {
  using C = typename Cx2<R>::T;
  constexpr int VB = NV == 2 ? 1 : 0;
  constexpr uint32_t pat[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
  const uint32_t pB8 = (uint32_t)(diag_phase_b(B, d) & 7) << 3;
  uint32_t cpm = 0;
#pragma unroll
  for (int j = 0; j < VB + 4; ++j)
    if (__popc(B & sp.N[j]) & 1) cpm ^= pat[j];
  const char *tb = reinterpret_cast<const char *>(tab);
#pragma unroll
  for (int s = 0; s < 16; ++s)
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      const int idx = (s << VB) | e;
      const uint32_t cross = (idx <= 5 ? (cpm << (5 - idx)) : (cpm >> (idx - 5))) & 32u;
      const uint32_t off = (pB8 + sp.P[idx] + cross) & 56u;
      const C w = *reinterpret_cast<const C *>(tb + off * (uint32_t)(sizeof(C) / 8));
      v[s][e] = cmul(v[s][e], w);
    }
  if (sp.has_proj) {
    const bool okB = (B & sp.Bpm) == sp.Bpv;
#pragma unroll
    for (int s = 0; s < 16; ++s)
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const int idx = (s << VB) | e;
        if (!okB || ((sp.notok >> idx) & 1u)) v[s][e].x = v[s][e].y = (R)0;
      }
  }
}

// SX' = [[1,-i],[-i,1]]: a' = a - i b, b' = b - i a;   SY' = [[1,-1],[1,1]]: a' = a - b, b' = a + b
template <typename R, int NV, int S>
__device__ __forceinline__ void slot_gate(typename Cx2<R>::T (&v)[16][NV], int kind) {
  if (kind == 1) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & (1 << S)) continue;
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        auto &a = v[r][e];
        auto &b = v[r | (1 << S)][e];
        const R ax = a.x, ay = a.y;
        a.x = ax + b.y;
        a.y = ay - b.x;
        b.x = b.x + ay;
        b.y = b.y - ax;
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & (1 << S)) continue;
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        auto &a = v[r][e];
        auto &b = v[r | (1 << S)][e];
        const R ax = a.x, ay = a.y;
        a.x = ax - b.x;
        a.y = ay - b.y;
        b.x = ax + b.x;
        b.y = ay + b.y;
      }
    }
  }
}

template <typename R, int NV>
__device__ __forceinline__ void vec_gate(typename Cx2<R>::T (&v)[16][NV], int kind) {
  using C = typename Cx2<R>::T;
  if constexpr (NV == 2) {
    if (kind == 1) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        C &a = v[r][0], &b = v[r][1];
        const R ax = a.x, ay = a.y;
        a.x = ax + b.y;
        a.y = ay - b.x;
        b.x = b.x + ay;
        b.y = b.y - ax;
      }
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        C &a = v[r][0], &b = v[r][1];
        const R ax = a.x, ay = a.y;
        a.x = ax - b.x;
        a.y = ay - b.y;
        b.x = ax + b.x;
        b.y = ay + b.y;
      }
    }
  }
}

template <typename R, int NV>
__device__ __forceinline__ void lane_gate(typename Cx2<R>::T (&v)[16][NV], int lb, int kind, int lane) {
  const int mask = 1 << lb;
  if (kind == 1) {  // both partners: v - i w
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const R wx = __shfl_xor_sync(0xffffffffu, v[r][e].x, mask);
        const R wy = __shfl_xor_sync(0xffffffffu, v[r][e].y, mask);
        v[r][e].x += wy;
        v[r][e].y -= wx;
      }
  } else {  // SY': lo = a - b, hi = a + b
    const R sg = ((lane >> lb) & 1) ? (R)1 : (R)-1;
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const R wx = __shfl_xor_sync(0xffffffffu, v[r][e].x, mask);
        const R wy = __shfl_xor_sync(0xffffffffu, v[r][e].y, mask);
        v[r][e].x = fma(sg, wx, v[r][e].x);
        v[r][e].y = fma(sg, wy, v[r][e].y);
      }
  }
}

// one stage: vector-bit gate, lane-bit gates (shuffles), register-slot gates, then a diagonal
template <typename R, int NV>
__device__ __forceinline__ void run_stage(typename Cx2<R>::T (&v)[16][NV], const SweepStage &st, const uint32_t B,
                                          const FusedSweepParams &p, const typename Cx2<R>::T (*tabs)[8],
                                          int lane) {
  if (st.vkind) vec_gate<R, NV>(v, st.vkind);
  for (int i = 0; i < st.nlane; ++i) lane_gate<R, NV>(v, st.lane_bit[i], st.lane_kind[i], lane);
  if (st.gkind[0]) slot_gate<R, NV, 0>(v, st.gkind[0]);
  if (st.gkind[1]) slot_gate<R, NV, 1>(v, st.gkind[1]);
  if (st.gkind[2]) slot_gate<R, NV, 2>(v, st.gkind[2]);
  if (st.gkind[3]) slot_gate<R, NV, 3>(v, st.gkind[3]);
  // static diag indices keep the DiagSplit tables as constant-bank operands
  switch (st.diag) {
    case 0: apply_split<R, NV>(v, B, p.diag[0], p.diag_s[0], tabs[1]); break;
    case 1: apply_split<R, NV>(v, B, p.diag[1], p.diag_s[1], tabs[2]); break;
    case 2: apply_split<R, NV>(v, B, p.diag[2], p.diag_s[2], tabs[3]); break;
    case 3: apply_split<R, NV>(v, B, p.diag[3], p.diag_s[3], tabs[4]); break;
    default: break;
  }
}

// shared-memory slot index of register slot r (pass register bits gsel)
__device__ __forceinline__ uint32_t slot_smem(uint32_t base, const uint8_t *gsel, int r) {
  uint32_t si = base;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (r & (1 << k)) si |= 1u << (5 + gsel[k]);
  return si;
}

// FUSED = 0: one layer (one stage per pass, the layer's diagonal = diag[0] at the end of
// the last pass): straight-line code with static parameter offsets.  FUSED = 1: general
// stage lists (several layers in one HBM pass).
#ifndef RELEASE_LATE
#define RELEASE_LATE 1  // single-layer path: release the stage after the gates (measured faster)
#endif
template <typename R, int PRE, int NPASS, int NST, int FUSED>
__global__ void __launch_bounds__(544, 1) fused_sweep_kernel(const __grid_constant__ FusedSweepParams p) {
  using C = typename Cx2<R>::T;
  using V = typename Cx2<R>::V;
  constexpr int VB = sizeof(R) == 4 ? 1 : 0;
  constexpr int NV = 1 << VB;
  constexpr int L = 5 + VB;
  constexpr int NVEC = kTileBytes / 16;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V *stages = reinterpret_cast<V *>(smem_raw);
  __shared__ __align__(8) uint64_t full_bar[NST][2], empty_bar[NST];
  __shared__ __align__(16) C tabs[1 + kMaxDiag][8];  // [0] pre, [1 + d] diag d

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 8 * (1 + kMaxDiag)) {
    const int t = tid >> 3, k = tid & 7;
    const double sc = t == 0 ? p.pre.scale : (t - 1 < p.ndiag ? p.diag[t - 1].scale : 1.0);
    tabs[t][k].x = (R)(c_omega[2 * k] * sc);
    tabs[t][k].y = (R)(c_omega[2 * k + 1] * sc);
  }
  // long contiguous runs: one cp.async.bulk per run (1 arrival + tx bytes); short runs
  // (< 2 KB): per-lane 16-byte cp.async, a warp instruction per 512-byte row (32 arrivals)
  const bool bulk = p.run_m >= 2;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s][0], bulk ? 1 : 32);
      mbar_init(&full_bar[s][1], bulk ? 1 : 32);
      mbar_init(&empty_bar[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint64_t ntiles = 1ull << p.log2_ntiles;
  auto tile_outer = [&](uint64_t t64) {
    uint32_t t = (uint32_t)t64, outer = 0;
    for (int q = 0; q < p.nruns; ++q) {
      outer |= (t & ((1u << p.run_len[q]) - 1u)) << p.run_start[q];
      t >>= p.run_len[q];
    }
    return outer;
  };

  if (warp == 16) {
    // ------------------------------------------------ producer
    const int m = p.run_m;
    const int rbits = kHiBits - m;
    const int nruns = 1 << rbits;
    const uint32_t run_log2 = L + m;
    const uint32_t run_bytes = (uint32_t)sizeof(C) << run_log2;
    const char *src = reinterpret_cast<const char *>(p.src);
    uint32_t hmask = 0;
    for (int j = 0; j < kHiBits; ++j) hmask |= 1u << p.hb[j];
    for (int it = 0;; ++it) {
      const uint64_t t = blockIdx.x + (uint64_t)it * gridDim.x;
      if (t >= ntiles) break;
      const int s = it % NST;
      const uint32_t par = (uint32_t)(it / NST) & 1u;
      mbar_wait(&empty_bar[s], par ^ 1u);
      uint64_t *fb = &full_bar[s][it & 1];
      const uint32_t outer = tile_outer(t);
      char *stage = reinterpret_cast<char *>(stages + (size_t)s * NVEC);
      if (bulk) {
        if (lane == 0) mbar_arrive_expect_tx(fb, kTileBytes);
        __syncwarp();
        for (int q = lane; q < nruns; q += 32) {
          uint32_t gi = outer;
          for (int j = 0; j < rbits; ++j)
            if ((q >> j) & 1) gi |= 1u << p.hb[m + j];
          bulk_g2s(stage + ((size_t)q << run_log2) * sizeof(C), src + (size_t)gi * sizeof(C), run_bytes, fb);
        }
      } else {
        // vector vi = lane + 32 q: row q of the tile = deposit of q's 7 bits on hb[]
        const char *srcl = src + (size_t)(outer | ((uint32_t)lane << VB)) * sizeof(C);
        char *dstl = stage + (size_t)lane * 16;
        uint32_t d = 0;
#pragma unroll 8
        for (int q = 0; q < NVEC / 32; ++q) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dstl + (size_t)q * 512)),
                       "l"(srcl + (size_t)d * sizeof(C))
                       : "memory");
          d = ((d | ~hmask) + 1u) & hmask;
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(fb)) : "memory");
      }
    }
    return;
  }

  // -------------------------------------------------- two ping-pong consumer groups
  const int grp = warp >> 3, wl = warp & 7;
  V *dst = reinterpret_cast<V *>(p.dst);
  for (int k = 0;; ++k) {
    const int it = 2 * k + grp;  // global tile order: the groups alternate
    const uint64_t t = blockIdx.x + (uint64_t)it * gridDim.x;
    if (t >= ntiles) break;
    const int s = it % NST;
    V *tile = stages + (size_t)s * NVEC;
    const uint32_t outer = tile_outer(t);
    C v[16][NV];
    // full_bar[s][grp] is used by this group only, once per use of stage s: with 2 stages
    // the group always uses stage grp (k-th use); with 3 its tiles cycle the stages
    // (2k + grp mod 3), so the k-th tile is the (k / 3)-th use of its stage
    const uint32_t use = NST == 2 ? (uint32_t)k : (uint32_t)(k / 3);
    mbar_wait(&full_bar[s][grp], use & 1u);

    uint32_t tg = 0;
#pragma unroll
    for (int q = 0; q < NPASS; ++q) {
      uint32_t ts = (uint32_t)lane;
      tg = outer | ((uint32_t)lane << VB);
#pragma unroll
      for (int w = 0; w < 3; ++w)
        if ((wl >> w) & 1) {
          ts |= 1u << (5 + p.wsel[q][w]);
          tg |= 1u << p.hb[p.wsel[q][w]];
        }
#pragma unroll
      for (int r = 0; r < 16; ++r) unpack<R, NV>(tile[slot_smem(ts, p.gsel[q], r)], v[r]);
      if (q == NPASS - 1 && (FUSED || !RELEASE_LATE)) {
        if (NPASS > 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);  // stage free: the next tile can land
      }
      if (PRE == 1 && q == 0) apply_split<R, NV>(v, tg, p.pre, p.pre_s, tabs[0]);
      if constexpr (FUSED) {
        for (int i = 0; i < p.nstage[q]; ++i) run_stage<R, NV>(v, p.stage[q][i], tg, p, tabs, lane);
      } else {
        const SweepStage &st = p.stage[q][0];
        if (q == 0) {
          if (st.vkind) vec_gate<R, NV>(v, st.vkind);
          for (int i = 0; i < st.nlane; ++i) lane_gate<R, NV>(v, st.lane_bit[i], st.lane_kind[i], lane);
        }
        if (st.gkind[0]) slot_gate<R, NV, 0>(v, st.gkind[0]);
        if (st.gkind[1]) slot_gate<R, NV, 1>(v, st.gkind[1]);
        if (st.gkind[2]) slot_gate<R, NV, 2>(v, st.gkind[2]);
        if (st.gkind[3]) slot_gate<R, NV, 3>(v, st.gkind[3]);
        if (q == NPASS - 1 && RELEASE_LATE) {
          if (NPASS > 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[s]);
        }
        if (q == NPASS - 1 && p.ndiag) apply_split<R, NV>(v, tg, p.diag[0], p.diag_s[0], tabs[1]);
      }
      if (q < NPASS - 1) {
#pragma unroll
        for (int r = 0; r < 16; ++r) tile[slot_smem(ts, p.gsel[q], r)] = pack<R, NV>(v[r]);
        asm volatile("bar.sync %0, 256;" ::"r"(1 + grp) : "memory");
      }
    }
    // store the last pass's registers straight to HBM
    constexpr int QL = NPASS - 1;
    V *d0 = dst + (tg >> VB);
    uint32_t ro[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) ro[kk] = 1u << (p.hb[p.gsel[QL][kk]] - VB);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      uint32_t off = 0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        if (r & (1 << kk)) off |= ro[kk];
      d0[off] = pack<R, NV>(v[r]);
    }
  }
}

constexpr int kStages = 2;  // one shared-memory stage per consumer group

template <typename R, int PRE, int NPASS, int FUSED>
static cudaError_t launch_fused_t(const FusedSweepParams &p, int grid, cudaStream_t s) {
  fused_sweep_kernel<R, PRE, NPASS, kStages, FUSED><<<grid, 544, (size_t)kStages * kTileBytes, s>>>(p);
  return cudaGetLastError();
}

template <typename R, int FUSED>
static cudaError_t launch_fused_r(const FusedSweepParams &p, int pre_mode, int grid, cudaStream_t s) {
  switch (p.npass * 2 + (pre_mode ? 1 : 0)) {
    case 2: return launch_fused_t<R, 0, 1, FUSED>(p, grid, s);
    case 3: return launch_fused_t<R, 1, 1, FUSED>(p, grid, s);
    case 4: return launch_fused_t<R, 0, 2, FUSED>(p, grid, s);
    case 5: return launch_fused_t<R, 1, 2, FUSED>(p, grid, s);
    case 6: return launch_fused_t<R, 0, 3, 1>(p, grid, s);
    case 7: return launch_fused_t<R, 1, 3, 1>(p, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fused_sweep(const FusedSweepParams &p, bool c128, int pre_mode, int grid, cudaStream_t s,
                               bool multi_layer) {
  if (multi_layer)
    return c128 ? launch_fused_r<double, 1>(p, pre_mode, grid, s) : launch_fused_r<float, 1>(p, pre_mode, grid, s);
  return c128 ? launch_fused_r<double, 0>(p, pre_mode, grid, s) : launch_fused_r<float, 0>(p, pre_mode, grid, s);
}

template <typename R>
static cudaError_t tma_setup_r() {
  const int bytes = kStages * kTileBytes;
  const void *fns[10] = {
      (const void *)fused_sweep_kernel<R, 0, 1, kStages, 1>, (const void *)fused_sweep_kernel<R, 1, 1, kStages, 1>,
      (const void *)fused_sweep_kernel<R, 0, 2, kStages, 1>, (const void *)fused_sweep_kernel<R, 1, 2, kStages, 1>,
      (const void *)fused_sweep_kernel<R, 0, 3, kStages, 1>, (const void *)fused_sweep_kernel<R, 1, 3, kStages, 1>,
      (const void *)fused_sweep_kernel<R, 0, 1, kStages, 0>, (const void *)fused_sweep_kernel<R, 1, 1, kStages, 0>,
      (const void *)fused_sweep_kernel<R, 0, 2, kStages, 0>, (const void *)fused_sweep_kernel<R, 1, 2, kStages, 0>};
  for (const void *f : fns) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t fused_sweep_setup(bool c128) { return c128 ? tma_setup_r<double>() : tma_setup_r<float>(); }

}  // namespace qsim
