// TMA-pipelined gate sweep for sm_100a (the hot loop of SURVEY §8(a) a3/a4).
//
// One persistent CTA per SM (544 threads): warp 16 is the producer, which streams each
// 64 KB tile (2^T amplitudes gathered from 2^(7-m) contiguous runs) into one of 3
// shared-memory stages with cp.async.bulk, completing on a "full" mbarrier.  Warps 0-15
// are two ping-pong consumer groups of 8 warps taking alternate tiles: a group moves
// its tile from shared memory into registers (16-byte vectors, conflict-free), applies
// every X^1/2 / Y^1/2 target of the layer (registers, warp shuffles for lane bits, a
// second register mapping through the same stage when more than 4 high targets),
// releases the stage on its "empty" mbarrier as soon as its last shared-memory read is
// done, applies the fused diagonal and stores straight to HBM.  While one group waits
// or computes, the other group and the next tile's TMA keep the memory system busy.
//
// The fused diagonal (§2.4, Eqs. 3-6) is evaluated through the host-computed
// DiagSplit decomposition: per element one add, one table lookup and one complex
// multiply instead of the full popcount formula.
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
// try_wait with a suspend-time hint: the warp sleeps in the barrier (NANOSLEEP.SYNCS) until
// the phase completes instead of re-polling, so waiting warps leave issue slots to working ones.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(0x989680u)
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
// phB = diag_phase_b(B, d) & 7, evaluated by the caller before the tile's values are live
// (the CZ term loops over pair distances; inside here it would spill)
template <typename R, int NV>
__device__ __forceinline__ void apply_split(typename Cx2<R>::T (&v)[16][NV], const uint32_t B, const uint32_t phB,
                                            const DiagSplit &sp, const typename Cx2<R>::T *tab) {
  using C = typename Cx2<R>::T;
  constexpr int VB = NV == 2 ? 1 : 0;
  constexpr uint32_t pat[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
  const uint32_t pB8 = phB << 3;
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

// Gate kinds (kernels.h): k = g + 2 f, g = 1 SX' / 2 SY', f = the deferred fork this sweep applies
// on the gate's own bit just before the gate (0 none, 1 Z^1: negate the bit-1 side, 2 P0: zero
// the bit-1 side, 3 P1: zero the bit-0 side; Eq. 1 / DESIGN.md §5): cheaper than a pre diagonal.
__device__ __forceinline__ int kind_gate(int k) { return ((k - 1) & 1) + 1; }
__device__ __forceinline__ int kind_fork(int k) { return (k - 1) >> 1; }
template <typename C>
__device__ __forceinline__ void fork_side(C &x, bool hi, int f) {
  if (f == 1) {
    if (hi) x.x = -x.x, x.y = -x.y;
  } else if ((f == 2 && hi) || (f == 3 && !hi)) {
    x.x = 0;
    x.y = 0;
  }
}
template <typename C>
__device__ __forceinline__ void bfly(C &a, C &b, int g) {
  using R = decltype(a.x);
  const R ax = a.x, ay = a.y;
  if (g == 1) {  // SX' = [[1,-i],[-i,1]]
    a.x = ax + b.y;
    a.y = ay - b.x;
    b.x = b.x + ay;
    b.y = b.y - ax;
  } else {  // SY' = [[1,-1],[1,1]]
    a.x = ax - b.x;
    a.y = ay - b.y;
    b.x = ax + b.x;
    b.y = ay + b.y;
  }
}

// gates on the 4 register hi bits of a pass (kinds are uniform: branch outside the loops)
template <typename R, int NV>
__device__ __forceinline__ void reg_gates(typename Cx2<R>::T (&v)[16][NV], const uint8_t *kinds) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int k = kinds[s];
    if (!k) continue;
    const int f = kind_fork(k), g = kind_gate(k);
    if (f) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int e = 0; e < NV; ++e) fork_side(v[r][e], (r >> s) & 1, f);
    }
    if (g == 1) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & (1 << s)) continue;
#pragma unroll
        for (int e = 0; e < NV; ++e) bfly(v[r][e], v[r | (1 << s)][e], 1);
      }
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & (1 << s)) continue;
#pragma unroll
        for (int e = 0; e < NV; ++e) bfly(v[r][e], v[r | (1 << s)][e], 2);
      }
    }
  }
}

// gates on the vector bit (c64, in registers) and on lane bits (warp shuffles)
template <typename R, int NV>
__device__ __forceinline__ void low_gates(typename Cx2<R>::T (&v)[16][NV], const TileSweepParams &p, int lane) {
  if constexpr (NV == 2) {
    const int k = p.lowkind[0];
    if (k) {
      const int f = kind_fork(k), g = kind_gate(k);
      if (f) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          fork_side(v[r][0], false, f);
          fork_side(v[r][1], true, f);
        }
      }
      if (g == 1) {
#pragma unroll
        for (int r = 0; r < 16; ++r) bfly(v[r][0], v[r][1], 1);
      } else {
#pragma unroll
        for (int r = 0; r < 16; ++r) bfly(v[r][0], v[r][1], 2);
      }
    }
  }
  for (int i = 0; i < p.n_lane; ++i) {
    const int lb = p.lane_bit[i];
    const int mask = 1 << lb;
    const int f = kind_fork(p.lane_kind[i]);
    if (f) {
      const bool hi = (lane >> lb) & 1;
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int e = 0; e < NV; ++e) fork_side(v[r][e], hi, f);
    }
    if (kind_gate(p.lane_kind[i]) == 1) {  // both partners: v - i w
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
}

// per-node fork factor (node-batched launches, kernels.h ForkDev) on the pass-0 registers.
// Element (s, e) has index tg | slot bits of s | e (c64: e = bit 0); the fork's zero / sign
// conditions are folded into two 32-bit masks over idx = (s << VB) | e, as in apply_split.
// fork_masks runs before the tile's values are live (register pressure), apply_fork after
template <int NV>
__device__ __forceinline__ void fork_masks(const uint32_t tg, const uint64_t node, const TileSweepParams &p,
                                           uint32_t &zero, uint32_t &neg) {
  constexpr int VB = NV == 2 ? 1 : 0;
  constexpr uint32_t pat[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
  uint32_t fm = 0, fv = 0, zm = 0;
  bool empty = false;  // P0 and P1 on one bit (two cuts on one qubit): the child is zero
  for (int j = 0; j < p.fork.n; ++j) {
    const uint32_t cb = (uint32_t)(node >> (p.fork.n - 1 - j)) & 1u;
    const uint32_t m = 1u << p.fork.bit[j];
    if ((p.fork.pmask >> j) & 1u) {
      if ((fm & m) && ((fv & m) != (cb ? m : 0u))) empty = true;
      fm |= m, fv |= cb ? m : 0u;
    } else if (cb) {
      zm ^= m;  // Z^2 = I
    }
  }
  uint32_t sb[VB + 4];  // state bit of index bit j
  if (VB) sb[0] = 1u;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) sb[VB + kk] = 1u << p.hb[p.gsel[0][kk]];
  uint32_t smask = 0;
#pragma unroll
  for (int j = 0; j < VB + 4; ++j) smask |= sb[j];
  zero = (empty || (((tg & fm) ^ fv) & ~smask)) ? 0xFFFFFFFFu : 0u;
  neg = (__popc(tg & zm & ~smask) & 1) ? 0xFFFFFFFFu : 0u;
#pragma unroll
  for (int j = 0; j < VB + 4; ++j) {
    if (fm & sb[j]) zero |= (fv & sb[j]) ? ~pat[j] : pat[j];
    if (zm & sb[j]) neg ^= pat[j];
  }
}

template <typename R, int NV>
__device__ __forceinline__ void apply_fork(typename Cx2<R>::T (&v)[16][NV], const uint32_t zero, const uint32_t neg) {
  constexpr int VB = NV == 2 ? 1 : 0;
  if (!(zero | neg)) return;
#pragma unroll
  for (int s = 0; s < 16; ++s)
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      const int idx = (s << VB) | e;
      if ((zero >> idx) & 1u) {
        v[s][e].x = v[s][e].y = (R)0;
      } else if ((neg >> idx) & 1u) {
        v[s][e].x = -v[s][e].x;
        v[s][e].y = -v[s][e].y;
      }
    }
}

// the node's branch bits on p.nb_skip (node-batched known-zero tiles)
__device__ __forceinline__ uint32_t nb_skip_value(const uint64_t node, const TileSweepParams &p) {
  uint32_t v = 0;
  if (!p.nb_skip) return 0;
  for (int j = 0; j < p.fork.n; ++j) {
    const uint32_t m = 1u << p.fork.bit[j];
    if ((p.nb_skip & m) && ((node >> (p.fork.n - 1 - j)) & 1u)) v |= m;
  }
  return v;
}

// shared-memory slot index of register slot r for pass q (incrementally OR-ed)
__device__ __forceinline__ uint32_t slot_smem(uint32_t base, const uint8_t *gsel, int r) {
  uint32_t si = base;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (r & (1 << k)) si |= 1u << (5 + gsel[k]);
  return si;
}

// SW = 1: the distributed-half variant whose stores implement a local / global bit swap (p.nswap)
// NB = 1: the node-batched variant (p.log2_nodes, p.node_*, p.fork; multi-part BFS levels)
template <typename R, int PRE, int NPASS, int NST, int SW = 0, int NB = 0>
__global__ void __launch_bounds__(544, 1) tile_sweep_tma_kernel(const __grid_constant__ TileSweepParams p) {
  using C = typename Cx2<R>::T;
  using V = typename Cx2<R>::V;
  constexpr int VB = sizeof(R) == 4 ? 1 : 0;
  constexpr int NV = 1 << VB;
  constexpr int L = 5 + VB;
  constexpr int NVEC = kTileBytes / 16;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V *stages = reinterpret_cast<V *>(smem_raw);
  __shared__ __align__(8) uint64_t full_bar[NST][2], empty_bar[NST];
  __shared__ __align__(16) C tab_pre[8], tab_post[8];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 8) {
    tab_pre[tid].x = (R)(c_omega[2 * tid] * p.pre.scale);
    tab_pre[tid].y = (R)(c_omega[2 * tid + 1] * p.pre.scale);
    tab_post[tid].x = (R)(c_omega[2 * tid] * p.post.scale);
    tab_post[tid].y = (R)(c_omega[2 * tid + 1] * p.post.scale);
  }
  // A projector in the pre diagonal (a deferred fork P_b on a bit of the tile, or on an outer bit)
  // zeroes every element where it fails, so those rows / tiles are not loaded: the contiguous run
  // is cut at the lowest projected hi bit (m_eff), and runs / rows / tiles whose projected bits
  // differ from the projector's values are skipped (their stale shared-memory contents are zeroed
  // by the projector in apply_split before any arithmetic uses them).
  const uint32_t ppm = (PRE != 2 && !p.no_pskip) ? p.ld_pm : 0u, ppv = p.ld_pv;
  int m_eff = p.run_m;
  for (int j = 0; j < p.run_m; ++j)
    if ((ppm >> p.hb[j]) & 1u) {
      m_eff = j;
      break;
    }
  if (m_eff < 2 && p.run_m >= 2) m_eff = p.run_m;  // do not trade bulk runs for per-row loads
  // long contiguous runs: one cp.async.bulk per run (1 arrival + tx bytes); short runs
  // (< 2 KB): per-lane 16-byte cp.async, a warp instruction per 512-byte row (32 arrivals)
  const bool bulk = m_eff >= 2;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s][0], bulk ? 1 : 32);
      mbar_init(&full_bar[s][1], bulk ? 1 : 32);
      mbar_init(&empty_bar[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint64_t ntiles = 1ull << (p.log2_ntiles + (NB ? p.log2_nodes : 0));
  const uint64_t tmask = (1ull << p.log2_ntiles) - 1ull;
  auto tile_outer = [&](uint64_t t64) {
    uint32_t t = (uint32_t)(NB ? (t64 & tmask) : t64), outer = 0;
    for (int q = 0; q < p.nruns; ++q) {
      outer |= (t & ((1u << p.run_len[q]) - 1u)) << p.run_start[q];
      t >>= p.run_len[q];
    }
    return outer;
  };

  if (warp == 16) {
    if constexpr (PRE == 2) return;  // generated sweep: nothing to load
    // ------------------------------------------------ producer: TMA bulk copies
    const int m = m_eff;
    const int rbits = kHiBits - m;
    const int nruns = 1 << rbits;
    const uint32_t run_log2 = L + m;
    const uint32_t run_bytes = (uint32_t)sizeof(C) << run_log2;
    const char *srcb = reinterpret_cast<const char *>(p.src[0]);
    uint32_t hmask = 0, runmask = 0;  // hi bits of the tile; those enumerating the runs
    for (int j = 0; j < kHiBits; ++j) {
      hmask |= 1u << p.hb[j];
      if (j >= m) runmask |= 1u << p.hb[j];
    }
    const uint32_t lowmask = (1u << L) - 1u;
    const uint32_t pout = ppm & ~(hmask | lowmask);          // projected outer bits: whole tiles
    const int npb = __popc(ppm & runmask);                   // projected run bits: 2^-npb of the runs
    const uint32_t tx_bytes = (uint32_t)kTileBytes >> npb;
    for (int it = 0;; ++it) {
      const uint64_t t = blockIdx.x + (uint64_t)it * gridDim.x;
      if (t >= ntiles) break;
      const int s = it % NST;
      const uint32_t par = (uint32_t)(it / NST) & 1u;
      mbar_wait(&empty_bar[s], par ^ 1u);
      uint64_t *fb = &full_bar[s][it & 1];
      const uint32_t outer = tile_outer(t);
      const char *src = srcb;
      if constexpr (NB == 1) src += (size_t)(((t >> p.log2_ntiles) >> p.node_src_shift) * p.node_stride) * sizeof(C);
      char *stage = reinterpret_cast<char *>(stages + (size_t)s * NVEC);
      uint32_t spm = p.skip_pm, spv = p.skip_pv;
      if constexpr (NB == 1) spv = nb_skip_value(t >> p.log2_ntiles, p), spm = p.nb_skip;
      {
        // known-zero tile, or a tile the pre projector zeroes: complete the phase without loading
        if ((outer & spm) != spv || (((outer | p.gbase) ^ ppv) & pout)) {
          if (bulk) {
            if (lane == 0) mbar_arrive(fb);
          } else {
            mbar_arrive(fb);
          }
          continue;
        }
      }
      if (bulk) {
        if (lane == 0) mbar_arrive_expect_tx(fb, tx_bytes);
        __syncwarp();
        for (int q = lane; q < nruns; q += 32) {
          uint32_t gi = outer;
          for (int j = 0; j < rbits; ++j)
            if ((q >> j) & 1) gi |= 1u << p.hb[m + j];
          if ((gi ^ ppv) & ppm & runmask) continue;  // zeroed by the projector
          bulk_g2s(stage + ((size_t)q << run_log2) * sizeof(C), src + (size_t)gi * sizeof(C), run_bytes, fb);
        }
      } else {
        // vector vi = lane + 32 q: row q of the tile = deposit of q's 7 bits on hb[]
        const char *srcl = src + (size_t)(outer | ((uint32_t)lane << VB)) * sizeof(C);
        char *dstl = stage + (size_t)lane * 16;
        const uint32_t rpm = ppm & hmask, rpv = ppv & rpm;
        uint32_t d = 0;
#pragma unroll 8
        for (int q = 0; q < NVEC / 32; ++q) {
          if ((d & rpm) == rpv)
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
  V *dst = reinterpret_cast<V *>(p.dst[0]);
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
    // B-phases of the pre (pass-0 thread base, bits 0-2) and post (last pass, bits 3-5) diagonals
    uint32_t phB = 0, fzero = 0, fneg = 0;
    {
      uint32_t b0 = outer | ((uint32_t)lane << VB) | p.gbase, b1 = b0;
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if ((wl >> j) & 1) {
          b0 |= 1u << p.hb[p.wsel[0][j]];
          b1 |= 1u << p.hb[p.wsel[NPASS - 1][j]];
        }
      if constexpr (PRE >= 1) phB = (uint32_t)diag_phase_b(b0, p.pre) & 7u;
      if (p.post.active) phB |= ((uint32_t)diag_phase_b(b1, p.post) & 7u) << 3;
      if constexpr (NB == 1)
        if (p.fork.n && p.fork_apply) fork_masks<NV>(b0 & ~p.gbase, t >> p.log2_ntiles, p, fzero, fneg);
    }
    if constexpr (PRE != 2) mbar_wait(&full_bar[s][grp], use & 1u);

    // pass 0: shared -> registers
    uint32_t ts = (uint32_t)lane, tg = outer | ((uint32_t)lane << VB);
#pragma unroll
    for (int s = 0; s < 3; ++s)
      if ((wl >> s) & 1) {
        ts |= 1u << (5 + p.wsel[0][s]);
        tg |= 1u << p.hb[p.wsel[0][s]];
      }
    if constexpr (PRE == 2) {  // generated: v = pre(i) (the H layer and the leading diagonals)
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int e = 0; e < NV; ++e) v[r][e].x = (R)1, v[r][e].y = (R)0;
    } else if (NB == 0 ? ((outer & p.skip_pm) != p.skip_pv)
                       : ((outer & p.nb_skip) != nb_skip_value(t >> p.log2_ntiles, p))) {  // known-zero tile
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int e = 0; e < NV; ++e) v[r][e].x = v[r][e].y = (R)0;
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) unpack<R, NV>(tile[slot_smem(ts, p.gsel[0], r)], v[r]);
    }
    if constexpr (NB == 1)
      if (p.fork.n && p.fork_apply) apply_fork<R, NV>(v, fzero, fneg);
    if constexpr (PRE >= 1) apply_split<R, NV>(v, tg | p.gbase, phB & 7u, p.pre_s, tab_pre);
    low_gates<R, NV>(v, p, lane);
    reg_gates<R, NV>(v, p.gkind[0]);

    if constexpr (NPASS == 2) {
#pragma unroll
      for (int r = 0; r < 16; ++r) tile[slot_smem(ts, p.gsel[0], r)] = pack<R, NV>(v[r]);
      asm volatile("bar.sync %0, 256;" ::"r"(1 + grp) : "memory");
      ts = (uint32_t)lane;
      tg = outer | ((uint32_t)lane << VB);
#pragma unroll
      for (int s = 0; s < 3; ++s)
        if ((wl >> s) & 1) {
          ts |= 1u << (5 + p.wsel[1][s]);
          tg |= 1u << p.hb[p.wsel[1][s]];
        }
#pragma unroll
      for (int r = 0; r < 16; ++r) unpack<R, NV>(tile[slot_smem(ts, p.gsel[1], r)], v[r]);
      // the stage is rewritten by TMA next: order our generic-proxy writes before it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    if constexpr (PRE != 2)
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    if constexpr (NPASS == 2) reg_gates<R, NV>(v, p.gkind[1]);

    constexpr int QL = NPASS - 1;
    if (p.post.active) apply_split<R, NV>(v, tg | p.gbase, phB >> 3, p.post_s, tab_post);
    V *dbase = dst;
    if constexpr (NB == 1) dbase += ((t >> p.log2_ntiles) * p.node_stride) >> VB;
    if constexpr (SW == 1) {  // distributed half: this tile's destination rank and address (kernels.h)
      uint32_t delta = 0;
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (j < p.nswap) {
          const uint32_t lb = (outer >> p.swap_l[j]) & 1u, rb = (p.rank >> p.swap_j[j]) & 1u;
          delta |= (lb ^ rb) << p.swap_j[j];
          tg = (tg & ~(1u << p.swap_l[j])) | (rb << p.swap_l[j]);
        }
      dbase = reinterpret_cast<V *>(p.peer[delta]);
    }
    V *d0 = dbase + (tg >> VB);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      uint32_t off = 0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        if (r & (1 << kk)) off |= 1u << (p.hb[p.gsel[QL][kk]] - VB);
      d0[off] = pack<R, NV>(v[r]);
    }
  }
}

template <typename R, int PRE, int NPASS, int NST, int SW = 0, int NB = 0>
static cudaError_t launch_tma_t(const TileSweepParams &p, int grid, cudaStream_t s) {
  tile_sweep_tma_kernel<R, PRE, NPASS, NST, SW, NB><<<grid, 544, (size_t)NST * kTileBytes, s>>>(p);
  return cudaGetLastError();
}

template <typename R, int NST, int SW = 0, int NB = 0>
static cudaError_t launch_tma_r(const TileSweepParams &p, int pre_mode, int npass, int grid, cudaStream_t s) {
  if (npass == 1)
    return pre_mode ? launch_tma_t<R, 1, 1, NST, SW, NB>(p, grid, s) : launch_tma_t<R, 0, 1, NST, SW, NB>(p, grid, s);
  return pre_mode ? launch_tma_t<R, 1, 2, NST, SW, NB>(p, grid, s) : launch_tma_t<R, 0, 2, NST, SW, NB>(p, grid, s);
}

cudaError_t launch_tile_sweep_tma(const TileSweepParams &p, bool c128, int pre_mode, int npass, int grid,
                                  cudaStream_t s, int stages) {
  if (pre_mode == 2) {  // generated sweep (no loads; two stages so the ping-pong groups never share one)
    if (c128)
      return npass == 1 ? launch_tma_t<double, 2, 1, 2>(p, grid, s) : launch_tma_t<double, 2, 2, 2>(p, grid, s);
    return npass == 1 ? launch_tma_t<float, 2, 1, 2>(p, grid, s) : launch_tma_t<float, 2, 2, 2>(p, grid, s);
  }
  if (p.log2_nodes > 0 || p.fork.n > 0) {  // node-batched (multi-part BFS levels)
    if (stages == 3)
      return c128 ? launch_tma_r<double, 3, 0, 1>(p, pre_mode, npass, grid, s)
                  : launch_tma_r<float, 3, 0, 1>(p, pre_mode, npass, grid, s);
    return c128 ? launch_tma_r<double, 2, 0, 1>(p, pre_mode, npass, grid, s)
                : launch_tma_r<float, 2, 0, 1>(p, pre_mode, npass, grid, s);
  }
  if (p.nswap)  // distributed-half swap sweeps: two stages
    return c128 ? launch_tma_r<double, 2, 1>(p, pre_mode, npass, grid, s)
                : launch_tma_r<float, 2, 1>(p, pre_mode, npass, grid, s);
  if (stages == 3)
    return c128 ? launch_tma_r<double, 3>(p, pre_mode, npass, grid, s)
                : launch_tma_r<float, 3>(p, pre_mode, npass, grid, s);
  return c128 ? launch_tma_r<double, 2>(p, pre_mode, npass, grid, s)
              : launch_tma_r<float, 2>(p, pre_mode, npass, grid, s);
}

template <typename R, int NST, int SW = 0, int NB = 0>
static cudaError_t tma_setup_r() {
  const int bytes = NST * kTileBytes;
  const void *fns[4] = {(const void *)tile_sweep_tma_kernel<R, 0, 1, NST, SW, NB>,
                        (const void *)tile_sweep_tma_kernel<R, 1, 1, NST, SW, NB>,
                        (const void *)tile_sweep_tma_kernel<R, 0, 2, NST, SW, NB>,
                        (const void *)tile_sweep_tma_kernel<R, 1, 2, NST, SW, NB>};
  for (const void *f : fns) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename R>
static cudaError_t tma_setup_gen() {
  const int bytes = 2 * kTileBytes;
  cudaError_t e = cudaFuncSetAttribute((const void *)tile_sweep_tma_kernel<R, 2, 1, 2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute((const void *)tile_sweep_tma_kernel<R, 2, 2, 2>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

cudaError_t tile_sweep_tma_setup(bool c128) {
  cudaError_t e = c128 ? tma_setup_r<double, 2>() : tma_setup_r<float, 2>();
  if (e != cudaSuccess) return e;
  e = c128 ? tma_setup_gen<double>() : tma_setup_gen<float>();
  if (e != cudaSuccess) return e;
  e = c128 ? tma_setup_r<double, 2, 1>() : tma_setup_r<float, 2, 1>();
  if (e != cudaSuccess) return e;
  e = c128 ? tma_setup_r<double, 2, 0, 1>() : tma_setup_r<float, 2, 0, 1>();
  if (e != cudaSuccess) return e;
  e = c128 ? tma_setup_r<double, 3, 0, 1>() : tma_setup_r<float, 3, 0, 1>();
  if (e != cudaSuccess) return e;
  return c128 ? tma_setup_r<double, 3>() : tma_setup_r<float, 3>();
}

}  // namespace qsim
