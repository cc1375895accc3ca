// Gate-sweep kernels for sm_100a: one HBM pass applies all X^1/2 / Y^1/2 gates of a
// layer plus the fused diagonal of every CZ / T / projector / Z around it
// (§2.4: the bottleneck is memory traffic, so a layer's diagonal
// gates are combined into one pass, Eqs. 3-6).
#include <type_traits>

#include "sweep_common.cuh"

namespace qsim {

// ----------------------------------------------------------------------------------
// Tile sweep.  Thread (warp w, lane l) in pass q owns the 16 x NV amplitudes with
//   u = [vector bit(s)] | l << VB | (w bits on hb[wsel[q][*]]) | (r bits on hb[gsel[q][*]])
// so for every register slot r the 32 lanes of a warp touch one contiguous 512-byte
// row (coalesced global access, conflict-free 16-byte shared access).
template <typename R, int PRE, int NPASS>
__global__ void __launch_bounds__(256, 2) tile_sweep_kernel(const __grid_constant__ TileSweepParams p) {
  using C = typename Cx2<R>::T;
  using V = typename Cx2<R>::V;
  constexpr int VB = sizeof(R) == 4 ? 1 : 0;
  constexpr int NV = 1 << VB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *tile = reinterpret_cast<V *>(smem_raw);
  __shared__ C tab_pre[8], tab_post[8];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 8) {
    const int k = threadIdx.x;
    tab_pre[k].x = (R)(c_omega[2 * k] * p.pre.scale);
    tab_pre[k].y = (R)(c_omega[2 * k + 1] * p.pre.scale);
    tab_post[k].x = (R)(c_omega[2 * k] * p.post.scale);
    tab_post[k].y = (R)(c_omega[2 * k + 1] * p.post.scale);
  }
  __syncthreads();

  const uint64_t tiles_per_job = 1ull << p.log2_ntiles;
  const uint64_t total = tiles_per_job * (uint64_t)p.njobs;
  for (uint64_t jt = blockIdx.x; jt < total; jt += gridDim.x) {
    const int job = (int)(jt >> p.log2_ntiles);
    uint32_t rem = (uint32_t)(jt & (tiles_per_job - 1));
    uint32_t outer = 0;
    for (int q = 0; q < p.nruns; ++q) {
      outer |= (rem & ((1u << p.run_len[q]) - 1u)) << p.run_start[q];
      rem >>= p.run_len[q];
    }
    C v[16][NV];

    // ------------------------------------------------------------ pass 0 (global load)
    {
      uint32_t tg = outer | ((uint32_t)lane << VB);
      uint32_t ts = (uint32_t)lane;
#pragma unroll
      for (int s = 0; s < 3; ++s)
        if ((warp >> s) & 1) {
          tg |= 1u << p.hb[p.wsel[0][s]];
          ts |= 1u << (5 + p.wsel[0][s]);
        }
      uint32_t rg[4], rs[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        rg[s] = 1u << p.hb[p.gsel[0][s]];
        rs[s] = 1u << (5 + p.gsel[0][s]);
      }
      const V *src = reinterpret_cast<const V *>(p.src[job]);
      const uint32_t pre_pv = p.job_pv[job], pre_zm = p.job_zm[job];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t gi = tg | ((r & 1) ? rg[0] : 0u) | ((r & 2) ? rg[1] : 0u) |
                            ((r & 4) ? rg[2] : 0u) | ((r & 8) ? rg[3] : 0u);
        if constexpr (PRE == 2) {
#pragma unroll
          for (int e = 0; e < NV; ++e) {
            const uint32_t idx = (gi + e) | p.gbase;  // global index (distributed half)
            C x = tab_pre[diag_phase(idx, p.pre, pre_zm)];
            if ((idx & p.pre.pm) != pre_pv) x.x = x.y = (R)0;
            v[r][e] = x;
          }
        } else {
          unpack<R, NV>(src[gi >> VB], v[r]);
          if constexpr (PRE == 1) {
#pragma unroll
            for (int e = 0; e < NV; ++e) {
              const uint32_t idx = (gi + e) | p.gbase;  // global index (distributed half)
              C x = cmul(v[r][e], tab_pre[diag_phase(idx, p.pre, pre_zm)]);
              if ((idx & p.pre.pm) != pre_pv) x.x = x.y = (R)0;
              v[r][e] = x;
            }
          }
        }
      }
      // gates on the vector bit (c64: global bit 0) - in registers
      if constexpr (VB == 1) {
        const int k = p.lowkind[0];
        if (k) {
#pragma unroll
          for (int r = 0; r < 16; ++r) butterfly(k, v[r][0], v[r][1]);
        }
      }
      // gates on lane bits - warp shuffles
#pragma unroll
      for (int lb = 0; lb < 5; ++lb) {
        const int k = p.lowkind[VB + lb];
        if (!k) continue;
        const bool hi = (lane >> lb) & 1;
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
          for (int e = 0; e < NV; ++e) {
            C w;
            w.x = __shfl_xor_sync(0xffffffffu, v[r][e].x, 1 << lb);
            w.y = __shfl_xor_sync(0xffffffffu, v[r][e].y, 1 << lb);
            C &a = v[r][e];
            if (k == 1) {  // v - i w (both halves)
              a.x = a.x + w.y;
              a.y = a.y - w.x;
            } else if (hi) {  // SY': hi = a + b
              a.x = w.x + a.x;
              a.y = w.y + a.y;
            } else {  // lo = a - b
              a.x = a.x - w.x;
              a.y = a.y - w.y;
            }
          }
      }
      // gates on register hi bits
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int k = p.gkind[0][s];
        if (!k) continue;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          if (r & (1 << s)) continue;
#pragma unroll
          for (int e = 0; e < NV; ++e) butterfly(k, v[r][e], v[r | (1 << s)][e]);
        }
      }
      if constexpr (NPASS == 1) {
        V *dst = reinterpret_cast<V *>(p.dst[job]);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const uint32_t gi = tg | ((r & 1) ? rg[0] : 0u) | ((r & 2) ? rg[1] : 0u) |
                              ((r & 4) ? rg[2] : 0u) | ((r & 8) ? rg[3] : 0u);
          if (p.post.active) {
#pragma unroll
            for (int e = 0; e < NV; ++e) {
              const uint32_t idx = (gi + e) | p.gbase;  // global index (distributed half)
              C x = cmul(v[r][e], tab_post[diag_phase(idx, p.post, p.post.zm)]);
              if ((idx & p.post.pm) != p.post.pv) x.x = x.y = (R)0;
              v[r][e] = x;
            }
          }
          dst[gi >> VB] = pack<R, NV>(v[r]);
        }
      } else {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const uint32_t si = ts | ((r & 1) ? rs[0] : 0u) | ((r & 2) ? rs[1] : 0u) |
                              ((r & 4) ? rs[2] : 0u) | ((r & 8) ? rs[3] : 0u);
          tile[si] = pack<R, NV>(v[r]);
        }
      }
    }

    // ------------------------------------------------------------ pass 1 (shared memory)
    if constexpr (NPASS == 2) {
      __syncthreads();
      uint32_t tg = outer | ((uint32_t)lane << VB);
      uint32_t ts = (uint32_t)lane;
#pragma unroll
      for (int s = 0; s < 3; ++s)
        if ((warp >> s) & 1) {
          tg |= 1u << p.hb[p.wsel[1][s]];
          ts |= 1u << (5 + p.wsel[1][s]);
        }
      uint32_t rg[4], rs[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        rg[s] = 1u << p.hb[p.gsel[1][s]];
        rs[s] = 1u << (5 + p.gsel[1][s]);
      }
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t si = ts | ((r & 1) ? rs[0] : 0u) | ((r & 2) ? rs[1] : 0u) |
                            ((r & 4) ? rs[2] : 0u) | ((r & 8) ? rs[3] : 0u);
        unpack<R, NV>(tile[si], v[r]);
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int k = p.gkind[1][s];
        if (!k) continue;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          if (r & (1 << s)) continue;
#pragma unroll
          for (int e = 0; e < NV; ++e) butterfly(k, v[r][e], v[r | (1 << s)][e]);
        }
      }
      V *dst = reinterpret_cast<V *>(p.dst[job]);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t gi = tg | ((r & 1) ? rg[0] : 0u) | ((r & 2) ? rg[1] : 0u) |
                            ((r & 4) ? rg[2] : 0u) | ((r & 8) ? rg[3] : 0u);
        if (p.post.active) {
#pragma unroll
          for (int e = 0; e < NV; ++e) {
            const uint32_t idx = (gi + e) | p.gbase;  // global index (distributed half)
            C x = cmul(v[r][e], tab_post[diag_phase(idx, p.post, p.post.zm)]);
            if ((idx & p.post.pm) != p.post.pv) x.x = x.y = (R)0;
            v[r][e] = x;
          }
        }
        dst[gi >> VB] = pack<R, NV>(v[r]);
      }
      __syncthreads();
    }
  }
}

int tile_low_bits(bool c128) { return c128 ? 5 : 6; }

template <typename R, int PRE, int NPASS>
static cudaError_t launch_tile_t(const TileSweepParams &p, int grid, cudaStream_t s) {
  const size_t smem = NPASS == 2 ? (size_t)65536 : 0;
  tile_sweep_kernel<R, PRE, NPASS><<<grid, 256, smem, s>>>(p);
  return cudaGetLastError();
}

template <typename R>
static cudaError_t launch_tile_r(const TileSweepParams &p, int pre_mode, int npass, int grid,
                                 cudaStream_t s) {
  if (npass == 1) {
    if (pre_mode == 0) return launch_tile_t<R, 0, 1>(p, grid, s);
    if (pre_mode == 1) return launch_tile_t<R, 1, 1>(p, grid, s);
    return launch_tile_t<R, 2, 1>(p, grid, s);
  }
  if (pre_mode == 0) return launch_tile_t<R, 0, 2>(p, grid, s);
  if (pre_mode == 1) return launch_tile_t<R, 1, 2>(p, grid, s);
  return launch_tile_t<R, 2, 2>(p, grid, s);
}

cudaError_t launch_tile_sweep(const TileSweepParams &p, bool c128, int pre_mode, int npass,
                              int grid, cudaStream_t s) {
  return c128 ? launch_tile_r<double>(p, pre_mode, npass, grid, s)
              : launch_tile_r<float>(p, pre_mode, npass, grid, s);
}

template <typename R>
static cudaError_t setup_r(int *b1, int *b2) {
  cudaError_t e;
#define QSIM_SET(PRE)                                                                              \
  e = cudaFuncSetAttribute(tile_sweep_kernel<R, PRE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           65536);                                                                 \
  if (e != cudaSuccess) return e;
  QSIM_SET(0)
  QSIM_SET(1)
  QSIM_SET(2)
#undef QSIM_SET
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(b1, tile_sweep_kernel<R, 1, 1>, 256, 0);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(b2, tile_sweep_kernel<R, 1, 2>, 256, 65536);
}

cudaError_t tile_sweep_setup(int *b1, int *b2, bool c128) {
  return c128 ? setup_r<double>(b1, b2) : setup_r<float>(b1, b2);
}

// ----------------------------------------------------------------------------------
// Small half states (h <= 12): whole state in shared memory, one CTA per branch,
// every sweep of every level of the half program, then the gather of S.
template <typename R>
__device__ __forceinline__ void apply_diag_smem(typename Cx2<R>::T *psi, int n, const DiagDev &d,
                                                bool gen) {
  using C = typename Cx2<R>::T;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int ph = diag_phase((uint32_t)i, d, d.zm);
    C w;
    w.x = (R)(c_omega[2 * ph] * d.scale);
    w.y = (R)(c_omega[2 * ph + 1] * d.scale);
    C x = gen ? w : cmul(psi[i], w);
    if (((uint32_t)i & d.pm) != d.pv) x.x = x.y = (R)0;
    psi[i] = x;
  }
}

template <typename R>
__global__ void __launch_bounds__(256) small_kernel(const SmallParams p) {
  using C = typename Cx2<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C *psi = reinterpret_cast<C *>(smem_raw);
  const int n = 1 << p.h;
  const uint64_t b = p.b0 + blockIdx.x;
  int consumed = 0;
  for (int l = 0; l < p.nlevels; ++l) {
    const SmallLevelDev &L = p.levels[l];
    uint32_t child = 0;
    if (l > 0) {
      consumed += L.k;
      child = (uint32_t)((b >> (p.c - consumed)) & ((1ull << L.k) - 1ull));
    }
    for (int s = 0; s < L.nsweeps; ++s) {
      const SmallSweepDev &S = p.sweeps[L.first_sweep + s];
      if (l > 0 && s == 0) {  // the cut CZs of this fork: P_bits (upper) / Z^bits (lower), Eq. 1
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          bool zero = false, neg = false;
          for (int j = 0; j < L.k; ++j) {
            const uint32_t cb = (child >> (L.k - 1 - j)) & 1u;
            const uint32_t ib = ((uint32_t)i >> L.cut_bits[j]) & 1u;
            if ((L.pmask >> j) & 1u)
              zero |= (ib != cb);
            else
              neg ^= (ib & cb) != 0;
          }
          C x = psi[i];
          if (zero) x.x = x.y = (R)0;
          if (neg) {
            x.x = -x.x;
            x.y = -x.y;
          }
          psi[i] = x;
        }
        __syncthreads();
      }
      if (S.gen || S.pre.active) {
        apply_diag_smem<R>(psi, n, S.pre, S.gen != 0);
        __syncthreads();
      }
      for (int g = 0; g < S.ngates; ++g) {
        const int bit = S.bit[g], kind = S.kind[g];
        const uint32_t lowmask = (1u << bit) - 1u;
        for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
          const uint32_t i0 = (((uint32_t)t & ~lowmask) << 1) | ((uint32_t)t & lowmask);
          butterfly(kind, psi[i0], psi[i0 | (1u << bit)]);
        }
        __syncthreads();
      }
      if (S.post.active) {
        apply_diag_smem<R>(psi, n, S.post, false);
        __syncthreads();
      }
    }
    if (l > 0 && L.nsweeps == 0) {  // fork at the last layer: apply it before the gather
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        bool zero = false, neg = false;
        for (int j = 0; j < L.k; ++j) {
          const uint32_t cb = (child >> (L.k - 1 - j)) & 1u;
          const uint32_t ib = ((uint32_t)i >> L.cut_bits[j]) & 1u;
          if ((L.pmask >> j) & 1u)
            zero |= (ib != cb);
          else
            neg ^= (ib & cb) != 0;
        }
        C x = psi[i];
        if (zero) x.x = x.y = (R)0;
        if (neg) {
          x.x = -x.x;
          x.y = -x.y;
        }
        psi[i] = x;
      }
      __syncthreads();
    }
  }
  C *out = reinterpret_cast<C *>(p.out) + (uint64_t)blockIdx.x * (uint64_t)p.nS;
  for (int64_t j = threadIdx.x; j < p.nS; j += blockDim.x) out[j] = psi[p.S[j]];
}

int small_max_h(bool c128) { return 12; }

cudaError_t launch_small(const SmallParams &p, bool c128, uint64_t nb, cudaStream_t s) {
  const size_t smem = ((size_t)1 << p.h) * (c128 ? 16 : 8);
  if (c128) {
    cudaError_t e = cudaFuncSetAttribute(small_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    small_kernel<double><<<(unsigned)nb, 256, smem, s>>>(p);
  } else {
    cudaError_t e = cudaFuncSetAttribute(small_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    small_kernel<float><<<(unsigned)nb, 256, smem, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace qsim
