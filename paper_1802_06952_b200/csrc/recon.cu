// Leaf gather, reconstruction contraction A += U^T L on the FP64 tensor pipe (DMMA),
// |a|^2, prefix tables and the Philox inverse-CDF sampler.
//
// "after sampling the data and performing the tensor product, the results are finally
// added to the resultant vector" (Fig. 1 caption P:175): for sampled
// blocks this is the complex contraction over the branch index b,
//     A[i, j] = sum_b U[b, i] * L[b, j].
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "sweep_common.cuh"

namespace qsim {

template <typename R>
struct CxT;
template <>
struct CxT<float> {
  using T = float2;
};
template <>
struct CxT<double> {
  using T = double2;
};


// ---------------------------------------------------------------- gather
template <typename R>
__global__ void gather_kernel(const typename CxT<R>::T *__restrict__ psi, const uint64_t *__restrict__ S,
                              int64_t n, typename CxT<R>::T *__restrict__ out, DiagDev d, uint64_t lmask,
                              uint64_t gsel, uint64_t xmask) {
  using C = typename CxT<R>::T;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = S[j];
    if ((i & ~lmask) != gsel) {  // another shard's amplitude (distributed half)
      out[j].x = out[j].y = (R)0;
      continue;
    }
    C x = psi[(i ^ xmask) & lmask];
    if (d.active) {
      const uint32_t ii = (uint32_t)i;
      const int ph = diag_phase(ii, d, d.zm);
      const R wr = (R)(c_omega[2 * ph] * d.scale), wi = (R)(c_omega[2 * ph + 1] * d.scale);
      C y;
      y.x = x.x * wr - x.y * wi;
      y.y = x.x * wi + x.y * wr;
      if ((ii & d.pm) != d.pv) y.x = y.y = (R)0;
      x = y;
    }
    out[j] = x;
  }
}

cudaError_t launch_gather(const void *psi, const uint64_t *S, int64_t n, void *out,
                          const DiagDev &pend, bool c128, cudaStream_t s, uint64_t lmask, uint64_t gsel,
                          uint64_t xmask) {
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((n + threads - 1) / threads, 4096);
  if (c128)
    gather_kernel<double><<<blocks, threads, 0, s>>>((const double2 *)psi, S, n, (double2 *)out, pend, lmask, gsel,
                                                     xmask);
  else
    gather_kernel<float><<<blocks, threads, 0, s>>>((const float2 *)psi, S, n, (float2 *)out, pend, lmask, gsel,
                                                    xmask);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- Walsh-Hadamard rows (R-zz)
// With Z^b forks on both endpoints of a block's free cuts, CZ = sum_{a,b} H_ab Z^a (x) Z^b with
// H = [[1, 1], [1, -1]] / 2 per cut, so the lower slice rows are replaced by sum_b H_ab L_b (DESIGN.md
// R-zz): one butterfly pass per branch bit, (a + b) / 2 and (a - b) / 2 (exact scaling).
// up to 8 row bits [b0, b0 + nb) in one pass: a CTA holds 2^nb rows x 16 columns in shared memory
template <typename R>
__global__ void __launch_bounds__(256) wht_rows_smem_kernel(typename CxT<R>::T *__restrict__ A, int b0, int nb,
                                                            int64_t nrows, int64_t ncols) {
  using C = typename CxT<R>::T;
  extern __shared__ __align__(16) unsigned char wraw[];
  C *sh = reinterpret_cast<C *>(wraw);  // [2^nb][16]
  const int64_t ngroups = nrows >> nb;  // row groups: rows r = lo | (q << b0) | (hi << (b0 + nb))
  const int64_t ncb = (ncols + 15) / 16;
  const int64_t blk = blockIdx.x;
  const int64_t grp = blk / ncb, cb = blk - grp * ncb;
  const int64_t lo = grp & ((1ll << b0) - 1), hi = grp >> b0;
  const int R2 = 1 << nb;
  for (int e = threadIdx.x; e < R2 * 16; e += blockDim.x) {
    const int q = e >> 4, c = e & 15;
    const int64_t row = lo | ((int64_t)q << b0) | (hi << (b0 + nb)), col = cb * 16 + c;
    C v{};
    if (col < ncols) v = A[row * ncols + col];
    sh[e] = v;
  }
  __syncthreads();
  for (int bit = 0; bit < nb; ++bit) {
    for (int e = threadIdx.x; e < R2 * 8; e += blockDim.x) {
      const int p = e >> 4, c = e & 15;
      const int q0 = ((p >> bit) << (bit + 1)) | (p & ((1 << bit) - 1)), q1 = q0 | (1 << bit);
      const C a = sh[q0 * 16 + c], b = sh[q1 * 16 + c];
      C s, d;
      s.x = (a.x + b.x) * (R)0.5;
      s.y = (a.y + b.y) * (R)0.5;
      d.x = (a.x - b.x) * (R)0.5;
      d.y = (a.y - b.y) * (R)0.5;
      sh[q0 * 16 + c] = s;
      sh[q1 * 16 + c] = d;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < R2 * 16; e += blockDim.x) {
    const int q = e >> 4, c = e & 15;
    const int64_t row = lo | ((int64_t)q << b0) | (hi << (b0 + nb)), col = cb * 16 + c;
    if (col < ncols) A[row * ncols + col] = sh[e];
  }
}

cudaError_t launch_wht_rows(void *A, bool c128, int m, int64_t ncols, cudaStream_t s) {
  if (m <= 0 || ncols <= 0) return cudaSuccess;
  const int64_t nrows = 1ll << m, ncb = (ncols + 15) / 16;
  for (int b0 = 0; b0 < m; b0 += 8) {  // passes of up to 8 bits (2^8 rows x 16 columns x 16 B = 64 KB)
    const int nb = std::min(8, m - b0);
    const int64_t blocks = (nrows >> nb) * ncb;
    const size_t sm = ((size_t)16 << nb) * (c128 ? 16 : 8);
    if (c128) {
      cudaFuncSetAttribute((const void *)wht_rows_smem_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           65536);
      wht_rows_smem_kernel<double><<<(unsigned)blocks, 256, sm, s>>>((double2 *)A, b0, nb, nrows, ncols);
    } else {
      wht_rows_smem_kernel<float><<<(unsigned)blocks, 256, sm, s>>>((float2 *)A, b0, nb, nrows, ncols);
    }
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- leaves through frames
// G = 0: term k reads psi[x ^ m_k] (scattered); G = 1: m_k indexes a row of the pre-gathered flips,
// g[m_k * n + j] = psi[S[j] ^ flip] (coalesced: one scattered pass per distinct flip, launch_flip_rows)
template <typename R, int G>
__global__ void frame_gather_kernel(const typename CxT<R>::T *__restrict__ psi, const uint64_t *__restrict__ S,
                                    int64_t n, typename CxT<R>::T *__restrict__ out, const DiagDev pend,
                                    const __grid_constant__ FrameBatch b) {
  using C = typename CxT<R>::T;
  const int64_t total = (int64_t)b.nleaf * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    const uint32_t x = (uint32_t)S[j];
    double sr = 0.0, si = 0.0;
    // the terms' scattered reads are issued 8 at a time (independent loads in flight), then summed
    const int k0 = b.off[i], k1 = b.off[i + 1];
    for (int kb = k0; kb < k1; kb += 8) {
      C v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (kb + u < k1)
          v[u] = G ? __ldg(psi + (size_t)b.term[kb + u].m * (size_t)n + j) : __ldg(psi + (x ^ b.term[kb + u].m));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (kb + u >= k1) break;
        const FrameTerm &f = b.term[kb + u];
        const int ph = (f.ph0 + __popc(x & f.t1) + 2 * __popc(x & f.t2) + 4 * __popc(x & f.zm)) & 7;
        const double wr = c_omega[2 * ph] * f.cr - c_omega[2 * ph + 1] * f.ci;
        const double wi = c_omega[2 * ph] * f.ci + c_omega[2 * ph + 1] * f.cr;
        sr += (double)v[u].x * wr - (double)v[u].y * wi;
        si += (double)v[u].x * wi + (double)v[u].y * wr;
      }
    }
    if (pend.active) {
      const int ph = diag_phase(x, pend, pend.zm);
      const double wr = c_omega[2 * ph] * pend.scale, wi = c_omega[2 * ph + 1] * pend.scale;
      const double tr = sr * wr - si * wi, ti = sr * wi + si * wr;
      sr = (x & pend.pm) != pend.pv ? 0.0 : tr;
      si = (x & pend.pm) != pend.pv ? 0.0 : ti;
    }
    C &o = out[(int64_t)b.row[i] * n + j];
    o.x += (R)sr;
    o.y += (R)si;
  }
}

cudaError_t launch_frame_gather(const void *psi, const uint64_t *S, int64_t n, void *out, const FrameBatch &b,
                                const DiagDev &pend, bool c128, cudaStream_t s, bool from_rows) {
  const int64_t total = (int64_t)b.nleaf * n;
  if (total <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (c128) {
    if (from_rows)
      frame_gather_kernel<double, 1><<<blocks, 256, 0, s>>>((const double2 *)psi, S, n, (double2 *)out, pend, b);
    else
      frame_gather_kernel<double, 0><<<blocks, 256, 0, s>>>((const double2 *)psi, S, n, (double2 *)out, pend, b);
  } else {
    if (from_rows)
      frame_gather_kernel<float, 1><<<blocks, 256, 0, s>>>((const float2 *)psi, S, n, (float2 *)out, pend, b);
    else
      frame_gather_kernel<float, 0><<<blocks, 256, 0, s>>>((const float2 *)psi, S, n, (float2 *)out, pend, b);
  }
  return cudaGetLastError();
}

template <typename R>
__global__ void flip_rows_kernel(const typename CxT<R>::T *__restrict__ psi, const uint64_t *__restrict__ S, int64_t n,
                                 const uint64_t *__restrict__ flips, int64_t nf, typename CxT<R>::T *__restrict__ g) {
  const int64_t total = nf * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    g[e] = __ldg(psi + (S[j] ^ flips[i]));
  }
}

cudaError_t launch_flip_rows(const void *psi, const uint64_t *S, int64_t n, const uint64_t *flips, int64_t nf, void *g,
                             bool c128, cudaStream_t s) {
  const int64_t total = nf * n;
  if (total <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
  if (c128)
    flip_rows_kernel<double><<<blocks, 256, 0, s>>>((const double2 *)psi, S, n, flips, nf, (double2 *)g);
  else
    flip_rows_kernel<float><<<blocks, 256, 0, s>>>((const float2 *)psi, S, n, flips, nf, (float2 *)g);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- sparse row combination (frame basis)
// out[r][j] = sum_{e in [off[r], off[r+1])} coef[e] * in[src[e]][j]  (complex, fp64 sums, ctx-precision rows)
template <typename R>
__global__ void __launch_bounds__(256) combine_rows_kernel(const typename CxT<R>::T *__restrict__ in, int64_t n,
                                                           const uint32_t *__restrict__ off,
                                                           const uint32_t *__restrict__ src,
                                                           const double2 *__restrict__ coef,
                                                           typename CxT<R>::T *__restrict__ out) {
  using C = typename CxT<R>::T;
  const int64_t r = blockIdx.y;
  const uint32_t e0 = off[r], e1 = off[r + 1];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double sr = 0.0, si = 0.0;
    for (uint32_t e = e0; e < e1; ++e) {
      const C v = in[(int64_t)src[e] * n + j];
      const double2 c = coef[e];
      sr += c.x * (double)v.x - c.y * (double)v.y;
      si += c.x * (double)v.y + c.y * (double)v.x;
    }
    C o;
    o.x = (R)sr;
    o.y = (R)si;
    out[r * n + j] = o;
  }
}

cudaError_t launch_combine_rows(const void *in, int64_t n, const uint32_t *off, const uint32_t *src, const void *coef,
                                int64_t nrows, void *out, bool c128, cudaStream_t s) {
  if (nrows <= 0 || n <= 0) return cudaSuccess;
  for (int64_t r0 = 0; r0 < nrows; r0 += 65535) {  // grid.y <= 65535
    const int64_t nr = std::min<int64_t>(65535, nrows - r0);
    dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 16), (unsigned)nr);
    if (c128)
      combine_rows_kernel<double><<<grid, 256, 0, s>>>((const double2 *)in, n, off + r0, src, (const double2 *)coef,
                                                       (double2 *)out + r0 * n);
    else
      combine_rows_kernel<float><<<grid, 256, 0, s>>>((const float2 *)in, n, off + r0, src, (const double2 *)coef,
                                                      (float2 *)out + r0 * n);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- node-batched leaves
template <typename R>
__global__ void gather_nodes_kernel(const typename CxT<R>::T *__restrict__ psi, uint64_t stride, int shift,
                                    int64_t nnodes, const uint64_t *__restrict__ S, int64_t n,
                                    typename CxT<R>::T *__restrict__ out, const __grid_constant__ ForkDev f,
                                    const DiagDev d, const uint32_t *__restrict__ rowmap) {
  using C = typename CxT<R>::T;
  const int64_t total = nnodes * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = e / n;
    const int64_t jj = e - node * n;
    const uint64_t x = S[jj];
    C v = psi[(uint64_t)(node >> shift) * stride + x];
    if (d.active) {
      const uint32_t ii = (uint32_t)x;
      const int ph = diag_phase(ii, d, d.zm);
      const R wr = (R)(c_omega[2 * ph] * d.scale), wi = (R)(c_omega[2 * ph + 1] * d.scale);
      C y;
      y.x = v.x * wr - v.y * wi;
      y.y = v.x * wi + v.y * wr;
      if ((ii & d.pm) != d.pv) y.x = y.y = (R)0;
      v = y;
    }
    bool zero = false, neg = false;
    for (int j = 0; j < f.n; ++j) {
      const uint64_t cb = ((uint64_t)node >> (f.n - 1 - j)) & 1u, xb = (x >> f.bit[j]) & 1u;
      if ((f.pmask >> j) & 1u)
        zero |= xb != cb;
      else
        neg ^= (xb & cb) != 0;
    }
    if (zero) v.x = v.y = (R)0;
    if (neg) {
      v.x = -v.x;
      v.y = -v.y;
    }
    out[(rowmap ? (int64_t)rowmap[node] : node) * n + jj] = v;
  }
}

cudaError_t launch_gather_nodes(const void *psi, uint64_t stride, int shift, int64_t nnodes, const uint64_t *S,
                                int64_t n, void *out, const ForkDev &fork, bool c128, cudaStream_t s,
                                const DiagDev *pend, const uint32_t *rowmap) {
  const int64_t total = nnodes * n;
  if (total <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  DiagDev d;
  std::memset(&d, 0, sizeof(d));
  if (pend) d = *pend;
  if (c128)
    gather_nodes_kernel<double><<<blocks, 256, 0, s>>>((const double2 *)psi, stride, shift, nnodes, S, n,
                                                       (double2 *)out, fork, d, rowmap);
  else
    gather_nodes_kernel<float><<<blocks, 256, 0, s>>>((const float2 *)psi, stride, shift, nnodes, S, n,
                                                      (float2 *)out, fork, d, rowmap);
  return cudaGetLastError();
}

__global__ void rowmap_kernel(uint32_t *__restrict__ out, int64_t n, const __grid_constant__ RowMapDev rm) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r = rm.base;
    for (int t = 0; t < rm.nbits; ++t) r |= (uint32_t)((e >> t) & 1) << rm.pos[t];
    out[e] = r;
  }
}

cudaError_t launch_rowmap(uint32_t *out, int64_t n, const RowMapDev &rm, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  rowmap_kernel<<<blocks, 256, 0, s>>>(out, n, rm);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- lazy last layer
// 2^min(k,5) lanes per sampled index x (a warp holds 32 >> min(k,5) indices, so layers with few
// targets do not idle most lanes): the lanes of an index split the 2^k input combinations y, each
// term is w^{ph(x,y)} pre(y) psi[y] with ph = 6 popc((x^y) & SX) + 4 popc(~x & y & SY) (the
// factored matrices SX' = [[1,-i],[-i,1]], SY' = [[1,-1],[1,1]]); segment sum, then post(x).
template <typename R>
__global__ void __launch_bounds__(256) gather_layer_kernel(const typename CxT<R>::T *__restrict__ psi,
                                                           const uint64_t *__restrict__ S, int64_t n,
                                                           typename CxT<R>::T *__restrict__ out,
                                                           const __grid_constant__ LazyLayer ll) {
  using C = typename CxT<R>::T;
  const int lane = threadIdx.x & 31;
  const int sb = ll.k < 5 ? ll.k : 5;  // log2 lanes per index
  const int sub = lane & ((1 << sb) - 1);
  const int64_t j = ((((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) << (5 - sb)) + (lane >> sb);
  const bool valid = j < n;
  bool own = false;
  uint32_t x = 0;
  int64_t jo = j;  // output index
  if (valid) {
    int64_t jj = j;
    if (ll.node_stride) {  // node-batched leaves
      const int64_t node = j / ll.nper;
      jj = j - node * ll.nper;
      psi += (uint64_t)node * ll.node_stride;
      if (ll.rowmap) jo = (int64_t)ll.rowmap[node] * ll.nper + jj;
    }
    const uint64_t xs = S[jj];
    own = (xs & ~ll.lmask) == ll.gsel;  // else another shard's index (distributed half)
    x = (uint32_t)xs;
  }
  const uint32_t base = x & ~ll.tmask;
  const uint32_t nterm = own ? (1u << ll.k) : 0u;
  R sr = 0, si = 0;
  for (uint32_t m = sub; m < nterm; m += (1u << sb)) {
    uint32_t y = base;
#pragma unroll 4
    for (int t = 0; t < ll.k; ++t) y |= ((m >> t) & 1u) << ll.bit[t];
    C v = psi[(y ^ (uint32_t)ll.xmask) & (uint32_t)ll.lmask];
    int ph = 6 * __popc((x ^ y) & ll.sxmask) + 4 * __popc(~x & y & ll.symask);
    if (ll.pre.active) {
      ph += diag_phase(y, ll.pre, ll.pre.zm);
      if ((y & ll.pre.pm) != ll.pre.pv) v.x = v.y = (R)0;
    }
    ph &= 7;
    const R wr = (R)c_omega[2 * ph], wi = (R)c_omega[2 * ph + 1];
    sr += v.x * wr - v.y * wi;
    si += v.x * wi + v.y * wr;
  }
  for (int o = (1 << sb) >> 1; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    si += __shfl_xor_sync(0xffffffffu, si, o);
  }
  if (sub == 0 && valid) {
    if (!own) {
      out[jo].x = out[jo].y = (R)0;
      return;
    }
    const double pre_scale = ll.pre.active ? ll.pre.scale : 1.0;
    const int ph = diag_phase(x, ll.post, ll.post.zm);
    const double sc = ll.post.scale * pre_scale;
    const R wr = (R)(c_omega[2 * ph] * sc), wi = (R)(c_omega[2 * ph + 1] * sc);
    C o;
    o.x = sr * wr - si * wi;
    o.y = sr * wi + si * wr;
    if ((x & ll.post.pm) != ll.post.pv) o.x = o.y = (R)0;
    out[jo] = o;
  }
}

cudaError_t launch_gather_layer(const void *psi, const uint64_t *S, int64_t n, void *out, const LazyLayer &ll,
                                bool c128, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int sb = ll.k < 5 ? ll.k : 5;
  const int64_t warps = (n + (32 >> sb) - 1) / (32 >> sb);
  const int64_t blocks = (warps * 32 + 255) / 256;
  if (c128)
    gather_layer_kernel<double><<<(unsigned)blocks, 256, 0, s>>>((const double2 *)psi, S, n, (double2 *)out, ll);
  else
    gather_layer_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float2 *)psi, S, n, (float2 *)out, ll);
  return cudaGetLastError();
}

__global__ void cone_kernel(const uint64_t *__restrict__ S, int64_t n, const __grid_constant__ LazyLayer ll,
                            uint64_t *__restrict__ cone) {
  const int64_t per = 1ll << ll.k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * per; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e >> ll.k;
    const uint32_t m = (uint32_t)(e & (per - 1));
    uint32_t z = (uint32_t)S[j] & ~ll.tmask;
    for (int t = 0; t < ll.k; ++t) z |= ((m >> t) & 1u) << ll.bit[t];
    cone[e] = z;
  }
}

cudaError_t launch_cone_indices(const uint64_t *S, int64_t n, const LazyLayer &ll, uint64_t *cone, cudaStream_t s) {
  const int64_t tot = n << ll.k;
  const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 16);
  cone_kernel<<<blocks, 256, 0, s>>>(S, n, ll, cone);
  return cudaGetLastError();
}

// layer d from the compact cone values V[j * 2^k + m] (same warp-per-output scheme)
template <typename R>
__global__ void __launch_bounds__(256) gather_layer_compact_kernel(const typename CxT<R>::T *__restrict__ V,
                                                                   const uint64_t *__restrict__ S, int64_t n,
                                                                   typename CxT<R>::T *__restrict__ out,
                                                                   const __grid_constant__ LazyLayer ll) {
  using C = typename CxT<R>::T;
  // 2^min(k,5) lanes per output (as gather_layer_kernel): a stage with few targets keeps every lane busy
  const int lane = threadIdx.x & 31;
  const int sb = ll.k < 5 ? ll.k : 5;
  const int sub = lane & ((1 << sb) - 1);
  const int64_t j = ((((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) << (5 - sb)) + (lane >> sb);
  const bool valid = j < n;
  int64_t jo = j;
  bool own = false;
  uint32_t x = 0;
  if (valid) {
    const int64_t jj = ll.node_stride ? j % ll.nper : j;  // node-batched: V, out are [node][nper]
    if (ll.node_stride && ll.rowmap) jo = (int64_t)ll.rowmap[j / ll.nper] * ll.nper + jj;
    own = (S[jj] & ~ll.lmask) == ll.gsel;  // else another shard's index
    x = (uint32_t)S[jj];
  }
  const uint32_t base = x & ~ll.tmask;
  const uint32_t nterm = own ? (1u << ll.k) : 0u;
  const C *Vj = V + ((size_t)(valid ? j : 0) << ll.k);
  R sr = 0, si = 0;
  for (uint32_t m = sub; m < nterm; m += (1u << sb)) {
    uint32_t y = base;
    for (int t = 0; t < ll.k; ++t) y |= ((m >> t) & 1u) << ll.bit[t];
    C v = Vj[m];
    int ph = 6 * __popc((x ^ y) & ll.sxmask) + 4 * __popc(~x & y & ll.symask);
    if (ll.pre.active) {
      ph += diag_phase(y, ll.pre, ll.pre.zm);
      if ((y & ll.pre.pm) != ll.pre.pv) v.x = v.y = (R)0;
    }
    ph &= 7;
    const R wr = (R)c_omega[2 * ph], wi = (R)c_omega[2 * ph + 1];
    sr += v.x * wr - v.y * wi;
    si += v.x * wi + v.y * wr;
  }
  for (int o = (1 << sb) >> 1; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    si += __shfl_xor_sync(0xffffffffu, si, o);
  }
  if (sub == 0 && valid) {
    if (!own) {
      out[jo].x = out[jo].y = (R)0;
      return;
    }
    const double pre_scale = ll.pre.active ? ll.pre.scale : 1.0;
    const int ph = diag_phase(x, ll.post, ll.post.zm);
    const double sc = ll.post.scale * pre_scale;
    const R wr = (R)(c_omega[2 * ph] * sc), wi = (R)(c_omega[2 * ph + 1] * sc);
    C o;
    o.x = sr * wr - si * wi;
    o.y = sr * wi + si * wr;
    if ((x & ll.post.pm) != ll.post.pv) o.x = o.y = (R)0;
    out[jo] = o;
  }
}

cudaError_t launch_gather_layer_compact(const void *V, const uint64_t *S, int64_t n, void *out, const LazyLayer &ll,
                                        bool c128, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int sb = ll.k < 5 ? ll.k : 5;
  const int64_t warps = (n + (32 >> sb) - 1) / (32 >> sb);
  const int64_t blocks = (warps * 32 + 255) / 256;
  if (c128)
    gather_layer_compact_kernel<double>
        <<<(unsigned)blocks, 256, 0, s>>>((const double2 *)V, S, n, (double2 *)out, ll);
  else
    gather_layer_compact_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float2 *)V, S, n, (float2 *)out, ll);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- branch GEMM (DMMA)
// CTA tile 64 x 64 (M x N), K step 16, 8 warps as 2 (M) x 4 (N), warp tile 32 x 16 =
// 4 x 2 m8n8k4 FP64 MMAs.  Complex product with 4 real MMAs per tile and K-step:
//   Re += Ur Lr + (-Ui) Li,   Im += Ur Li + Ui Lr   (fp64 accumulate for both precisions)
constexpr int GB_M = 64, GB_N = 64, GB_K = 16, GB_PAD = 8;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <typename R>
__global__ void __launch_bounds__(256) branch_gemm_kernel(const typename CxT<R>::T *__restrict__ U,
                                                          const typename CxT<R>::T *__restrict__ L,
                                                          int64_t K, int64_t M, int64_t N,
                                                          double *__restrict__ A, int64_t sU, int64_t sA,
                                                          int64_t N2) {
  using C = typename CxT<R>::T;
  U += (int64_t)blockIdx.z * sU;  // batch z: its own U and A (multi-part contraction), L shared
  A += (int64_t)blockIdx.z * sA;
  __shared__ double sUr[GB_K][GB_M + GB_PAD], sUi[GB_K][GB_M + GB_PAD];
  __shared__ double sLr[GB_K][GB_N + GB_PAD], sLi[GB_K][GB_N + GB_PAD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int64_t m0 = (int64_t)blockIdx.y * GB_M, n0 = (int64_t)blockIdx.x * GB_N;

  double accr[4][2][2], acci[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) accr[a][b][0] = accr[a][b][1] = acci[a][b][0] = acci[a][b][1] = 0.0;

  // each thread moves 4 elements of the U tile and 4 of the L tile per K step;
  // the next step is fetched into registers while the current one is multiplied
  C ru[4], rl[4];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + q * 256;  // 0..1023 = 16 x 64
      const int kk = e >> 6, mm = e & 63;
      const int64_t k = k0 + kk;
      C u{}, l{};
      if (k < K) {
        if (m0 + mm < M) u = U[k * M + m0 + mm];
        if (n0 + mm < N) l = L[k * N + n0 + mm];
      }
      ru[q] = u;
      rl[q] = l;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + q * 256;
      const int kk = e >> 6, mm = e & 63;
      sUr[kk][mm] = (double)ru[q].x;
      sUi[kk][mm] = (double)ru[q].y;
      sLr[kk][mm] = (double)rl[q].x;
      sLi[kk][mm] = (double)rl[q].y;
    }
  };

  const int64_t nk = (K + GB_K - 1) / GB_K;
  fetch(0);
  stash();
  __syncthreads();
  for (int64_t kb = 0; kb < nk; ++kb) {
    if (kb + 1 < nk) fetch((kb + 1) * GB_K);
#pragma unroll
    for (int ks = 0; ks < GB_K; ks += 4) {
      const int kr = ks + (lane & 3);
      double ar[4], ai[4], br[2], bi[2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int mm = wm * 32 + mt * 8 + (lane >> 2);
        ar[mt] = sUr[kr][mm];
        ai[mt] = sUi[kr][mm];
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int nn = wn * 16 + nt * 8 + (lane >> 2);
        br[nt] = sLr[kr][nn];
        bi[nt] = sLi[kr][nn];
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          dmma(accr[mt][nt], ar[mt], br[nt]);
          dmma(accr[mt][nt], -ai[mt], bi[nt]);
          dmma(acci[mt][nt], ar[mt], bi[nt]);
          dmma(acci[mt][nt], ai[mt], br[nt]);
        }
    }
    __syncthreads();
    if (kb + 1 < nk) {
      stash();
      __syncthreads();
    }
  }
  // epilogue: D fragment row = lane >> 2, cols (lane & 3) * 2 + {0, 1}
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int64_t m = m0 + wm * 32 + mt * 8 + (lane >> 2);
        const int64_t n = n0 + wn * 16 + nt * 8 + (lane & 3) * 2 + c;
        if (m < M && n < N) {
          // N2 > 0: n = (n1, n2) with n2 < N2 and the output is laid out [n1][m][n2]
          const int64_t o = N2 > 0 ? (n / N2) * (M * N2) + m * N2 + (n % N2) : m * N + n;
          double *a = A + 2 * o;
          a[0] += accr[mt][nt][c];
          a[1] += acci[mt][nt][c];
        }
      }
}

// ---------------------------------------------------------------- branch GEMM, 3M form (DMMA)
// The reconstruction contraction A += U^T L with complex entries as three real products (Gauss):
//   T1 = Ur Lr, T2 = Ui Li, T3 = (Ur + Ui)(Lr + Li);  Re A += T1 - T2,  Im A += T3 - T1 - T2
// (3 DMMAs per complex fragment product instead of 4).  CTA tile 64 x 64, K step 16, 8 warps as
// 2 (M) x 4 (N) with 32 x 16 warp tiles of m8n8k4 FP64 MMAs; operands stream through a 3-stage
// cp.async ring of interleaved complex tiles [k][m] (row stride padded so that the fragment loads are
// bank-conflict free: 66 double2 / 68 float2); tiles are visited in bands of 16 tile rows so that the
// CTAs in flight share their U and L panels in L2.
constexpr int G3_BAND = 16;
// row stride (elements) of a [k][m] tile of width W: 16-byte (double2) fragment loads are conflict free
// when the stride is 2 mod 8 (in 16-byte units), 8-byte (float2) ones when it is 4 mod 16
template <typename R, int W>
__host__ __device__ constexpr int g3_stride() { return sizeof(R) == 8 ? W + 2 : W + 4; }
template <typename R, int TM, int TN, int G3_K, int G3_ST>
constexpr size_t g3_smem() {
  return (size_t)G3_ST * G3_K * (g3_stride<R, TM>() + g3_stride<R, TN>()) * sizeof(typename CxT<R>::T);
}

template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void *dst, const void *src, bool ok) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const int n = ok ? BYTES : 0;
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}

// CTA tile TM x TN, 8 warps of (MT x 8) x (NT x 8) fragments, MINB CTAs per SM, K step G3_K, G3_ST stages
// FULL: M, N, K are multiples of the tile (no bounds checks; per-thread source pointers advance by k).
// (Forming the 3M sums once per element into real planes of the stage instead of per fragment was
// measured slower, 27.3 vs 29.2 TF/s executed: profiles/r02/r02x_gemm_configs.txt.)
template <typename R, int TM, int TN, int MT, int NT, int MINB, int G3_K, int G3_ST, bool FULL>
__global__ void __launch_bounds__(256, MINB) branch_gemm3m_kernel(const typename CxT<R>::T *__restrict__ U,
                                                                  const typename CxT<R>::T *__restrict__ L,
                                                                  int64_t K, int64_t M, int64_t N,
                                                                  double *__restrict__ A, int tiles_m, int tiles_n) {
  using C = typename CxT<R>::T;
  constexpr int SU = g3_stride<R, TM>(), SL = g3_stride<R, TN>();
  constexpr int WN = TN / (NT * 8), WM = TM / (MT * 8);
  static_assert(WM * WN == 8, "8 warps");
  extern __shared__ __align__(16) unsigned char g3_raw[];
  C *sU = reinterpret_cast<C *>(g3_raw);
  C *sL = sU + G3_ST * G3_K * SU;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  // banded tile order
  const int pid = blockIdx.x, per_band = G3_BAND * tiles_n, band = pid / per_band;
  const int first = band * G3_BAND, rows = min(tiles_m - first, G3_BAND), in = pid - band * per_band;
  const int64_t m0 = (int64_t)(first + in % rows) * TM, n0 = (int64_t)(in / rows) * TN;

  constexpr int QU = G3_K * TM / 256, QL = G3_K * TN / 256;
  const C *gU[QU], *gL[QL];
  int oU[QU], oL[QL];
#pragma unroll
  for (int q = 0; q < QU; ++q) {
    const int e = tid + q * 256, kk = e / TM, mm = e % TM;
    gU[q] = U + (int64_t)kk * M + m0 + mm;
    oU[q] = kk * SU + mm;
  }
#pragma unroll
  for (int q = 0; q < QL; ++q) {
    const int e = tid + q * 256, kk = e / TN, nn = e % TN;
    gL[q] = L + (int64_t)kk * N + n0 + nn;
    oL[q] = kk * SL + nn;
  }
  auto load = [&](int st, int64_t k0) {
    if constexpr (FULL) {
      const int64_t du = k0 * M, dl = k0 * N;
#pragma unroll
      for (int q = 0; q < QU; ++q) cp_async_zfill<sizeof(C)>(sU + st * G3_K * SU + oU[q], gU[q] + du, true);
#pragma unroll
      for (int q = 0; q < QL; ++q) cp_async_zfill<sizeof(C)>(sL + st * G3_K * SL + oL[q], gL[q] + dl, true);
      return;
    }
#pragma unroll
    for (int q = 0; q < G3_K * TM / 256; ++q) {
      const int e = tid + q * 256;
      const int kk = e / TM, mm = e % TM;
      const int64_t k = k0 + kk;
      const bool ok = k < K && m0 + mm < M;
      cp_async_zfill<sizeof(C)>(sU + (st * G3_K + kk) * SU + mm, ok ? (const void *)(U + k * M + m0 + mm) : (const void *)U, ok);
    }
#pragma unroll
    for (int q = 0; q < G3_K * TN / 256; ++q) {
      const int e = tid + q * 256;
      const int kk = e / TN, nn = e % TN;
      const int64_t k = k0 + kk;
      const bool ok = k < K && n0 + nn < N;
      cp_async_zfill<sizeof(C)>(sL + (st * G3_K + kk) * SL + nn, ok ? (const void *)(L + k * N + n0 + nn) : (const void *)L, ok);
    }
  };
  double t1[MT][NT][2], t2[MT][NT][2], t3[MT][NT][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) t1[a][b][c] = t2[a][b][c] = t3[a][b][c] = 0.0;

  const int64_t nk = (K + G3_K - 1) / G3_K;
#pragma unroll
  for (int s = 0; s < G3_ST - 1; ++s) {
    if (s < nk) load(s, (int64_t)s * G3_K);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t kb = 0; kb < nk; ++kb) {
    asm volatile("cp.async.wait_group %0;" ::"n"(G3_ST - 2) : "memory");
    const int st = (int)(kb % G3_ST);
    __syncthreads();
    if (kb + G3_ST - 1 < nk) load((int)((kb + G3_ST - 1) % G3_ST), (kb + G3_ST - 1) * G3_K);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const C *tu = sU + st * G3_K * SU, *tl = sL + st * G3_K * SL;
#pragma unroll
    for (int ks = 0; ks < G3_K; ks += 4) {
      const int kr = ks + (lane & 3);
      double ar[MT], ai[MT], as[MT], br[NT], bi[NT], bs[NT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int mm = wm * MT * 8 + mt * 8 + (lane >> 2);
        const C u = tu[kr * SU + mm];
        ar[mt] = (double)u.x;
        ai[mt] = (double)u.y;
        as[mt] = ar[mt] + ai[mt];
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int nn = wn * NT * 8 + nt * 8 + (lane >> 2);
        const C l = tl[kr * SL + nn];
        br[nt] = (double)l.x;
        bi[nt] = (double)l.y;
        bs[nt] = br[nt] + bi[nt];
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma(t1[mt][nt], ar[mt], br[nt]);
          dmma(t2[mt][nt], ai[mt], bi[nt]);
          dmma(t3[mt][nt], as[mt], bs[nt]);
        }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int64_t m = m0 + wm * MT * 8 + mt * 8 + (lane >> 2);
        const int64_t n = n0 + wn * NT * 8 + nt * 8 + (lane & 3) * 2 + c;
        if (m < M && n < N) {
          double *a = A + 2 * (m * N + n);
          a[0] += t1[mt][nt][c] - t2[mt][nt][c];
          a[1] += t3[mt][nt][c] - t1[mt][nt][c] - t2[mt][nt][c];
        }
      }
}

template <typename R, int TM, int TN, int MT, int NT, int MINB, int KS = 16, int ST = 3>
static cudaError_t launch_gemm3m(const void *U, const void *L, int64_t K, int64_t M, int64_t N, double *A,
                                 cudaStream_t s) {
  static bool attr = false;
  const bool full = M % TM == 0 && N % TN == 0 && K % KS == 0;
  auto *fn = full ? branch_gemm3m_kernel<R, TM, TN, MT, NT, MINB, KS, ST, true>
                  : branch_gemm3m_kernel<R, TM, TN, MT, NT, MINB, KS, ST, false>;
  constexpr size_t smem = g3_smem<R, TM, TN, KS, ST>();
  if (!attr) {
    for (auto *f : {branch_gemm3m_kernel<R, TM, TN, MT, NT, MINB, KS, ST, true>,
                    branch_gemm3m_kernel<R, TM, TN, MT, NT, MINB, KS, ST, false>}) {
      cudaError_t e = cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  const int tm = (int)((M + TM - 1) / TM), tn = (int)((N + TN - 1) / TN);
  using C = typename CxT<R>::T;
  fn<<<(unsigned)((int64_t)tm * tn), 256, smem, s>>>((const C *)U, (const C *)L, K, M, N, A, tm, tn);
  return cudaGetLastError();
}

template <typename R>
static cudaError_t launch_gemm3m_cfg(const void *U, const void *L, int64_t K, int64_t M, int64_t N, double *A,
                                     cudaStream_t s) {
  // QSIM_GEMM_CFG (A/B): 1 (default) = 64x64 tile, 32x16 warps, 1 CTA/SM, K step 32, 3 stages (202 KB of
  // shared memory); 0 = K step 16 (whole C5 job: 2.21 vs 2.28 s of GEMM)
  static const int cfg = std::getenv("QSIM_GEMM_CFG") ? std::atoi(std::getenv("QSIM_GEMM_CFG")) : 1;
  // (measured on B200, K = 16384, M = N = 8192: 64x32 / 32x64 tiles with 2 CTAs per SM 28.3 / 28.2, K steps of
  // 32 with 2 / 3 stages 29.3 / 29.4, 4 stages of 16 29.0, this one 29.0 TF/s executed: the DMMA pipe, not
  // occupancy or the pipeline depth, is the limit; profiles/r02/r02x_gemm_configs.txt)
  if (cfg == 1) return launch_gemm3m<R, 64, 64, 4, 2, 1, 32, 3>(U, L, K, M, N, A, s);
  return launch_gemm3m<R, 64, 64, 4, 2, 1>(U, L, K, M, N, A, s);
}

cudaError_t launch_branch_gemm(const void *U, const void *L, int64_t K, int64_t M, int64_t N,
                               double *A, bool c128, cudaStream_t s) {
  if (K <= 0 || M <= 0 || N <= 0) return cudaSuccess;
  // A/B: QSIM_GEMM=4m runs the four-product kernel below.  (An m16n8k8 form was measured equal: ptxas
  // splits it into the same DMMA.8x8x4 instructions, the only FP64 MMA of sm_100a.)
  static const bool four = std::getenv("QSIM_GEMM") && std::string(std::getenv("QSIM_GEMM")) == "4m";
  if (!four) return c128 ? launch_gemm3m_cfg<double>(U, L, K, M, N, A, s) : launch_gemm3m_cfg<float>(U, L, K, M, N, A, s);
  dim3 grid((unsigned)((N + GB_N - 1) / GB_N), (unsigned)((M + GB_M - 1) / GB_M));
  if (c128)
    branch_gemm_kernel<double><<<grid, 256, 0, s>>>((const double2 *)U, (const double2 *)L, K, M, N, A, 0, 0, 0);
  else
    branch_gemm_kernel<float><<<grid, 256, 0, s>>>((const float2 *)U, (const float2 *)L, K, M, N, A, 0, 0, 0);
  return cudaGetLastError();
}

cudaError_t launch_branch_gemm_batched(const double *U, const double *L, int64_t K, int64_t M, int64_t N,
                                       double *A, int64_t batch, cudaStream_t s, int64_t N2) {
  if (K <= 0 || M <= 0 || N <= 0 || batch <= 0) return cudaSuccess;
  const int64_t sU = 2 * K * M, sA = 2 * M * N;  // in doubles
  for (int64_t z0 = 0; z0 < batch; z0 += 65535) {
    dim3 grid((unsigned)((N + GB_N - 1) / GB_N), (unsigned)((M + GB_M - 1) / GB_M),
              (unsigned)std::min<int64_t>(65535, batch - z0));
    branch_gemm_kernel<double><<<grid, 256, 0, s>>>((const double2 *)(U + z0 * sU), (const double2 *)L, K, M, N,
                                                    A + z0 * sA, sU / 2, sA, N2);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- multi-part slices
// dst[rowmap[r], :] = src[r, :] as double2 (row r of a part's leaf slice in tree order goes to
// its (beta_{k-1}, beta_k) row of the contraction operand)
template <typename R>
__global__ void permute_rows_kernel(const typename CxT<R>::T *__restrict__ src, const uint32_t *__restrict__ rowmap,
                                    int64_t nrows, int64_t ncols, double2 *__restrict__ dst) {
  const int64_t total = nrows * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ncols, j = e - r * ncols;
    const auto v = src[e];
    dst[(int64_t)rowmap[r] * ncols + j] = make_double2((double)v.x, (double)v.y);
  }
}

cudaError_t launch_permute_rows(const void *src, bool c128, const uint32_t *rowmap, int64_t nrows, int64_t ncols,
                                double *dst, cudaStream_t s) {
  const int64_t total = nrows * ncols;
  if (total <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (c128)
    permute_rows_kernel<double><<<blocks, 256, 0, s>>>((const double2 *)src, rowmap, nrows, ncols, (double2 *)dst);
  else
    permute_rows_kernel<float><<<blocks, 256, 0, s>>>((const float2 *)src, rowmap, nrows, ncols, (double2 *)dst);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- probabilities
__global__ void abs2_kernel(const double2 *__restrict__ A, int64_t n, double *__restrict__ p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = A[i];
    p[i] = fma(a.x, a.x, a.y * a.y);
  }
}

cudaError_t launch_abs2(const double *A, int64_t n, double *p, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  abs2_kernel<<<blocks, 256, 0, s>>>((const double2 *)A, n, p);
  return cudaGetLastError();
}

// One warp per 32 rows: 32 x 32 tiles are staged through shared memory so that global
// access is coalesced while every lane scans its own row strictly left to right.
// A != nullptr: p = fma(re, re, im*im) of the complex block A is computed here and written to p
// (|a|^2 fused into the scan's load: one pass over the block instead of two)
__global__ void __launch_bounds__(128) row_scan_kernel(const double *__restrict__ pin, const double2 *__restrict__ A,
                                                       double *__restrict__ pout, int64_t M, int64_t N,
                                                       double *__restrict__ Cp, double *__restrict__ r) {
  __shared__ double tile[4][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t row0 = ((int64_t)blockIdx.x * 4 + w) * 32;
  if (row0 >= M) return;
  double run = 0.0;
  const int64_t myrow = row0 + lane;
  for (int64_t j0 = 0; j0 < N; j0 += 32) {
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t row = row0 + rr, col = j0 + lane;
      double v = 0.0;
      if (row < M && col < N) {
        if (A) {
          const double2 a = A[row * N + col];
          v = fma(a.x, a.x, a.y * a.y);
          pout[row * N + col] = v;
        } else {
          v = pin[row * N + col];
        }
      }
      tile[w][rr][lane] = v;
    }
    __syncwarp();
    const int lim = (int)std::min<int64_t>(32, N - j0);
    for (int jj = 0; jj < lim; ++jj) {
      run = run + tile[w][lane][jj];
      tile[w][lane][jj] = run;
    }
    __syncwarp();
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t row = row0 + rr, col = j0 + lane;
      if (row < M && col < N) Cp[row * N + col] = tile[w][rr][lane];
    }
    __syncwarp();
  }
  if (myrow < M) r[myrow] = run;
}

cudaError_t launch_row_scan(const double *p, int64_t M, int64_t N, double *Cp, double *r,
                            cudaStream_t s) {
  const int blocks = (int)((M + 127) / 128);
  row_scan_kernel<<<blocks, 128, 0, s>>>(p, nullptr, nullptr, M, N, Cp, r);
  return cudaGetLastError();
}

cudaError_t launch_row_scan_abs2(const double *A, int64_t M, int64_t N, double *p, double *Cp, double *r,
                                 cudaStream_t s) {
  const int blocks = (int)((M + 127) / 128);
  row_scan_kernel<<<blocks, 128, 0, s>>>(nullptr, (const double2 *)A, p, M, N, Cp, r);
  return cudaGetLastError();
}

// R = inclusive prefix of r in strictly sequential order (run = run + r[i], i = 0, 1, ...: the
// oracle's definition, bit-exact): one warp, 32 values per coalesced load, the running sum passed
// through the lanes by shuffles (the additions stay one dependent chain in index order).
__global__ void row_prefix_kernel(const double *__restrict__ r, int64_t M, double *__restrict__ R,
                                  double *__restrict__ W) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  double run = 0.0;
  double next = lane < M ? r[lane] : 0.0;
  for (int64_t base = 0; base < M; base += 32) {
    const double v = next;
    next = base + 32 + lane < M ? r[base + 32 + lane] : 0.0;  // prefetch the next chunk
    const int lim = (int)(M - base < 32 ? M - base : 32);
    double mine = 0.0;
    for (int j = 0; j < lim; ++j) {
      run = run + __shfl_sync(0xffffffffu, v, j);
      if (lane == j) mine = run;
    }
    if (lane < lim) R[base + lane] = mine;
  }
  if (lane == 0) *W = run;
}

cudaError_t launch_row_prefix(const double *r, int64_t M, double *R, double *W, cudaStream_t s) {
  row_prefix_kernel<<<1, 32, 0, s>>>(r, M, R, W);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- Philox4x32-10 sampler
__device__ __forceinline__ void philox10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// first index in [0, n) with a[idx] > t (n if none); a non-decreasing
__device__ __forceinline__ int64_t upper_bound(const double *a, int64_t n, double t) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] > t)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

// Rows [row0, row0 + nrows) of p / C are held here (the whole block on one GPU; a row shard with
// several): a draw whose row another rank owns writes 0 (the ranks' outputs are summed).
__global__ void draws_kernel(const double *__restrict__ p, const double *__restrict__ Cp,
                             const double *__restrict__ r, const double *__restrict__ R,
                             const double *__restrict__ Wp, int64_t M, int64_t N,
                             const uint64_t *__restrict__ Su, const uint64_t *__restrict__ Sl,
                             uint32_t hl, uint64_t seed, int64_t n, uint64_t *__restrict__ out,
                             int64_t row0, int64_t nrows) {
  const double W = *Wp;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c[4] = {(uint32_t)k, (uint32_t)((uint64_t)k >> 32), 0u, 0u};
    philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t v = ((uint64_t)c[1] << 32) | c[0];
    const double u = (double)(v >> 11) * 0x1.0p-53;
    const double t = u * W;
    int64_t i = upper_bound(R, M, t);
    if (i >= M) {
      i = M - 1;
      while (i > 0 && !(r[i] > 0.0)) --i;
    }
    if (i < row0 || i >= row0 + nrows) {
      out[k] = 0;
      continue;
    }
    const double t2 = t - (i > 0 ? R[i - 1] : 0.0);
    const int64_t il = i - row0;
    int64_t j = upper_bound(Cp + il * N, N, t2);
    if (j >= N) {
      j = N - 1;
      while (j > 0 && !(p[il * N + j] > 0.0)) --j;
    }
    out[k] = (Su[i] << hl) | Sl[j];
  }
}

cudaError_t launch_draws(const double *p, const double *Cp, const double *r, const double *R,
                         const double *W, int64_t M, int64_t N, const uint64_t *Su,
                         const uint64_t *Sl, uint32_t hl, uint64_t seed, int64_t n,
                         uint64_t *out, cudaStream_t s, int64_t row0, int64_t nrows) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  draws_kernel<<<blocks, 256, 0, s>>>(p, Cp, r, R, W, M, N, Su, Sl, hl, seed, n, out, row0, nrows < 0 ? M : nrows);
  return cudaGetLastError();
}

__global__ void cast_kernel(const double *__restrict__ A, int64_t n, float *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)A[i];
}

cudaError_t launch_cast_c128_to_c64(const double *A, int64_t n, float *out, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  cast_kernel<<<blocks, 256, 0, s>>>(A, n, out);
  return cudaGetLastError();
}

}  // namespace qsim
