// Porter-Thomas / Gumbel analyzer (Eq. 7, Fig. 5).
//
// One HBM pass over the block: x = N p (p = fma(re, re, im*im) as the sampler computes it),
// moments sum x and sum x^2 (per-CTA partials, summed in a fixed order => deterministic),
// a shared-memory histogram of z = ln x (Fig. 5) and a 2^20-bin global histogram of
// u = F(z) = 1 - exp(-x) (Eq. 7's CDF, alpha = 1) from which a one-CTA pass brackets the
// Kolmogorov-Smirnov distance.  HBM-bound: 16 B (complex block) or 8 B per entry.
#include <cstdint>

#include "kernels.h"

namespace qsim {

namespace {

struct PtLayout {
  unsigned *uh;   // PT_U_BINS
  unsigned *zh;   // PT_MAX_Z_BINS
  double *part;   // PT_CTAS * 2
  PtResult *res;
};

__host__ __device__ inline PtLayout pt_layout(void *scratch) {
  char *b = (char *)scratch;
  PtLayout L;
  L.uh = (unsigned *)b;
  L.zh = (unsigned *)(b + (size_t)PT_U_BINS * 4);
  L.part = (double *)(b + (size_t)PT_U_BINS * 4 + (size_t)PT_MAX_Z_BINS * 4);
  L.res = (PtResult *)(b + (size_t)PT_U_BINS * 4 + (size_t)PT_MAX_Z_BINS * 4 + (size_t)PT_CTAS * 16);
  return L;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned warp_sum_u(unsigned v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <bool CPLX>
__global__ void __launch_bounds__(256) pt_accumulate_kernel(const void *__restrict__ in, int64_t n, double Nq,
                                                            double z_lo, double zscale, int nb,
                                                            PtLayout L) {
  extern __shared__ unsigned szh[];
  __shared__ double red[2][8];
  for (int k = threadIdx.x; k < nb; k += blockDim.x) szh[k] = 0u;
  __syncthreads();
  double s1 = 0.0, s2 = 0.0;
  unsigned zeros = 0, below = 0, above = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double p;
    if constexpr (CPLX) {
      const double2 a = reinterpret_cast<const double2 *>(in)[i];
      p = fma(a.x, a.x, a.y * a.y);
    } else {
      p = reinterpret_cast<const double *>(in)[i];
    }
    const double x = p * Nq;  // Nq = 2^n: exact
    s1 += x;
    s2 = fma(x, x, s2);
    if (!(x > 0.0)) {
      ++zeros;
      continue;
    }
    const double fb = floor((log(x) - z_lo) * zscale);
    if (fb < 0.0)
      ++below;
    else if (fb >= (double)nb)
      ++above;
    else
      atomicAdd(&szh[(int)fb], 1u);
    const double u = -expm1(-x);  // F(z) = 1 - exp(-e^z), e^z = x
    int ub = (int)(u * (double)PT_U_BINS);
    if (ub >= PT_U_BINS) ub = PT_U_BINS - 1;
    atomicAdd(&L.uh[ub], 1u);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  zeros = warp_sum_u(zeros);
  below = warp_sum_u(below);
  above = warp_sum_u(above);
  if (lane == 0) {
    red[0][w] = s1;
    red[1][w] = s2;
    if (zeros) atomicAdd(&L.res->zeros, (unsigned long long)zeros);
    if (below) atomicAdd(&L.res->below, (unsigned long long)below);
    if (above) atomicAdd(&L.res->above, (unsigned long long)above);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      a += red[0][k];
      b += red[1][k];
    }
    L.part[2 * blockIdx.x] = a;
    L.part[2 * blockIdx.x + 1] = b;
  }
  for (int k = threadIdx.x; k < nb; k += blockDim.x)
    if (szh[k]) atomicAdd(&L.zh[k], szh[k]);
}

// One CTA of 1024 threads: moments from the CTA partials (fixed order), then the KS bracket.
// For bin k = [t_k, t_k+1) of u with C_k entries below it (t_k = k 2^-20, exact):
//   F_emp(t_k-) = C_k / n exactly  =>  ks_lo = max_k |C_k/n - t_k|  <= D
//   F_emp(t) in [C_k/n, C_k+1/n] on the bin  =>  D <= ks_hi = max_k max(C_k+1/n - t_k, t_k+1 - C_k/n)
__global__ void __launch_bounds__(1024) pt_finish_kernel(PtLayout L, int nparts) {
  constexpr int PER = PT_U_BINS / 1024;
  __shared__ unsigned long long scan[1024];
  __shared__ double mx[2][32];
  const int t = threadIdx.x;
  if (t == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < nparts; ++k) {
      a += L.part[2 * k];
      b += L.part[2 * k + 1];
    }
    L.res->s1 = a;
    L.res->s2 = b;
  }
  const unsigned *h = L.uh + (size_t)t * PER;
  unsigned long long mine = 0;
  for (int k = 0; k < PER; ++k) mine += h[k];
  scan[t] = mine;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const unsigned long long v = t >= off ? scan[t - off] : 0ull;
    __syncthreads();
    scan[t] += v;
    __syncthreads();
  }
  const unsigned long long total = scan[1023];
  unsigned long long C = scan[t] - mine;
  double lo = 0.0, hi = 0.0;
  if (total > 0) {
    const double inv = 1.0 / (double)total;
    for (int k = 0; k < PER; ++k) {
      const double tk = (double)(t * PER + k) * (1.0 / PT_U_BINS);
      const double tk1 = (double)(t * PER + k + 1) * (1.0 / PT_U_BINS);
      const double F0 = (double)C * inv;
      C += h[k];
      const double F1 = (double)C * inv;
      lo = fmax(lo, fabs(F0 - tk));
      hi = fmax(hi, fmax(F1 - tk, tk1 - F0));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmax(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((t & 31) == 0) {
    mx[0][t >> 5] = lo;
    mx[1][t >> 5] = hi;
  }
  __syncthreads();
  if (t == 0) {
    for (int k = 1; k < 32; ++k) {
      lo = fmax(lo, mx[0][k]);
      hi = fmax(hi, mx[1][k]);
    }
    L.res->ks_lo = lo;
    L.res->ks_hi = hi;
  }
}

}  // namespace

unsigned *pt_zhist(void *scratch) { return pt_layout(scratch).zh; }
const PtResult *pt_result(void *scratch) { return pt_layout(scratch).res; }

cudaError_t launch_porter_thomas(const void *in, bool complex_in, int64_t n, int n_qubits, double z_lo,
                                 double z_hi, int n_bins, void *scratch, cudaStream_t s) {
  if (n_bins < 1 || n_bins > PT_MAX_Z_BINS || !(z_hi > z_lo)) return cudaErrorInvalidValue;
  const PtLayout L = pt_layout(scratch);
  cudaError_t e = cudaMemsetAsync(L.uh, 0, (size_t)PT_U_BINS * 4 + (size_t)PT_MAX_Z_BINS * 4, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(L.res, 0, sizeof(PtResult), s);
  if (e != cudaSuccess) return e;
  const double Nq = ldexp(1.0, n_qubits);
  const double zscale = (double)n_bins / (z_hi - z_lo);
  const size_t smem = (size_t)n_bins * 4;
  if (complex_in)
    pt_accumulate_kernel<true><<<PT_CTAS, 256, smem, s>>>(in, n, Nq, z_lo, zscale, n_bins, L);
  else
    pt_accumulate_kernel<false><<<PT_CTAS, 256, smem, s>>>(in, n, Nq, z_lo, zscale, n_bins, L);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  pt_finish_kernel<<<1, 1024, 0, s>>>(L, PT_CTAS);
  return cudaGetLastError();
}

}  // namespace qsim
