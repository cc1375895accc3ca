// Device helpers shared by the gate-sweep kernels.
#pragma once

#include <cstdint>

#include "kernels.h"

namespace qsim {

template <typename R>
struct Cx2;
template <>
struct Cx2<float> {
  using T = float2;
  using V = float4;  // 16-byte vector = 2 amplitudes
};
template <>
struct Cx2<double> {
  using T = double2;
  using V = double2;  // 16-byte vector = 1 amplitude
};

// w^k = e^{i k pi / 4}, k = 0..7 (re, im)
static __constant__ double c_omega[16] = {1.0,
                                          0.0,
                                          0.70710678118654752440,
                                          0.70710678118654752440,
                                          0.0,
                                          1.0,
                                          -0.70710678118654752440,
                                          0.70710678118654752440,
                                          -1.0,
                                          0.0,
                                          -0.70710678118654752440,
                                          -0.70710678118654752440,
                                          0.0,
                                          -1.0,
                                          0.70710678118654752440,
                                          -0.70710678118654752440};

// CZ pair term of the fused diagonal mod 2: parity of sum_k popc(i & i>>czd[k] & czm[k]).  The first
// kCzFast distances use static parameter offsets (no dynamic indexing, no extra live registers).
constexpr int kCzFast = 8;
__device__ __forceinline__ int diag_cz(uint32_t i, const DiagDev &d) {
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < kCzFast; ++k)
    if (k < d.ncz) x ^= i & (i >> d.czd[k]) & d.czm[k];
  for (int k = kCzFast; k < d.ncz; ++k) x ^= i & (i >> d.czd[k]) & d.czm[k];
  return __popc(x) & 1;
}

// full phase of the fused diagonal at index i (see DiagDev), zm passed separately
__device__ __forceinline__ int diag_phase(uint32_t i, const DiagDev &d, uint32_t zm) {
  const int ph = d.ph0 + __popc(i & d.t1) + 2 * __popc(i & d.t2) + 4 * (__popc(i & zm) + diag_cz(i, d));
  return ph & 7;
}

// the same without ph0 (the B part of the DiagSplit decomposition)
__device__ __forceinline__ int diag_phase_b(uint32_t i, const DiagDev &d) {
  return __popc(i & d.t1) + 2 * __popc(i & d.t2) + 4 * (__popc(i & d.zm) + diag_cz(i, d));
}

template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
  C r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}

// Butterflies of the factored gates on a register pair (a has the bit clear):
//   SX' = [[1,-i],[-i,1]]: a' = a - i b, b' = b - i a;   SY' = [[1,-1],[1,1]]: a' = a - b, b' = a + b
template <typename C>
__device__ __forceinline__ void butterfly(int kind, C &a, C &b) {
  const C x = a, y = b;
  if (kind == 1) {
    a.x = x.x + y.y;
    a.y = x.y - y.x;
    b.x = y.x + x.y;
    b.y = y.y - x.x;
  } else {
    a.x = x.x - y.x;
    a.y = x.y - y.y;
    b.x = x.x + y.x;
    b.y = x.y + y.y;
  }
}

template <typename R, int NV>
__device__ __forceinline__ void unpack(const typename Cx2<R>::V &x, typename Cx2<R>::T (&v)[NV]) {
  if constexpr (NV == 2) {
    v[0].x = x.x;
    v[0].y = x.y;
    v[1].x = x.z;
    v[1].y = x.w;
  } else {
    v[0].x = x.x;
    v[0].y = x.y;
  }
}

template <typename R, int NV>
__device__ __forceinline__ typename Cx2<R>::V pack(const typename Cx2<R>::T (&v)[NV]) {
  typename Cx2<R>::V x;
  if constexpr (NV == 2) {
    x.x = v[0].x;
    x.y = v[0].y;
    x.z = v[1].x;
    x.w = v[1].y;
  } else {
    x.x = v[0].x;
    x.y = v[0].y;
  }
  return x;
}

}  // namespace qsim
