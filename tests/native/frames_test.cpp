// Dense-matrix check of the Pauli-frame algebra (tests/test_frames_native.py).
#include "program.h"
#include <algorithm>
#include <complex>
#include <cstdio>
#include <random>
#include <vector>
using namespace qsim;
using cd = std::complex<double>;
const int n = 5, N = 1 << n;
typedef std::vector<cd> Mat;  // N x N row-major
Mat mul(const Mat &a, const Mat &b) { Mat c(N * N); for (int i = 0; i < N; ++i) for (int k = 0; k < N; ++k) if (a[i*N+k] != 0.0) for (int j = 0; j < N; ++j) c[i*N+j] += a[i*N+k] * b[k*N+j]; return c; }
Mat diag(const Diag &d) { Mat m(N * N); for (int x = 0; x < N; ++x) { double ang = M_PI / 4 * d.phase(x); cd v = std::polar(d.scale(), ang); if ((x & d.pm) != d.pv || d.allzero) v = 0; m[x*N+x] = v; } return m; }
Mat flip(uint64_t msk) { Mat m(N * N); for (int x = 0; x < N; ++x) m[x*N + (x ^ (int)msk)] = 1; return m; }
Mat gate(int t, int kind) { Mat m(N * N); for (int x = 0; x < N; ++x) { int y = x ^ (1 << t); m[x*N+x] += 1; int bx = (x >> t) & 1, by = (y >> t) & 1; cd v; if (kind == 1) v = cd(0, -1); else v = (bx == 0 ? -1.0 : 1.0); /* -iY: [[0,-1],[1,0]] row bx col by */ if (kind == 2) v = (bx == 0 && by == 1) ? -1.0 : 1.0; m[x*N+y] += v; } return m; }
int main_dense() {
  std::mt19937_64 r(7);
  int ok = 0, tot = 0, bad = 0;
  for (int it = 0; it < 3000; ++it) {
    Sweep sw;
    std::vector<int> bits = {0,1,2,3,4};
    std::shuffle(bits.begin(), bits.end(), r);
    int ng = 1 + r() % 3;
    for (int k = 0; k < ng; ++k) sw.gates.push_back(Gate1{(uint8_t)bits[k], (uint8_t)(1 + r() % 2)});
    for (int k = 0; k < 3; ++k) { sw.post.add_T(r() % n); sw.pre.add_T(r() % n); }
    for (int k = 0; k < 2; ++k) { int a = r() % n, b = r() % n; if (a != b) sw.post.add_cz(a, b); }
    if (r() % 2) { int a = r() % n, b = r() % n; if (a != b) sw.pre.add_cz(a, b); }
    sw.post.nhalf = ng; sw.post.ph0 = r() % 8;
    Diag phi; uint64_t m = r() % N;
    for (int k = 0; k < 2; ++k) phi.add_Z(r() % n);
    if (r() % 3 == 0) phi.add_T(r() % n);
    phi.ph0 = r() % 8;
    Diag p2 = phi; uint64_t m2 = m;
    Mat G = diag(sw.pre);
    for (auto &g : sw.gates) G = mul(gate(g.bit, g.kind), G);
    G = mul(diag(sw.post), G);
    ++tot;
    if (!frame_through(sw, p2, m2)) continue;
    ++ok;
    Mat L = mul(G, mul(diag(phi), flip(m))), R = mul(mul(diag(p2), flip(m2)), G);
    double e = 0; for (int i = 0; i < N * N; ++i) e = std::max(e, std::abs(L[i] - R[i]));
    if (e > 1e-12) ++bad;
  }
  // compose / inverse
  for (int it = 0; it < 500; ++it) {
    Diag a, b; uint64_t ma = r() % N, mb = r() % N;
    for (int k = 0; k < 3; ++k) { a.add_T(r() % n); b.add_T(r() % n); }
    int x0 = r() % n, x1 = (x0 + 1) % n; a.add_cz(x0, x1);
    Diag c; uint64_t mc; frame_compose(b, mb, a, ma, c, mc);
    Mat L = mul(mul(diag(b), flip(mb)), mul(diag(a), flip(ma))), R = mul(diag(c), flip(mc));
    Diag ai; frame_inverse(a, ma, ai);
    Mat I = mul(mul(diag(ai), flip(ma)), mul(diag(a), flip(ma)));
    double e = 0; for (int i = 0; i < N * N; ++i) { e = std::max(e, std::abs(L[i] - R[i])); e = std::max(e, std::abs(I[i] - (i % (N + 1) == 0 ? 1.0 : 0.0))); }
    if (e > 1e-12) ++bad;
  }
  printf("propagated %d of %d, bad %d\n", ok, tot, bad);
  return bad != 0;
}
// ---- LinFrame vs Diag frames
int lin_check() {
  std::mt19937_64 r(11);
  int bad = 0, okc = 0;
  auto same = [&](const LinFrame &a, const Diag &d, uint64_t m) {
    if (a.m != m) return false;
    Diag ad = a.diag();
    for (int x = 0; x < 64; ++x) if (ad.phase(x) != d.phase(x)) return false;
    return true;
  };
  for (int it = 0; it < 5000; ++it) {
    const int nb = 6;
    Sweep sw;
    std::vector<int> bits = {0,1,2,3,4,5};
    std::shuffle(bits.begin(), bits.end(), r);
    int ng = 1 + r() % 3;
    for (int k = 0; k < ng; ++k) sw.gates.push_back(Gate1{(uint8_t)bits[k], (uint8_t)(1 + r() % 2)});
    for (int k = 0; k < 3; ++k) { sw.post.add_T(r() % nb); sw.pre.add_T(r() % nb); }
    for (int k = 0; k < 3; ++k) { int a = r() % nb, b = r() % nb; if (a != b) sw.post.add_cz(a, b); }
    if (r() % 2) { int a = r() % nb, b = r() % nb; if (a != b) sw.pre.add_cz(a, b); }
    LinFrame f; f.m = r() % 64; f.ph0 = r() % 8;
    for (int k = 0; k < 3; ++k) { int a = r() % nb; int c = r() % 8; if (r() % 2) c &= 4; f.add_counts((c & 1) ? 1ull << a : 0, (c & 2) ? 1ull << a : 0, (c & 4) ? 1ull << a : 0); }
    Diag d = f.diag(); uint64_t m = f.m;
    LinFrame g = f;
    bool a1 = lin_through(sw, g), a2 = frame_through(sw, d, m);
    if (a1 != a2) { ++bad; continue; }
    if (a1) { ++okc; if (!same(g, d, m)) ++bad; }
    // compose / inverse
    LinFrame h; h.m = r() % 64; h.ph0 = r() % 8; h.add_counts(r() % 64, r() % 64, r() % 64);
    Diag hc; uint64_t hm; frame_compose(h.diag(), h.m, f.diag(), f.m, hc, hm);
    if (!same(lin_compose(h, f), hc, hm)) ++bad;
    Diag fi; frame_inverse(f.diag(), f.m, fi);
    if (!same(lin_inverse(f), fi, f.m)) ++bad;
  }
  printf("lin: propagated %d, bad %d\n", okc, bad);
  return bad;
}
int main2() { return lin_check(); }

// ---- expansion of a breaking frame into a sum of frames
int expand_check() {
  std::mt19937_64 r(5);
  int bad = 0, multi = 0;
  for (int it = 0; it < 3000; ++it) {
    Sweep sw;
    std::vector<int> bits = {0, 1, 2, 3, 4};
    std::shuffle(bits.begin(), bits.end(), r);
    int ng = 1 + r() % 3;
    for (int k = 0; k < ng; ++k) sw.gates.push_back(Gate1{(uint8_t)bits[k], (uint8_t)(1 + r() % 2)});
    for (int k = 0; k < 3; ++k) { sw.post.add_T(r() % n); sw.pre.add_T(r() % n); }
    for (int k = 0; k < 2; ++k) { int a = r() % n, b = r() % n; if (a != b) sw.post.add_cz(a, b); }
    sw.post.nhalf = ng;
    LinFrame f; f.m = r() % N; f.ph0 = r() % 8;
    for (int k = 0; k < 3; ++k) { int a = r() % n; f.add_counts(1ull << a, (r() % 2) ? 1ull << a : 0, 0); }
    LinFrame out[64]; double coef[128];
    const int nt = lin_expand_through(sw, f, 64, out, coef);
    if (nt == 0) continue;
    if (nt > 1) ++multi;
    Mat G = diag(sw.pre);
    for (auto &g : sw.gates) G = mul(gate(g.bit, g.kind), G);
    G = mul(diag(sw.post), G);
    Mat L = mul(G, mul(diag(f.diag()), flip(f.m)));
    Mat R(N * N);
    for (int i = 0; i < nt; ++i) {
      Mat T = mul(mul(diag(out[i].diag()), flip(out[i].m)), G);
      for (int e = 0; e < N * N; ++e) R[e] += cd(coef[2 * i], coef[2 * i + 1]) * T[e];
    }
    double e = 0; for (int i = 0; i < N * N; ++i) e = std::max(e, std::abs(L[i] - R[i]));
    if (e > 1e-12) ++bad;
  }
  printf("expand: %d multi-term, bad %d\n", multi, bad);
  return bad;
}
int main() { int a = main_dense(); int b = lin_check(); int c = expand_check(); return a || b || c; }
