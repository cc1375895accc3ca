// Front end: validation, cut list, branch-tree levels and fused sweeps (see program.h).
#include "program.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <set>
#include <sstream>

namespace qsim {

int Diag::count(int bit) const {
  return (int)((t1 >> bit) & 1u) + 2 * (int)((t2 >> bit) & 1u) + 4 * (int)((zm >> bit) & 1u);
}

void Diag::set_count(int bit, int c) {
  c &= 7;
  const uint64_t m = 1ull << bit;
  t1 = (t1 & ~m) | ((c & 1) ? m : 0ull);
  t2 = (t2 & ~m) | ((c & 2) ? m : 0ull);
  zm = (zm & ~m) | ((c & 4) ? m : 0ull);
}

void Diag::add_proj(int bit, int value) {
  const uint64_t m = 1ull << bit;
  const uint64_t v = value ? m : 0ull;
  if ((pm & m) && ((pv & m) != v)) allzero = true;  // P0 P1 = 0
  pm |= m;
  pv = (pv & ~m) | v;
}

void Diag::add_cz(int b0, int b1) {
  const int lo = std::min(b0, b1), d = std::abs(b0 - b1);
  cz[d] ^= 1ull << lo;  // CZ^2 = I
}

int Diag::phase(uint64_t i) const {
  int ph = ph0 + __builtin_popcountll(i & t1) + 2 * __builtin_popcountll(i & t2) + 4 * __builtin_popcountll(i & zm);
  for (int d = 1; d < 64; ++d) ph += 4 * __builtin_popcountll(i & (i >> d) & cz[d]);
  return ph & 7;
}

Diag Diag::merge(const Diag &a, const Diag &b) {
  Diag d = a;
  for (int bit = 0; bit < 64; ++bit) {
    const int cb = b.count(bit);
    if (cb) d.set_count(bit, d.count(bit) + cb);
  }
  for (int k = 0; k < 64; ++k) d.cz[k] ^= b.cz[k];  // CZ^2 = I
  const uint64_t overlap = a.pm & b.pm;
  if ((a.pv & overlap) != (b.pv & overlap)) d.allzero = true;
  d.pm = a.pm | b.pm;
  d.pv = (a.pv & a.pm) | (b.pv & b.pm);
  d.ph0 = (a.ph0 + b.ph0) & 7;
  d.nhalf = a.nhalf + b.nhalf;
  d.allzero = d.allzero || a.allzero || b.allzero;
  return d;
}

Diag Diag::restrict_low(int hl, uint64_t g) const {
  if (hl >= 64) return *this;
  const uint64_t low = (1ull << hl) - 1ull;
  Diag r = *this;
  for (int bit = hl; bit < 64; ++bit) {  // counts on fixed bits: constants
    const int c = count(bit);
    if (!c) continue;
    if ((g >> bit) & 1u) r.ph0 = (r.ph0 + c) & 7;
    r.set_count(bit, 0);
  }
  const uint64_t fixed_pm = pm & ~low;  // projectors on fixed bits: pass or zero
  if ((g & fixed_pm) != (pv & fixed_pm)) r.allzero = true;
  r.pm &= low;
  r.pv &= low;
  for (int d = 1; d < 64; ++d) {
    uint64_t keep = 0;
    for (int a = 0; a + d < 64; ++a) {
      if (!((cz[d] >> a) & 1u)) continue;
      const int b = a + d;
      const bool fa = a >= hl, fb = b >= hl;
      if (!fa && !fb) {
        keep |= 1ull << a;
      } else if (fa && fb) {
        if (((g >> a) & 1u) && ((g >> b) & 1u)) r.ph0 = (r.ph0 + 4) & 7;
      } else if (fb && ((g >> b) & 1u)) {  // CZ with a set fixed bit: Z on the other one
        r.set_count(a, r.count(a) + 4);
      }
    }
    r.cz[d] = keep;
  }
  return r;
}

bool Diag::below(int bits) const {
  const uint64_t hi = bits >= 64 ? 0ull : ~((1ull << bits) - 1ull);
  if ((t1 | t2 | zm | pm | pv) & hi) return false;
  for (int d = 1; d < 64; ++d)
    if (cz[d] && (d >= bits || (cz[d] & hi))) return false;
  return true;
}

double Diag::scale() const {
  // 2^(-nhalf/2) for either sign of nhalf (inverse diagonals carry nhalf < 0)
  const int q = nhalf >= 0 ? nhalf / 2 : -((1 - nhalf) / 2);  // floor(nhalf / 2)
  double s = std::ldexp(1.0, -q);
  if (nhalf - 2 * q) s *= 0.70710678118654752440;
  return s;
}

Diag Diag::shift(uint64_t m) const {
  Diag r = *this;
  if (!m) return r;
  r.pv = (pv ^ (m & pm)) & pm;
  for (uint64_t rest = m; rest; rest &= rest - 1) {
    const int a = __builtin_ctzll(rest);
    const int c = count(a);
    r.ph0 = (r.ph0 + c) & 7;
    r.set_count(a, (8 - c) & 7);
  }
  for (int d = 1; d < 64; ++d) {
    for (uint64_t rest = cz[d]; rest; rest &= rest - 1) {
      const int a = __builtin_ctzll(rest);
      const int b = a + d;
      const bool fa = (m >> a) & 1u, fb = (m >> b) & 1u;
      if (fa) r.set_count(b, r.count(b) + 4);
      if (fb) r.set_count(a, r.count(a) + 4);
      if (fa && fb) r.ph0 = (r.ph0 + 4) & 7;
    }
  }
  return r;
}

Diag Diag::inverse() const {
  if (pm || allzero) throw std::invalid_argument("inverse of a projector");
  Diag r = *this;
  for (int a = 0; a < 64; ++a) {
    const int c = count(a);
    if (c) r.set_count(a, (8 - c) & 7);
  }
  r.ph0 = (8 - ph0) & 7;
  r.nhalf = -nhalf;
  return r;
}

Diag Diag::phase_only() const {
  Diag r = *this;
  r.pm = r.pv = 0;
  r.nhalf = 0;
  r.allzero = false;
  return r;
}

// ---------------------------------------------------------------- Pauli frames (program.h)
static bool cz_touches(const Diag &d, int t) {
  for (int k = 1; k < 64; ++k) {
    if (!d.cz[k]) continue;
    if ((d.cz[k] >> t) & 1u) return true;
    if (t >= k && ((d.cz[k] >> (t - k)) & 1u)) return true;
  }
  return false;
}

// phi * D / D^m (phases only; a projector of D must not meet m)
static bool frame_ratio(Diag &phi, const Diag &D, uint64_t m) {
  if (!m) return true;
  if (D.pm & m) return false;
  const Diag p = D.phase_only();
  phi = Diag::merge(phi, Diag::merge(p, p.shift(m).inverse()));
  return true;
}

bool frame_through(const Sweep &sw, Diag &phi0, uint64_t &m0) {
  Diag phi = phi0;
  uint64_t m = m0;
  if (sw.gen) return false;
  if (!frame_ratio(phi, sw.pre, m)) return false;
  for (const Gate1 &g : sw.gates) {
    const int t = g.bit;
    if ((phi.pm >> t) & 1u) return false;
    const int c = phi.count(t);
    if ((c & 3) || cz_touches(phi, t)) return false;
    // D X^f with D = diag(1, w^c) on t, conjugated by I - iX (kind 1) / I - iY (kind 2):
    // I - iX: X -> X, Z -> -Y = w^2 Z X, Z X (= iY) -> iZ = w^2 Z
    // I - iY: X -> -Z = w^4 Z, Z -> X, Z X -> Z X
    const int f = (int)((m >> t) & 1u), z = c >> 2;
    int nf = f, nz = z, ph = 0;
    if (g.kind == 1) {
      if (!f && z) nf = 1, nz = 1, ph = 2;
      else if (f && z) nf = 0, nz = 1, ph = 2;
    } else {
      if (f && !z) nf = 0, nz = 1, ph = 4;
      else if (!f && z) nf = 1, nz = 0;
    }
    phi.set_count(t, 4 * nz);
    phi.ph0 = (phi.ph0 + ph) & 7;
    m = (m & ~(1ull << t)) | ((uint64_t)nf << t);
  }
  if (!frame_ratio(phi, sw.post, m)) return false;
  phi0 = phi;
  m0 = m;
  return true;
}

void frame_compose(const Diag &phi2, uint64_t m2, const Diag &phi1, uint64_t m1, Diag &phi, uint64_t &m) {
  phi = Diag::merge(phi2, phi1.shift(m2));
  m = m1 ^ m2;
}

void frame_inverse(const Diag &phi, uint64_t m, Diag &inv_phi) { inv_phi = phi.inverse().shift(m); }

// ---------------------------------------------------------------- linear frames (program.h)
void LinFrame::add_counts(uint64_t b1, uint64_t b2, uint64_t b4) {
  const uint64_t s0 = t1 ^ b1, c0 = t1 & b1;
  const uint64_t s1 = t2 ^ b2 ^ c0, c1 = (t2 & b2) | (c0 & (t2 ^ b2));
  t1 = s0;
  t2 = s1;
  zm = zm ^ b4 ^ c1;
}

void LinFrame::negate(uint64_t mask) {  // -c = ~c + 1 (mod 8)
  t1 ^= mask;
  t2 ^= mask;
  zm ^= mask;
  add_counts(mask, 0, 0);
}

LinFrame LinFrame::shift(uint64_t s) const {
  LinFrame r = *this;
  if (!s) return r;
  r.ph0 = (ph0 + __builtin_popcountll(s & t1) + 2 * __builtin_popcountll(s & t2) + 4 * __builtin_popcountll(s & zm)) & 7;
  r.negate(s);
  return r;
}

Diag LinFrame::diag() const {
  Diag d;
  d.t1 = t1;
  d.t2 = t2;
  d.zm = zm;
  d.ph0 = ph0 & 7;
  return d;
}

// phi * D / D^m, D a program diagonal (phases; a projector must not meet m)
static bool lin_ratio(LinFrame &f, const Diag &D) {
  const uint64_t m = f.m;
  if (!m) return true;
  if (D.pm & m) return false;
  // bits a in m: weight 2 c_a(D), ph0 -= c_a(D)
  uint64_t b2 = 0, b4 = 0;
  int ph = 0;
  for (uint64_t r = m & (D.t1 | D.t2 | D.zm); r; r &= r - 1) {
    const int a = __builtin_ctzll(r), ca = D.count(a);
    ph -= ca;
    if (ca & 1) b2 ^= 1ull << a;  // 2 c_a mod 8: bit plane 2 gets c_a bit 0, plane 4 gets c_a bit 1
    if (ca & 2) b4 ^= 1ull << a;
  }
  uint64_t z4 = 0;
  for (int d = 1; d < 64; ++d)
    for (uint64_t r = D.cz[d]; r; r &= r - 1) {
      const int a = __builtin_ctzll(r), b = a + d;
      const bool fa = (m >> a) & 1u, fb = (m >> b) & 1u;
      if (fa) z4 ^= 1ull << b;
      if (fb) z4 ^= 1ull << a;
      if (fa && fb) ph += 4;
    }
  f.add_counts(0, b2, b4);
  f.add_counts(0, 0, z4);
  f.ph0 = ((f.ph0 + ph) % 8 + 8) % 8;
  return true;
}

// the gate stage of a frame move (every target's count must be 0 or 4)
static bool lin_gates(const Sweep &sw, LinFrame &f) {
  for (const Gate1 &g : sw.gates) {
    const int t = g.bit;
    const int c = f.count(t);
    if (c & 3) return false;
    const int fl = (int)((f.m >> t) & 1u), z = c >> 2;
    int nf = fl, nz = z, ph = 0;
    if (g.kind == 1) {  // I - iX: X -> X, Z -> w^2 Z X, Z X -> w^2 Z
      if (!fl && z) nf = 1, nz = 1, ph = 2;
      else if (fl && z) nf = 0, nz = 1, ph = 2;
    } else {  // I - iY: X -> w^4 Z, Z -> X, Z X -> Z X
      if (fl && !z) nf = 0, nz = 1, ph = 4;
      else if (!fl && z) nf = 1, nz = 0;
    }
    const uint64_t bit = 1ull << t;
    f.zm = nz ? (f.zm | bit) : (f.zm & ~bit);
    f.ph0 = (f.ph0 + ph) & 7;
    f.m = nf ? (f.m | bit) : (f.m & ~bit);
  }
  return true;
}

bool lin_through(const Sweep &sw, LinFrame &f0) {
  if (sw.gen) return false;
  LinFrame f = f0;
  if (!lin_ratio(f, sw.pre) || !lin_gates(sw, f) || !lin_ratio(f, sw.post)) return false;
  f0 = f;
  return true;
}

int lin_expand_through(const Sweep &sw, const LinFrame &f0, int max_terms, LinFrame *out, double *coef) {
  if (sw.gen) return 0;
  LinFrame f = f0;
  if (!lin_ratio(f, sw.pre)) return 0;
  int bad[32], nb = 0;
  for (const Gate1 &g : sw.gates)
    if (f.count(g.bit) & 3) {
      if (nb == 32) return 0;
      bad[nb++] = g.bit;
    }
  if (nb > 30 || (1ll << nb) > max_terms) return 0;
  const int n = 1 << nb;
  for (int s = 0; s < n; ++s) {
    LinFrame h = f;
    double cr = 1.0, ci = 0.0;
    for (int i = 0; i < nb; ++i) {
      const int t = bad[i], cnt = h.count(t);
      static const double r2 = 0.70710678118654752440;
      static const double W[8][2] = {{1, 0}, {r2, r2}, {0, 1}, {-r2, r2}, {-1, 0}, {-r2, -r2}, {0, -1}, {r2, -r2}};
      const double wr = W[cnt & 7][0], wi = W[cnt & 7][1];
      const bool z = (s >> i) & 1;
      const double xr = z ? 0.5 * (1.0 - wr) : 0.5 * (1.0 + wr), xi = z ? -0.5 * wi : 0.5 * wi;
      const double nr = cr * xr - ci * xi, ni = cr * xi + ci * xr;
      cr = nr;
      ci = ni;
      const uint64_t bit = 1ull << t;
      h.t1 &= ~bit;
      h.t2 &= ~bit;
      h.zm = z ? (h.zm | bit) : (h.zm & ~bit);
    }
    if (!lin_gates(sw, h) || !lin_ratio(h, sw.post)) return 0;
    out[s] = h;
    coef[2 * s] = cr;
    coef[2 * s + 1] = ci;
  }
  return n;
}

LinFrame lin_compose(const LinFrame &f2, const LinFrame &f1) {
  LinFrame r = f1.shift(f2.m);
  r.add_counts(f2.t1, f2.t2, f2.zm);
  r.ph0 = (r.ph0 + f2.ph0) & 7;
  r.m = f1.m ^ f2.m;
  return r;
}

LinFrame lin_inverse(const LinFrame &f) {
  LinFrame r = f;
  r.negate(~0ull);
  r.ph0 = (8 - f.ph0) & 7;
  r = r.shift(f.m);
  r.m = f.m;
  return r;
}

Diag HalfProgram::fork_diag(int level, uint64_t child) const {
  Diag d;
  if (level <= 0) return d;
  const Level &L = levels[level];
  for (int j = 0; j < L.k; ++j) {
    const int bit = (int)((child >> (L.k - 1 - j)) & 1u);
    if ((L.pmask >> j) & 1u)
      d.add_proj(L.cut_bits[j], bit);
    else if (bit)
      d.add_Z(L.cut_bits[j]);
  }
  return d;
}

size_t HalfProgram::total_sweeps() const {
  size_t s = 0;
  for (auto &l : levels) s += l.sweeps.size();
  return s;
}

static bool neighbours(uint32_t a, uint32_t b, uint32_t cols) {
  const uint32_t ra = a / cols, ca = a % cols, rb = b / cols, cb = b % cols;
  if (ra == rb) return (ca + 1 == cb) || (cb + 1 == ca);
  if (ca == cb) return (ra + 1 == rb) || (rb + 1 == ra);
  return false;
}

std::string build_circuit(uint32_t rows, uint32_t cols, uint32_t depth, const qsim_gate *gates,
                          size_t n_gates, uint32_t cut_row, const uint32_t *cut_layers,
                          size_t n_cut_layers, Circuit &out) {
  std::ostringstream err;
  if (rows < 2 || cols < 1) return "grid must have rows >= 2 and cols >= 1";
  // 72 qubits: the paper's largest grids (Table 1, 36-qubit halves sharded over ranks)
  if ((uint64_t)rows * cols > 72) return "at most 72 qubits";
  if (depth > 100000) return "depth too large";
  if (cut_row == 0) cut_row = rows / 2;
  if (cut_row < 1 || cut_row >= rows) return "cut_row must be in [1, rows)";
  Circuit c;
  c.rows = rows;
  c.cols = cols;
  c.depth = depth;
  c.cut_row = cut_row;
  c.n = rows * cols;
  c.h_u = cut_row * cols;
  c.h_l = c.n - c.h_u;
  if (c.h_u > 36 || c.h_l > 36) {  // > 32: only as distributed halves (QSIM_OPT_DISTRIBUTE)
    err << "each half must have at most 36 qubits (h_u=" << c.h_u << ", h_l=" << c.h_l << ")";
    return err.str();
  }
  if (n_gates && !gates) return "gates is NULL";
  std::map<uint32_t, std::set<uint32_t>> used;  // layer -> qubits
  c.gates.assign(gates, gates + n_gates);
  for (size_t i = 0; i < n_gates; ++i) {
    const qsim_gate &g = gates[i];
    if (g.layer < 1 || g.layer > depth) {
      err << "gate " << i << ": layer " << g.layer << " outside 1.." << depth;
      return err.str();
    }
    if (g.kind < QSIM_SX || g.kind > QSIM_CZ) {
      err << "gate " << i << ": unknown kind " << g.kind;
      return err.str();
    }
    if (g.q0 >= c.n) {
      err << "gate " << i << ": qubit " << g.q0 << " >= n = " << c.n;
      return err.str();
    }
    auto &u = used[g.layer];
    if (g.kind == QSIM_CZ) {
      if (g.q1 >= c.n || g.q1 == g.q0) {
        err << "gate " << i << ": bad CZ partner " << g.q1;
        return err.str();
      }
      if (!neighbours(g.q0, g.q1, cols)) {
        err << "gate " << i << ": CZ(" << g.q0 << "," << g.q1 << ") is not a grid edge";
        return err.str();
      }
      if (u.count(g.q0) || u.count(g.q1)) {
        err << "gate " << i << ": qubit used twice in layer " << g.layer << " (P:285)";
        return err.str();
      }
      u.insert(g.q0);
      u.insert(g.q1);
      const bool a_up = g.q0 < c.h_u, b_up = g.q1 < c.h_u;
      if (a_up != b_up) {
        qsim_cut cut;
        cut.layer = g.layer;
        cut.q_upper = a_up ? g.q0 : g.q1;
        cut.q_lower = a_up ? g.q1 : g.q0;
        c.cuts.push_back(cut);
      }
    } else {
      if (g.q1 != QSIM_NO_QUBIT) {
        err << "gate " << i << ": single-qubit gate with q1 != QSIM_NO_QUBIT";
        return err.str();
      }
      if (u.count(g.q0)) {
        err << "gate " << i << ": qubit used twice in layer " << g.layer << " (P:285)";
        return err.str();
      }
      u.insert(g.q0);
    }
  }
  std::sort(c.cuts.begin(), c.cuts.end(), [](const qsim_cut &a, const qsim_cut &b) {
    return a.layer != b.layer ? a.layer < b.layer : a.q_upper < b.q_upper;
  });
  for (auto &cut : c.cuts) {
    if (c.fork_layers.empty() || c.fork_layers.back() != (int)cut.layer) {
      c.fork_layers.push_back((int)cut.layer);
      c.fork_k.push_back(0);
    }
    c.fork_k.back()++;
  }
  if (cut_layers) {
    std::set<uint32_t> given(cut_layers, cut_layers + n_cut_layers);
    std::set<uint32_t> derived;
    for (int l : c.fork_layers) derived.insert((uint32_t)l);
    if (given != derived) {
      err << "cut_layers disagree with the cut CZs of the circuit (derived:";
      for (auto l : derived) err << " " << l;
      err << ")";
      return err.str();
    }
  }
  out = std::move(c);
  return "";
}

namespace {
struct LayerSpec {
  std::vector<Gate1> gates;
  Diag diag;
};
}  // namespace

HalfProgram compile_half(const Circuit &c, bool upper, const std::vector<int> &perm) {
  const int h = (int)(upper ? c.h_u : c.h_l);
  std::vector<int> p = perm;
  if (p.empty())
    for (int b = 0; b < h; ++b) p.push_back(b);
  return compile_half_layers(c, upper, std::vector<std::vector<int>>(c.depth + 2, p), p);
}

std::vector<PartCut> half_cuts(const Circuit &c, bool upper, const std::vector<char> *p_upper) {
  std::vector<PartCut> cuts;
  for (size_t g = 0; g < c.cuts.size(); ++g) {
    const qsim_cut &cut = c.cuts[g];
    const bool pu = p_upper ? (*p_upper)[g] != 0 : true;
    cuts.push_back(PartCut{(int)cut.layer, upper ? cut.q_upper : cut.q_lower, upper ? pu : !pu});
  }
  return cuts;
}

HalfProgram compile_half_layers(const Circuit &c, bool upper, const std::vector<std::vector<int>> &layer_perm,
                                const std::vector<int> &final_perm) {
  return compile_part(c, upper ? 0 : c.h_u, upper ? c.h_u : c.n, upper, half_cuts(c, upper), layer_perm, final_perm);
}

std::vector<int> first_targets(const Circuit &c, const std::vector<PartCut> &cuts) {
  std::vector<int> ft;
  for (const PartCut &cut : cuts) {
    int t = (int)c.depth + 1;
    for (const qsim_gate &g : c.gates)
      if ((g.kind == QSIM_SX || g.kind == QSIM_SY) && g.q0 == cut.q && (int)g.layer > cut.layer)
        t = std::min(t, (int)g.layer);
    ft.push_back(t);
  }
  return ft;
}

std::vector<int> gate_layers(const Circuit &c, uint32_t lo, uint32_t hi) {
  std::set<int> s;
  for (const qsim_gate &g : c.gates)
    if ((g.kind == QSIM_SX || g.kind == QSIM_SY) && g.q0 >= lo && g.q0 < hi) s.insert((int)g.layer);
  return std::vector<int>(s.begin(), s.end());
}

HalfProgram compile_part(const Circuit &c, uint32_t lo, uint32_t hi, bool upper, const std::vector<PartCut> &cuts,
                         const std::vector<std::vector<int>> &layer_perm, const std::vector<int> &final_perm,
                         const std::vector<int> *apply) {
  HalfProgram hp;
  hp.upper = upper;
  hp.h = (int)(hi - lo);
  hp.hl = hp.h;
  hp.perm = final_perm;
  hp.ncuts = (int)cuts.size();
  // forks: the cuts grouped by the layer at whose input they apply (in cut order inside a group)
  std::vector<int> app(cuts.size());
  for (size_t i = 0; i < cuts.size(); ++i) {
    app[i] = apply ? (*apply)[i] : cuts[i].layer + 1;
    if (app[i] <= cuts[i].layer || app[i] > (int)c.depth + 1) throw std::invalid_argument("fork apply layer");
  }
  std::vector<int> order(cuts.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return app[a] < app[b]; });
  std::vector<int> fork_layers, fork_k;  // fork_layers: apply layer - 1
  for (int i : order) {
    if (fork_layers.empty() || fork_layers.back() != app[i] - 1) {
      fork_layers.push_back(app[i] - 1);
      fork_k.push_back(0);
    }
    fork_k.back()++;
  }
  auto bit_at = [&](uint32_t q, int layer) { return layer_perm[layer][hp.h - 1 - (int)(q - lo)]; };

  std::vector<LayerSpec> layers(c.depth + 1);
  for (const qsim_gate &g : c.gates) {
    LayerSpec &L = layers[g.layer];
    if (g.kind == QSIM_CZ) {
      const bool in0 = g.q0 >= lo && g.q0 < hi, in1 = g.q1 >= lo && g.q1 < hi;
      if (!(in0 && in1)) continue;  // cut CZ (handled as a fork) or the other half
      L.diag.add_cz(bit_at(g.q0, (int)g.layer), bit_at(g.q1, (int)g.layer));
    } else {
      if (!(g.q0 >= lo && g.q0 < hi)) continue;
      const int b = bit_at(g.q0, (int)g.layer);
      if (g.kind == QSIM_T) {
        L.diag.add_T(b);
      } else {
        L.gates.push_back(Gate1{(uint8_t)b, (uint8_t)(g.kind == QSIM_SX ? 1 : 2)});
      }
    }
  }
  for (auto &L : layers) {
    std::sort(L.gates.begin(), L.gates.end(),
              [](const Gate1 &a, const Gate1 &b) { return a.bit < b.bit; });
    // each factored gate carries the global factor w / sqrt2
    L.diag.ph0 = (L.diag.ph0 + (int)L.gates.size()) & 7;
    L.diag.nhalf += (int)L.gates.size();
  }

  const int F = (int)fork_layers.size();
  hp.levels.resize(F + 1);
  int g0 = 0;
  for (int l = 0; l <= F; ++l) {
    Level &lev = hp.levels[l];
    if (l > 0) {
      lev.fork_layer = fork_layers[l - 1];
      lev.k = fork_k[l - 1];
      lev.g0 = order[g0];
      for (int j = 0; j < lev.k; ++j) {
        const PartCut &cut = cuts[order[g0 + j]];
        lev.cut_g.push_back(order[g0 + j]);
        // the fork acts on the child level's input: the layout of its first layer
        lev.cut_bits.push_back(bit_at(cut.q, std::min(lev.fork_layer + 1, (int)c.depth + 1)));
        if (cut.proj) lev.pmask |= 1u << j;
      }
      g0 += lev.k;
    }
    const int first = (l == 0) ? 1 : fork_layers[l - 1] + 1;
    const int last = (l < F) ? fork_layers[l] : (int)c.depth;
    Diag pending;
    if (l == 0) pending.nhalf = hp.h;  // H^{(x)h}|0> = 2^{-h/2} everywhere (layer 0)
    for (int t = first; t <= last; ++t) {
      const LayerSpec &L = layers[t];
      if (!L.gates.empty()) {
        Sweep s;
        s.gates = L.gates;
        s.pre = pending;
        s.post = L.diag;
        s.gen = (l == 0 && lev.sweeps.empty());
        s.first_layer = s.last_layer = t;
        pending = Diag();
        lev.sweeps.push_back(s);
      } else if (!lev.sweeps.empty()) {
        lev.sweeps.back().post = Diag::merge(lev.sweeps.back().post, L.diag);
        lev.sweeps.back().last_layer = t;
      } else {
        pending = Diag::merge(pending, L.diag);
      }
    }
    if (lev.sweeps.empty() && (l == 0 || first <= last)) {
      Sweep s;
      s.pre = pending;
      s.gen = (l == 0);
      s.first_layer = first;
      s.last_layer = last;
      lev.sweeps.push_back(s);
    }
  }
  return hp;
}

}  // namespace qsim
