// Front end of the partitioned simulator (host C++, no CUDA).
//
// Turns a validated grid circuit into two "half programs" (upper / lower), one per
// half of the bipartition of PAPER.md Supp. A, organised as the levels of
// the branch tree: level 0 = layers 1..f_1 (shared by every branch), level l >= 1 =
// the children created by the k_l cut CZs of fork layer f_l, covering layers
// f_l+1 .. f_{l+1}.  Each level is a list of Sweeps; one Sweep is one memory pass
// over a 2^h half state that applies
//     post-diagonal  o  (X^1/2 / Y^1/2 gates on distinct bits)  o  pre-diagonal
// where every run of diagonal gates (CZ, T, projectors P0/P1, Z) is fused into a
// single phase pass "as the paper does" (§2.4, Eqs. 3-6).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/qsim.h"

namespace qsim {

// D(i) = 2^(-nhalf/2) * w^ph(i) * [(i & pm) == pv],  w = e^{i pi/4},
// ph(i) = ph0 + popc(i&t1) + 2 popc(i&t2) + 4 (popc(i&zm) + sum_d popc(i & i>>d & cz[d]))  (mod 8).
// t1/t2/zm carry the per-bit T count mod 8 (T = w on |1>; Z = w^4), cz[d] the CZ pairs
// (bit b with bit b+d, mask bit at b; CZ = w^4 on |11>) — in the identity layout the
// horizontal pairs sit at d = 1 and the vertical ones at d = cols, under a qubit relabelling
// anywhere — pm/pv the projector constraint (P0 / P1, Eq. 1), nhalf the 1/sqrt2 factors.
// Masks are 64-bit on the host (halves of up to 36 qubits); the device form
// (kernels.h DiagDev) is 32-bit: a distributed half's diagonals are first restricted to the shard
// (restrict_low: its global bits are constants of the rank).
struct Diag {
  uint64_t t1 = 0, t2 = 0, zm = 0, pm = 0, pv = 0;
  uint64_t cz[64] = {};
  int ph0 = 0;
  int nhalf = 0;
  bool allzero = false;

  bool has_cz() const {
    for (uint64_t m : cz)
      if (m) return true;
    return false;
  }
  bool identity() const {
    return !allzero && !t1 && !t2 && !zm && !has_cz() && !pm && ph0 == 0 && nhalf == 0;
  }
  int count(int bit) const;          // T count (mod 8) at bit
  void set_count(int bit, int c);
  void add_T(int bit) { set_count(bit, count(bit) + 1); }
  void add_Z(int bit) { set_count(bit, count(bit) + 4); }
  void add_cz(int b0, int b1);        // CZ between two distinct bits
  void add_proj(int bit, int value);  // P0 (value 0) or P1 (value 1)
  // the product of two diagonals (they commute)
  static Diag merge(const Diag &a, const Diag &b);
  double scale() const;  // 2^(-nhalf/2)
  int phase(uint64_t i) const;  // ph(i) mod 8 (host reference of the device formula)
  // The diagonal on the indices whose bits >= hl equal those of g, as a diagonal over bits < hl:
  // T / Z counts and projectors on fixed bits become constants, a CZ pair with one fixed bit a Z
  // (or nothing) on the other bit, a pair of fixed bits a constant.
  Diag restrict_low(int hl, uint64_t g) const;
  bool below(int bits) const;  // every mask is below bit `bits`
  // D^m(i) = D(i ^ m): the diagonal conjugated by the bit flip X^m (sibling flips of the tree
  // executor, Engine::flip_node).  Per bit a in m: count c_a -> -c_a with c_a added to ph0; a CZ
  // pair with one flipped bit adds Z on the other bit, with both flipped Z on both and ph0 += 4.
  Diag shift(uint64_t m) const;
  // 1 / D (no projector): phases negated (CZ terms are their own negation mod 8), scale inverted
  Diag inverse() const;
  // the phase of D only (scale 1, no projector)
  Diag phase_only() const;
};

// One non-diagonal gate of a sweep after factoring out its global phase:
// SX = (w/sqrt2) [[1,-i],[-i,1]] (kind 1), SY = (w/sqrt2) [[1,-1],[1,1]] (kind 2).
struct Gate1 {
  uint8_t bit;
  uint8_t kind;
};

struct Sweep {
  std::vector<Gate1> gates;  // distinct bits
  Diag pre, post;
  bool gen = false;  // input not read: value = pre(i) (the H layer and leading diagonals)
  int first_layer = 0, last_layer = 0;
  // distributed half: after this sweep, exchange local bit .first with global
  // bit .second (physical positions) — fused into the sweep's stores over peer memory
  std::vector<std::pair<int, int>> swaps;
};

struct Level {
  int fork_layer = 0;          // 0 for the root; the fork applies at the input of layer fork_layer + 1
  int k = 0;                   // cuts at this fork (children = 2^k)
  int g0 = 0;                  // index of the first of them in the cut list
  std::vector<int> cut_g;      // index in the cut list (= branch bit c-1-g) of fork bit j, ascending
  std::vector<int> cut_bits;   // half-local bit of each cut endpoint in this half
  uint32_t pmask = 0;          // bit j: cut j acts as P_b on this part (upper endpoint), else Z^b
  std::vector<Sweep> sweeps;
};

struct HalfProgram {
  bool upper = true;
  int h = 0;
  int ncuts = 0;  // cut bits of this program's branch index (sum of the levels' k)
  int hl = 0;  // qubits per shard: h, or h - log2(ranks) for a distributed half (f3)
  std::vector<int> perm;  // physical bit of canonical local bit c (h-1-k' for local qubit k'):
                          // the layout of the leaf (and of every sweep unless the layout changes)
  std::vector<Level> levels;
  // Diagonal of fork child c at level l (P_{bits} on the upper endpoints, Z^{bits} on the lower)
  Diag fork_diag(int level, uint64_t child) const;
  // physical index of canonical half index x (bit c of x moves to bit perm[c])
  uint64_t phys(uint64_t x) const {
    uint64_t y = 0;
    for (int c = 0; c < h; ++c)
      if ((x >> c) & 1u) y |= 1ull << perm[c];
    return y;
  }
  size_t total_sweeps() const;
};

struct Circuit {
  uint32_t rows = 0, cols = 0, depth = 0, cut_row = 0;
  uint32_t n = 0, h_u = 0, h_l = 0;
  std::vector<qsim_gate> gates;
  std::vector<qsim_cut> cuts;       // ordered by (layer, q_upper)
  std::vector<int> fork_layers;     // distinct cut layers, ascending
  std::vector<int> fork_k;          // cuts per fork layer
};

// Validates and derives the cut list.  Returns "" or an error message (EINVAL).
std::string build_circuit(uint32_t rows, uint32_t cols, uint32_t depth, const qsim_gate *gates,
                          size_t n_gates, uint32_t cut_row, const uint32_t *cut_layers,
                          size_t n_cut_layers, Circuit &out);

// A cut endpoint inside one part of a multi-part partition: the cut CZ of
// `layer` acts on `q` as P_b (proj, the part above the boundary) or Z^b (the part below).
struct PartCut {
  int layer;
  uint32_t q;
  bool proj;
};

// Program of the qubit range [lo, hi) whose branch index enumerates `cuts` (ordered by
// (layer, upper qubit); one fork level per distinct layer).  Halves are the case
// [0, h_u) with every cut as P and [h_u, n) with every cut as Z.
// apply (optional, one entry per cut): the layer at whose input the cut's P_b / Z^b is applied,
// in (cut layer, depth + 1] (depth + 1: after the last layer, at the leaf).  Default: the layer
// after the cut CZ.  A later layer is exact as long as no X^1/2 / Y^1/2 acts on the cut's qubit
// in between (P_b and Z^b commute with every diagonal and with gates on other qubits): the
// deferred forks of the tree executor (Engine::choose_tree).
HalfProgram compile_part(const Circuit &c, uint32_t lo, uint32_t hi, bool upper, const std::vector<PartCut> &cuts,
                         const std::vector<std::vector<int>> &layer_perm, const std::vector<int> &final_perm,
                         const std::vector<int> *apply = nullptr);

// Layer of the first X^1/2 / Y^1/2 gate on the cut's qubit after the cut layer (depth + 1: none):
// the latest layer at whose input the cut's fork may be applied.
std::vector<int> first_targets(const Circuit &c, const std::vector<PartCut> &cuts);
// The cut list of a half as PartCuts.  p_upper[g] = 1 (default for every cut): P_b on the upper
// endpoint, Z^b on the lower one (Eq. 1; R6); 0: the same identity read the other
// way round, CZ = I (x) P0 + Z (x) P1 (P_b on the lower endpoint, Z^b on the upper one).
std::vector<PartCut> half_cuts(const Circuit &c, bool upper, const std::vector<char> *p_upper = nullptr);
// Layers in [1, depth] holding at least one X^1/2 / Y^1/2 gate on a qubit in [lo, hi).
std::vector<int> gate_layers(const Circuit &c, uint32_t lo, uint32_t hi);

// ---- Pauli frames of the branch tree (DESIGN.md §5 "Frames").  A frame F = phi . X^m (X^m: flip
// of the bits in m, then the diagonal phi) relates a branch state to another one: psi_b = F psi_a.
// A fork Z^b is a frame; it moves through a sweep G = post . gates . pre as G F G^-1 = F' while
// every target t of G sees F as I or Z (phi's count at t in {0, 4}, no CZ term on t): the factored
// gates I - iX, I - iY are Clifford, and diagonals conjugate a flip into a flip times a ratio
// D / D^m.  frame_through replaces (phi, m) by F' and returns true, or returns false (F unchanged)
// where the frame breaks: from there the two states need sweeps of their own.
bool frame_through(const Sweep &sw, Diag &phi, uint64_t &m);
// F2 . F1 (apply F1 first): phi2 . phi1^{m2} . X^{m1 ^ m2}
void frame_compose(const Diag &phi2, uint64_t m2, const Diag &phi1, uint64_t m1, Diag &phi, uint64_t &m);
// F^-1 = (1 / phi)^m . X^m
void frame_inverse(const Diag &phi, uint64_t m, Diag &inv_phi);

// The frames of Z^b forks stay linear (D / D^m of a quadratic D is linear): phi(x) = w^{ph0 + sum_a
// c_a x_a} with the counts c_a = t1_a + 2 t2_a + 4 zm_a held as bit planes, so that moving, composing
// and inverting a frame are a few word operations (the executor keeps one frame per tree node).
struct LinFrame {
  uint64_t t1 = 0, t2 = 0, zm = 0, m = 0;
  int ph0 = 0;
  bool identity() const { return !t1 && !t2 && !zm && !m && ph0 == 0; }
  int count(int a) const { return (int)((t1 >> a) & 1u) + 2 * (int)((t2 >> a) & 1u) + 4 * (int)((zm >> a) & 1u); }
  void add_counts(uint64_t b1, uint64_t b2, uint64_t b4);  // c_a += b1_a + 2 b2_a + 4 b4_a (mod 8)
  void negate(uint64_t mask);                              // c_a = -c_a on the bits of mask
  void add_Z(int a) { zm ^= 1ull << a; }
  LinFrame shift(uint64_t s) const;                        // phi^s (x -> x ^ s), flip unchanged
  Diag diag() const;                                       // phi as a Diag
};
bool lin_through(const Sweep &sw, LinFrame &f);
// Where f breaks on phases alone (a target t whose count c is not 0 or 4), f is a sum of two frames:
// w^{c x_t} = a + b (-1)^{x_t} with a = (1 + w^c) / 2, b = (1 - w^c) / 2 (count 0 and count 4 at t).
// Writes the terms moved through sw (frames to out, complex coefficients to coef[2 i], coef[2 i + 1])
// and returns their number (1 when f moves as it is), or 0 when f breaks otherwise (a projector
// meets the flip) or would need more than max_terms terms.
int lin_expand_through(const Sweep &sw, const LinFrame &f, int max_terms, LinFrame *out, double *coef);
LinFrame lin_compose(const LinFrame &f2, const LinFrame &f1);  // f2 . f1
LinFrame lin_inverse(const LinFrame &f);

// perm: physical bit of each canonical local bit (identity when empty); every bit position of the
// program (gates, diagonals, forks) is physical.
HalfProgram compile_half(const Circuit &c, bool upper, const std::vector<int> &perm = {});
// The same with a layout per gate layer (layer_perm[t], t = 0..depth; a layer's diagonal and fork
// bits use the layout of the sweep that applies them); perm of the result = final_perm.
HalfProgram compile_half_layers(const Circuit &c, bool upper, const std::vector<std::vector<int>> &layer_perm,
                                const std::vector<int> &final_perm);

}  // namespace qsim
