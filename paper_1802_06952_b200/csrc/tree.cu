// Branch-tree executors of one half: deferred-fork placement and the
// depth-first / level-synchronous tree executors, sibling flips, and the Pauli-frame executor (the
// default), with their leaf gathers.
#include "engine.h"
#include "engine_internal.h"

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <set>
#include <sstream>
#include <unordered_map>
#include <unordered_set>

namespace qsim {

// ---------------------------------------------------------------- deferred-fork branch trees
// SURVEY §8(a) a4 (prefix sharing).  Eq. 1 replaces a cut CZ by P_b (upper endpoint) and
// Z^b (lower endpoint) at the cut layer.  Both are diagonal on the cut's qubit, so they commute
// with every later diagonal (T, CZ, other projectors) and with every gate on other qubits: the
// fork may be applied at the input of any layer up to the first X^1/2 / Y^1/2 on that qubit
// (HalfExec::ft), and the branches stay one shared state until then.  Cuts never targeted again
// (or targeted only in the lazily evaluated tail) fork inside the leaf gather.  choose_tree
// places the forks of a block of branches (a dynamic programme over the half's sweeps, bounded by
// the state buffers that fit in HBM); the executor below runs the resulting tree depth-first.

// Lazy tail of a tree path: its last L sweeps (L <= 3) evaluated at the sampled indices (stage 0 on
// a cone of nS * 2^{k_1 + .. + k_{L-1}} points, each summing 2^{k_0} scattered reads of the state;
// later stages from those values).  Cost in bytes: ~64 per scattered read (32-byte sectors shared
// by neighbouring targets; the C5 launch lists give ~9e10 reads/s), ~16 per compact read, against
// 2 * 2^h * amp per sweep saved.  QSIM_OPT_LAZY_LAST: 0 off, 1 one sweep, 2 (default) up to three by
// this model, 3 / 4 two / three whenever possible (tests).
int Engine::tree_lazy(int half, int64_t nS) const { return tree_lazy_of(half_[half].prog, nS); }

int Engine::tree_lazy_of(const HalfProgram &hp, int64_t nS) const {
  std::vector<const Sweep *> sw;
  for (auto &l : hp.levels)
    for (auto &s : l.sweeps) sw.push_back(&s);
  if (full_leaf_ || lazy_depth_ < 1 || sw.size() < 2) return 0;
  const int S = (int)sw.size();
  const double sweep = 2.0 * std::ldexp(1.0, hp.hl) * (double)amp_;
  auto feasible = [&](int L) {
    if (L + 1 > S) return false;
    double pts = (double)nS;
    for (int s = S - 1; s >= S - L; --s) {
      if (sw[s]->gen || sw[s]->gates.size() > 12) return false;
      if (s > S - L) pts *= std::ldexp(1.0, (int)sw[s]->gates.size());
    }
    return pts <= (double)(1 << 27);
  };
  auto cost = [&](int L) {  // bytes of the lazy stages minus the sweeps they save
    double pts = (double)nS, c = 0.0;
    for (int s = S - 1; s >= S - L; --s) {
      const double terms = std::ldexp(1.0, (int)sw[s]->gates.size());
      c += (s == S - L ? 64.0 : 16.0) * pts * terms;
      pts *= terms;
    }
    return c - L * sweep;
  };
  if (!feasible(1)) return 0;
  if (lazy_depth_ == 1) return 1;
  if (lazy_depth_ == 3) return feasible(2) ? 2 : 1;
  if (lazy_depth_ == 4) return feasible(3) ? 3 : feasible(2) ? 2 : 1;
  int best = 1;
  for (int L = 2; L <= 3; ++L)
    if (feasible(L) && cost(L) < cost(best)) best = L;
  return best;
}

// Fork placement for the aligned block of 2^m branches whose top c - m cut bits are fixed.
// Sweep i of the half (one per gate layer gl[i]; sweep 0 generates the state) is materialised for
// i < Sm = S - lz.  A free cut g may fork at the input of sweep p with cut layer < gl[p] <=
// ft_g (p >= 1), or in the gather when ft_g is a lazy layer or never comes (allow_gather).
// With fork points p_1 < .. < p_K and every cut at the latest point <= its ft, the states between
// p_i and p_{i+1} number 2^{#cuts with ft index < p_{i+1}}, so the cost of a segment does not
// depend on the earlier points: a DP over (last point, points used), K <= nbuf - 1 (each
// branching level keeps its parent state).  Pinning the j cuts that must fork first (the
// executor enumerates them, recomputing the path above) trades recomputation for buffers.
TreeChoice Engine::choose_tree(int half, int m, int lz, int64_t nS, int nbuf, bool allow_gather) const {
  const HalfExec &he = half_[half];
  const int c = (int)circ_.cuts.size();
  const std::vector<int> &gl = he.glayers;
  const int S = (int)gl.size(), Sm = S - lz;
  const int Kmax = std::max(0, nbuf - 1);
  auto W = [&](int a, int b) {  // sweep units of sweeps [a, b)
    double w = 0;
    for (int i = a; i < b; ++i) w += i == 0 ? 0.5 : 1.0;
    return w;
  };
  auto idx_after = [&](int layer) {  // first sweep with gl > layer
    int i = 0;
    while (i < S && gl[i] <= layer) ++i;
    return i;
  };
  // per cut: lo = earliest sweep it may fork at (a branching point is >= 1: sweep 0 generates the
  // root), e = index of its first target (S: none); pinned cuts apply at sweep lo0
  std::vector<int> lo(c), lo0(c), e(c);
  for (int g = 0; g < c; ++g) {
    lo0[g] = idx_after((int)circ_.cuts[g].layer);
    lo[g] = std::max(1, lo0[g]);
    int ei = S;
    for (int i = 0; i < S; ++i)
      if (gl[i] == he.ft[g]) ei = i;
    e[g] = ei;
  }
  // one more fork value in the gather: a lazy stage (~96 bytes per scattered read) or a gather
  const double sweep_bytes = 2.0 * std::ldexp(1.0, half_[half].prog.hl) * (double)amp_;
  int kd = 0;
  for (auto &l : he.prog.levels)
    if (!l.sweeps.empty()) kd = (int)l.sweeps.back().gates.size();
  const double gamma = lz > 0 ? 96.0 * (double)nS * std::ldexp(1.0, kd) / sweep_bytes : 32.0 * (double)nS / sweep_bytes;
  std::vector<int> forced, freec;
  for (int g = c - m; g < c; ++g) {
    const bool gather = e[g] >= Sm;
    const int ee = gather ? Sm - 1 : e[g];
    if (gather && allow_gather) {
      freec.push_back(g);
      continue;
    }
    if (ee < 1 || lo[g] > ee)
      forced.push_back(g);
    else
      freec.push_back(g);
  }
  auto eff = [&](int g) { return e[g] >= Sm ? (allow_gather ? S : Sm - 1) : e[g]; };
  std::sort(freec.begin(), freec.end(), [&](int a, int b) { return eff(a) != eff(b) ? eff(a) < eff(b) : a < b; });
  TreeChoice best;
  best.cost = -1;
  const int jmax = Kmax == 0 ? (int)freec.size() : std::min<int>((int)freec.size(), 16);
  for (int j = 0; j <= jmax; ++j) {
    std::vector<int> R, G;  // materialised forks, gather forks
    for (size_t t = (size_t)j; t < freec.size(); ++t) (eff(freec[t]) >= S ? G : R).push_back(freec[t]);
    const int nR = (int)R.size();
    // dp[q][k]: cost of sweeps [0, q) with k points, the last at q (q >= 1); -1 = infeasible
    std::vector<std::vector<double>> dp(Sm + 1, std::vector<double>(Kmax + 2, -1.0));
    std::vector<std::vector<int>> from(Sm + 1, std::vector<int>(Kmax + 2, -1));
    auto cnt_lt = [&](int q) {
      int n = 0;
      for (int g : R) n += eff(g) < q;
      return n;
    };
    auto seg_ok = [&](int p, int q) {  // cuts with eff in [p, q) fork at p
      for (int g : R)
        if (eff(g) >= p && eff(g) < q && lo[g] > p) return false;
      return true;
    };
    for (int q = 1; q < Sm && Kmax >= 1; ++q) {
      if (cnt_lt(q) == 0) dp[q][1] = W(0, q), from[q][1] = 0;
      for (int k = 2; k <= Kmax; ++k)
        for (int p = 1; p < q; ++p) {
          if (dp[p][k - 1] < 0 || !seg_ok(p, q)) continue;
          const double v = dp[p][k - 1] + std::ldexp(W(p, q), cnt_lt(q));
          if (dp[q][k] < 0 || v < dp[q][k]) dp[q][k] = v, from[q][k] = p;
        }
    }
    double cost = -1;
    int bq = -1, bk = 0;
    if (nR == 0) cost = W(0, Sm);
    for (int q = 1; q < Sm; ++q)
      for (int k = 1; k <= Kmax; ++k) {
        if (dp[q][k] < 0 || !seg_ok(q, Sm)) continue;
        const double v = dp[q][k] + std::ldexp(W(q, Sm), nR);
        if (cost < 0 || v < cost - 1e-9) cost = v, bq = q, bk = k;
      }
    if (cost < 0) continue;
    cost += std::ldexp(gamma, nR + (int)G.size());
    const double total = std::ldexp(cost, j + (int)forced.size());
    if (best.cost >= 0 && total >= best.cost - 1e-9) continue;
    best.cost = total;
    best.points = bk;
    best.qlist.assign(forced.begin(), forced.end());
    for (int t = 0; t < j; ++t) best.qlist.push_back(freec[t]);
    std::vector<int> pts;
    for (int q = bq, k = bk; q > 0 && k > 0; q = from[q][k], --k) pts.push_back(q);
    std::sort(pts.begin(), pts.end());
    best.apply.assign(c, 0);
    for (int g = 0; g < c; ++g) best.apply[g] = lo0[g] < S ? gl[lo0[g]] : (int)circ_.depth + 1;  // pinned
    for (int g : G) best.apply[g] = he.ft[g];
    for (int g : R) {
      int p = -1;
      for (int x : pts)
        if (x <= eff(g)) p = x;
      best.apply[g] = gl[p];
    }
  }
  if (best.cost < 0) throw Error(QSIM_EINVAL, "no feasible fork placement");
  return best;
}

TreeVariant &Engine::variant(int half, const std::vector<int> &apply, const std::vector<char> &roles) {
  HalfExec &he = half_[half];
  std::vector<int> key = apply;
  for (char r : roles) key.push_back(r ? -1 : -2);
  auto it = he.variants.find(key);
  if (it != he.variants.end()) return *it->second;
  if (he.variants.size() >= 64) he.variants.clear();
  auto v = std::make_unique<TreeVariant>();
  const bool up = half == 0;
  const std::vector<int> &perm = he.prog.perm;
  v->prog = compile_part(circ_, up ? 0 : circ_.h_u, up ? circ_.h_u : circ_.n, up,
                         half_cuts(circ_, up, roles.empty() ? nullptr : &roles),
                         std::vector<std::vector<int>>(circ_.depth + 2, perm), perm, &apply);
  plan_levels(v->prog, v->plans, true);
  TreeVariant &ref = *v;
  he.variants[key] = std::move(v);
  return ref;
}

// Which endpoint of each cut gets the projector (Eq. 1 both ways, program.h half_cuts).  The sweep
// that applies a deferred P_b fork does not load the half of its tile the projector zeroes
// (sweep_tma.cu), a Z^b fork saves nothing: P goes to the half whose fork of that cut runs on
// more tree nodes (2^{forks placed before it} for the whole-range tree of each half).
void Engine::choose_roles() {
  roles_chosen_ = true;
  roles_.clear();
  const int c = (int)circ_.cuts.size();
  if (!roles_auto_ || dist_ || c == 0 || !half_[0].tree || !half_[1].tree) return;
  std::vector<double> w[2];
  for (int h = 0; h < 2; ++h) {
    HalfExec &he = half_[h];
    if (he.glayers.empty()) {
      const bool up = h == 0;
      he.glayers = gate_layers(circ_, up ? 0 : circ_.h_u, up ? circ_.h_u : circ_.n);
      he.ft = first_targets(circ_, half_cuts(circ_, up));
    }
    const int64_t nS = (int64_t)(h == 0 ? Su_.size() : Sl_.size());
    const int lz = tree_lazy(h, nS);
    const TreeChoice tc = choose_tree(h, c, lz, nS, 6, true);
    w[h].assign(c, 0.0);
    const int S = (int)he.glayers.size();
    const int last_mat = S - lz > 0 ? he.glayers[S - lz - 1] : 0;
    for (int g = 0; g < c; ++g) {
      if (tc.apply[g] > last_mat) continue;  // forks in the gather: no sweep reads it
      int before = 0;
      for (int x = 0; x < c; ++x) before += tc.apply[x] < tc.apply[g];
      w[h][g] = std::ldexp(1.0, before);
    }
  }
  roles_.assign(c, 1);
  bool any = false;
  for (int g = 0; g < c; ++g)
    if (w[1][g] > w[0][g]) roles_[g] = 0, any = true;
  if (!any) roles_.clear();
  if (std::getenv("QSIM_DEBUG_TREE")) {
    std::fprintf(stderr, "roles (1 = P on the upper endpoint):");
    for (int g = 0; g < c; ++g) std::fprintf(stderr, " %d", roles_.empty() ? 1 : (int)roles_[g]);
    std::fprintf(stderr, "\n");
  }
}

// [b0, b1) as aligned power-of-two blocks; slice row r = branch b0 + r
void Engine::evolve_tree(int half, uint64_t b0, uint64_t b1, void *slice, const uint64_t *dS, int64_t nS,
                         bool canonical, bool flip, bool zz) {
  Nvtx nv(half == 0 ? "upper half tree" : "lower half tree");
  HalfExec &he = half_[half];
  if (he.glayers.empty()) {
    const bool up = half == 0;
    he.glayers = gate_layers(circ_, up ? 0 : circ_.h_u, up ? circ_.h_u : circ_.n);
    he.ft = first_targets(circ_, half_cuts(circ_, up));
  }
  const int c = (int)circ_.cuts.size();
  for (uint64_t s = b0; s < b1;) {
    int m = 0;
    while (m < c && ((s >> m) & 1u) == 0 && s + (2ull << m) <= b1) ++m;
    static const std::vector<char> none;
    basis_row0_ = s - b0;  // the block's first row in the slice (frame basis entries)
    // zz: Z^b on the upper endpoint of every free cut of the block (evolve_block keeps the fixed ones)
    const std::vector<char> zroles(zz && half == 0 ? (size_t)c : 0, 0);
    evolve_block(half, s, m, (char *)slice + (s - b0) * (uint64_t)nS * amp_, dS, nS,
                 canonical ? none : zz ? (half == 0 ? zroles : none) : roles_, flip);
    s += 1ull << m;
  }
}

void Engine::evolve_block(int half, uint64_t b0, int m, void *slice, const uint64_t *dS, int64_t nS,
                          const std::vector<char> &roles, bool flip) {
  HalfExec &he = half_[half];
  const int c = (int)circ_.cuts.size();
  const int T = tile_low_bits(c128_) + kHiBits;
  if (he.prog.hl < T) throw Error(QSIM_EINVAL, "tree mode needs h >= tile bits");
  lazy_idx_valid_ = false;  // the block's indices may have been re-uploaded since the last block
  state_bytes_ = ((size_t)1 << he.prog.hl) * amp_;
  // level-synchronous subtrees for small states (launch-bound otherwise): gather forks pinned
  if (!(bfs_ && sweep_kernel_ != 1 && state_bytes_ <= ((size_t)256 << 20))) {  // their buffers are state memory now
    bfs_buf_[0].release();
    bfs_buf_[1].release();
  }
  size_t free_b = 0, total_b = 0;
  check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  size_t have = bfs_buf_[0].bytes + bfs_buf_[1].bytes;
  for (auto *b : states_) have += b->bytes;
  const bool bfs = bfs_ && sweep_kernel_ != 1 && state_bytes_ <= ((size_t)256 << 20);
  const int lz = bfs ? std::min(2, tree_lazy(half, nS)) : tree_lazy(half, nS);  // bfs_tree: <= 2 stages
  size_t margin = (size_t)512 << 20;
  {  // cone index / value buffers of the lazy tail
    std::vector<const Sweep *> sw;
    for (auto &l : he.prog.levels)
      for (auto &x : l.sweeps) sw.push_back(&x);
    double pts = (double)nS;
    for (int s2 = (int)sw.size() - 1; s2 > (int)sw.size() - lz; --s2) {
      pts *= std::ldexp(1.0, (int)sw[s2]->gates.size());
      margin += (size_t)(pts * (double)(amp_ + 8));
    }
  }
  const size_t avail = free_b + have > margin ? free_b + have - margin : 0;
  const size_t nfit = avail / state_bytes_;
  if (nfit < 1) {
    std::ostringstream msg;
    msg << "a " << he.prog.h << "-qubit half state needs " << state_bytes_ << " bytes; only " << avail
        << " bytes available for state buffers";
    throw Error(QSIM_ENOMEM, msg.str());
  }
  int nbuf = (int)std::min<size_t>(nfit, 12);
  if (mem_budget_ > 0) nbuf = std::max(1, std::min<int>(nbuf, (int)((size_t)mem_budget_ / state_bytes_)));
  // a swapped cut (P on the lower endpoint) changes the single branches, only the sum over both
  // values of its bit is CZ: the block's fixed bits keep the canonical roles (qsim.h: U_b, L_b)
  std::vector<char> eff = roles;
  for (int g = 0; g < c - m && g < (int)eff.size(); ++g) eff[g] = 1;
  if (std::find(eff.begin(), eff.end(), 0) == eff.end()) eff.clear();
  std::vector<int> pin(c, -1);
  for (int g = 0; g < c - m; ++g) pin[g] = (int)((b0 >> (c - 1 - g)) & 1u);
  if (flip && (!bfs || frames_)) {  // frames / sibling flips; false: not applicable, the executors below
    const TreeChoice fc = flip_choice(half, m);
    const TreeVariant &fv = variant(half, fc.apply, eff);
    if (std::getenv("QSIM_DEBUG_TREE")) {
      std::fprintf(stderr, "flip tree half %d b0=%llu m=%d nbuf=%d levels", half, (unsigned long long)b0, m, nbuf);
      for (auto &l : fv.prog.levels) std::fprintf(stderr, " [%d:k%d s%zu]", l.fork_layer + 1, l.k, l.sweeps.size());
      std::fprintf(stderr, "\n");
    }
    if (frames_ && run_tree_frames(half, fv, pin, m, slice, dS, nS, nbuf)) return;
    if (!bfs && run_tree_flip(half, fv, lz, pin, m, slice, dS, nS, nbuf)) return;
  }
  const TreeChoice tc = choose_tree(half, m, lz, nS, nbuf, !bfs);
  const TreeVariant &v = variant(half, tc.apply, eff);
  ensure_states(half, tc.points + 1);
  size_t bfs_avail = 0;  // memory the level-synchronous buffers may take (0: none)
  if (bfs) {
    size_t used = 0;
    for (auto *b : states_) used += b->bytes;
    bfs_avail = avail > used ? avail - used : 1;
  }
  if (std::getenv("QSIM_DEBUG_TREE")) {
    std::fprintf(stderr, "tree half %d b0=%llu m=%d lz=%d nbuf=%d: cost %.1f sweeps, %d points, %zu pinned, levels",
                 half, (unsigned long long)b0, m, lz, nbuf, tc.cost, tc.points, tc.qlist.size());
    for (auto &l : v.prog.levels) std::fprintf(stderr, " [%d:k%d s%zu]", l.fork_layer + 1, l.k, l.sweeps.size());
    std::fprintf(stderr, "\n");
  }
  const size_t nq = tc.qlist.size();
  for (uint64_t q = 0; q < (1ull << nq); ++q) {
    for (size_t i = 0; i < nq; ++i) pin[tc.qlist[i]] = (int)((q >> i) & 1u);
    run_tree(half, v, lz, pin, m, slice, dS, nS, bfs_avail);
  }
}

namespace {
// the fork values of level `lev` consistent with the pinned cuts: child index (bit k-1-j = fork
// bit j) and the branch bits it sets
struct ChildSet {
  uint64_t base = 0;
  std::vector<int> free;  // fork bits j that are free
};
ChildSet child_set(const Level &lev, const std::vector<int> &pin) {
  ChildSet cs;
  for (int j = 0; j < lev.k; ++j) {
    const int p = pin[lev.cut_g[j]];
    if (p < 0)
      cs.free.push_back(j);
    else if (p)
      cs.base |= 1ull << (lev.k - 1 - j);
  }
  return cs;
}
uint64_t child_of(const Level &lev, const ChildSet &cs, uint64_t f) {
  uint64_t ch = cs.base;
  for (size_t t = 0; t < cs.free.size(); ++t)
    if ((f >> t) & 1u) ch |= 1ull << (lev.k - 1 - cs.free[t]);
  return ch;
}
uint64_t branch_bits(const Level &lev, uint64_t ch, int c) {
  uint64_t b = 0;
  for (int j = 0; j < lev.k; ++j)
    if ((ch >> (lev.k - 1 - j)) & 1u) b |= 1ull << (c - 1 - lev.cut_g[j]);
  return b;
}
}  // namespace

namespace {
// diagonal of the pinned fork bits of a level (free bits left out)
Diag pinned_diag(const Level &lev, const std::vector<int> &pin) {
  Diag d;
  for (int j = 0; j < lev.k; ++j) {
    const int p = pin[lev.cut_g[j]];
    if (p < 0) continue;
    if ((lev.pmask >> j) & 1u)
      d.add_proj(lev.cut_bits[j], p);
    else if (p)
      d.add_Z(lev.cut_bits[j]);
  }
  return d;
}
// lazy stages of a tree path: (sweep, level whose fork enters its pre or -1), the last lz sweeps
std::vector<std::pair<const Sweep *, int>> lazy_stages(const HalfProgram &hp, int lz) {
  std::vector<std::pair<const Sweep *, int>> st;
  for (int l = (int)hp.levels.size() - 1; l >= 0 && (int)st.size() < lz; --l) {
    const auto &sw = hp.levels[l].sweeps;
    for (int i = (int)sw.size() - 1; i >= 0 && (int)st.size() < lz; --i) st.push_back({&sw[i], i == 0 ? l : -1});
  }
  std::reverse(st.begin(), st.end());
  return st;
}
}  // namespace

// The subtree below a level-l node, level by level (SURVEY §8(a) a4 for small states, where one
// launch per node and sweep is launch-bound): the sweeps of level q run as ONE node-batched launch
// over its 2^{free bits of levels l+1..q} states (node = (parent << n) | child; the first launch
// reads the parent and applies the fork per node, the pinned bits' diagonal merged into its pre);
// the leaves are gathered by batched launches whose output rows follow the branch order.  Needs
// the gather forks pinned (choose_tree with allow_gather = false).  false: does not fit.
bool Engine::bfs_tree(const TreeVariant &v, int lz, int M, const std::vector<int> &skip, const std::vector<int> &pin,
                      int l, const void *state, uint64_t bacc, int m, void *slice, const uint64_t *dS, int64_t nS,
                      size_t avail) {
  const HalfProgram &hp = v.prog;
  const int F = (int)hp.levels.size() - 1, c = (int)circ_.cuts.size();
  std::vector<ChildSet> cs(M + 1);
  std::vector<int> sb(M + 1, 0);
  for (int q = l + 1; q <= M; ++q) {
    cs[q] = child_set(hp.levels[q], pin);
    sb[q] = sb[q - 1] + (int)cs[q].free.size();
  }
  const int nb = sb[M];
  if (nb < 1 || nb > 30) return false;
  for (int q = M + 1; q <= F; ++q)
    if (!child_set(hp.levels[q], pin).free.empty()) return false;
  for (int q = l + 1; q <= M; ++q) {
    const auto &launches = v.plans[q][std::min<size_t>((size_t)skip[q], v.plans[q].size() - 1)];
    if (launches.empty()) return false;
    for (const TilePlan &tp : launches)
      if (tp.gen || !tp.swaps.empty()) return false;
  }
  size_t need[2] = {0, 0};
  for (int q = l + 1; q <= M; ++q) need[q & 1] = std::max(need[q & 1], state_bytes_ << sb[q]);
  const size_t extra = ((size_t)256 << 20) + (lz == 2 ? ((size_t)1 << 30) : 0);  // + the lazy cone chunk
  if (need[0] + need[1] + extra > avail) return false;
  // avail counts the buffers already held as reclaimable: drop them when growing in place would not fit
  if (std::max(bfs_buf_[0].bytes, need[0]) + std::max(bfs_buf_[1].bytes, need[1]) + extra > avail) {
    bfs_buf_[0].release();
    bfs_buf_[1].release();
  }
  bfs_buf_[0].reserve(need[0]);
  bfs_buf_[1].reserve(need[1]);
  const void *src = state;
  for (int q = l + 1; q <= M; ++q) {
    const Level &lev = hp.levels[q];
    const auto &launches = v.plans[q][std::min<size_t>((size_t)skip[q], v.plans[q].size() - 1)];
    void *dst = bfs_buf_[q & 1].ptr;
    ForkDev f;
    std::memset(&f, 0, sizeof(f));
    f.n = (int)cs[q].free.size();
    uint32_t proj = 0;
    for (int t = 0; t < f.n; ++t) {
      const int j = cs[q].free[t];
      f.bit[t] = (uint8_t)lev.cut_bits[j];
      if ((lev.pmask >> j) & 1u) {
        f.pmask |= 1u << t;
        proj |= 1u << lev.cut_bits[j];
      }
    }
    const Diag pinned = pinned_diag(lev, pin);
    for (size_t i = 0; i < launches.size(); ++i)
      launch_nodes(launches[i], i == 0 ? src : dst, dst, sb[q], i == 0 ? f.n : 0, f, hp, i == 0, proj,
                   i == 0 ? &pinned : nullptr);
    src = dst;
  }
  // leaf node N (bits of level q's fork entry t at N's bit (sb[M] - sb[q]) + (n_q - 1 - t)) -> row
  RowMapDev rm;
  std::memset(&rm, 0, sizeof(rm));
  rm.nbits = nb;
  uint64_t fixed = bacc;
  for (int q = l + 1; q <= F; ++q) fixed |= branch_bits(hp.levels[q], child_set(hp.levels[q], pin).base, c);
  const uint64_t rmask = m >= 64 ? ~0ull : ((1ull << m) - 1ull);
  rm.base = (uint32_t)(fixed & rmask);
  for (int q = l + 1; q <= M; ++q) {
    const int n = (int)cs[q].free.size();
    for (int t = 0; t < n; ++t) {
      const int nbit = (sb[M] - sb[q]) + (n - 1 - t);
      rm.pos[nbit] = (uint8_t)(c - 1 - hp.levels[q].cut_g[cs[q].free[t]]);
    }
  }
  const int64_t nleaves = (int64_t)1 << nb;
  rowmap_.reserve((size_t)nleaves * 4);
  check(launch_rowmap(rowmap_.as<uint32_t>(), nleaves, rm, stream_), "rowmap launch");
  st_.kernel_launches++;
  // gather: forks of the gather levels are pinned (constant diagonals)
  const auto st = lazy_stages(hp, lz);
  const int pl = (F > M && hp.levels[F].sweeps.empty()) ? F : -1;
  auto fork_of = [&](int q) { return q < 0 ? Diag() : pinned_diag(hp.levels[q], pin); };
  const uint64_t stride = (uint64_t)1 << hp.hl;
  if (lz == 0) {
    ForkDev f0;
    std::memset(&f0, 0, sizeof(f0));
    const DiagDev pend = to_dev(fork_of(pl));
    check(launch_gather_nodes(src, stride, 0, nleaves, dS, nS, slice, f0, c128_, stream_, &pend, rowmap_.as<uint32_t>()),
          "gather nodes launch");
    st_.kernel_launches++;
    return true;
  }
  auto lazy = [&](const Sweep &sw, const Diag &pre, const Diag &post) {
    LazyLayer ll = lazy_layer(sw, pre);
    ll.post = to_dev(post, true);
    ll.node_stride = stride;
    return ll;
  };
  if (lz == 1) {
    const Sweep &sw = *st[0].first;
    LazyLayer ll = lazy(sw, Diag::merge(sw.pre, fork_of(st[0].second)), Diag::merge(sw.post, fork_of(pl)));
    ll.nper = nS;
    ll.rowmap = rowmap_.as<uint32_t>();
    check(launch_gather_layer(src, dS, nS * nleaves, slice, ll, c128_, stream_), "gather_layer launch");
    st_.kernel_launches++;
    st_.lazy_gathers += (uint64_t)nleaves;
    return true;
  }
  const Sweep &s1 = *st[0].first, &s2 = *st[1].first;
  LazyLayer l1 = lazy(s1, Diag::merge(s1.pre, fork_of(st[0].second)), s1.post);
  LazyLayer l2 = lazy(s2, Diag::merge(s2.pre, fork_of(st[1].second)), Diag::merge(s2.post, fork_of(pl)));
  const int64_t ncone = nS << l2.k;
  cone_idx_.reserve((size_t)ncone * 8);
  check(launch_cone_indices(dS, nS, l2, cone_idx_.as<uint64_t>(), stream_), "cone launch");
  st_.kernel_launches++;
  // leaves in chunks whose cone values fit in 1 GiB
  const int64_t per = std::max<int64_t>(1, ((int64_t)1 << 30) / (ncone * (int64_t)amp_));
  int64_t chunk = 1;
  while (chunk * 2 <= per && chunk < nleaves) chunk *= 2;
  cone_val_.reserve((size_t)(ncone * std::min(chunk, nleaves)) * amp_);
  for (int64_t a = 0; a < nleaves; a += chunk) {
    const int64_t cl = std::min(chunk, nleaves - a);
    l1.nper = ncone;
    check(launch_gather_layer((const char *)src + (size_t)a * stride * amp_, cone_idx_.as<uint64_t>(), ncone * cl,
                              cone_val_.ptr, l1, c128_, stream_),
          "gather_layer launch");
    l2.nper = nS;
    l2.rowmap = rowmap_.as<uint32_t>() + a;
    check(launch_gather_layer_compact(cone_val_.ptr, dS, nS * cl, slice, l2, c128_, stream_),
          "gather_layer_compact launch");
    st_.kernel_launches += 2;
  }
  st_.lazy_gathers += (uint64_t)nleaves;
  return true;
}

// ---------------------------------------------------------------- sibling flips
// DESIGN.md §5 "Sibling flips".  Let G = post . gates . pre be the first sweep of a fork level
// and Z^b the fork (the block's free cuts carry Z^b on both endpoints in qsim_evolve_range, R-zz).
// For a qubit q that G targets with g, G Z_q G^-1 = post (g Z g^-1)_q post^-1 with g Z g^-1 = -Y
// for X^1/2 and X for Y^1/2 (the factored forms I - iX, I - iY); Z_q on a qubit G does not target
// commutes with G.  So child b of the fork is child 0 seen through a bit flip and a diagonal:
//   c_b(x) = Phi_b(x) c_0(x ^ m_b),   Phi_b = post / post^{m_b} * psi_b * Z^{untargeted bits of b},
// m_b = the targeted fork qubits of b, psi_b(x) = i (-1)^{x_q} per X^1/2-targeted one (-Y is a
// flip with that phase), D^m(x) = D(x ^ m) (Diag::shift).  Only child 0 runs G.  A sweep reading a
// state V(x) = phi(x) buf[x ^ m] runs conjugated by the flip,
//   G V = X^m [post^m Z_Ym] gates [Z_Ym pre^m phi^m] buf,
// (X^m SY' X^m = Z SY' Z on the Y^1/2 targets Ym in m; X^1/2 commutes with X), so no kernel reads a
// permuted address: the output stays in the flipped coordinates and the leaf gather reads x ^ m.
bool Engine::flip_half(int half) const {
  const HalfExec &he = half_[half];
  if (!flip_ || !deferred_ || dist_ || !he.tree || sweep_kernel_ == 1 || he.prog.hl > 32) return false;
  if (frames_) return true;  // the frame executor needs few sweeps at any state size
  const size_t sb = ((size_t)1 << he.prog.hl) * amp_;
  return !(bfs_ && sb <= ((size_t)256 << 20));  // small states: level-synchronous subtrees
}

// every free cut forks at the input of its first target layer (latest placement; with sibling flips
// a level costs one sweep per parent plus its remaining sweeps per child, so later is never worse),
// or in the leaf gather (lazy tail / never targeted); the block's fixed cuts at the first gate layer
// after the cut (their P_b / Z^b are constants of the block)
TreeChoice Engine::flip_choice(int half, int m) const {
  const HalfExec &he = half_[half];
  const int c = (int)circ_.cuts.size();
  const std::vector<int> &gl = he.glayers;
  TreeChoice tc;
  tc.apply.assign(c, 0);
  for (int g = 0; g < c; ++g) {
    if (g >= c - m) {
      tc.apply[g] = he.ft[g];
      continue;
    }
    size_t i = 0;
    while (i < gl.size() && gl[i] <= (int)circ_.cuts[g].layer) ++i;
    tc.apply[g] = i < gl.size() ? gl[i] : (int)circ_.depth + 1;
  }
  return tc;
}

// runs the launches `tps` (one or more sweeps of a level) on the state `in` into buffer dst (in
// place when dst == in.buf), conjugated by in's flip; `fork` joins the first launch's pre diagonal
void Engine::flip_exec(const std::vector<const TilePlan *> &tps, const Diag &fork, const VState &in, int dst,
                       const HalfProgram &hp, std::vector<Executed> *rec) {
  for (size_t i = 0; i < tps.size(); ++i) {
    const TilePlan &tp = *tps[i];
    Diag zy;  // Z on the Y^1/2 targets of this launch inside the flip
    for (int q = 0; q < 32; ++q)
      if (((tp.sy_targets & (uint32_t)in.m) >> q) & 1u) zy.add_Z(q);
    const Diag base = i == 0 ? Diag::merge(fork, tp.pre) : (tp.use_pre ? tp.pre : Diag());
    Diag pre = Diag::merge(zy, base.shift(in.m));
    if (i == 0 && in.has_phi) pre = Diag::merge(pre, in.phi.shift(in.m));
    const Diag post = Diag::merge(tp.post.shift(in.m), zy);
    const void *src = tp.gen ? nullptr : states_[i == 0 ? in.buf : dst]->ptr;
    launch_plan(tp, Diag(), i == 0, src, states_[dst]->ptr, hp, -1, nullptr, &pre, &post);
    if (rec) rec->push_back(Executed{&tp, pre, post});
  }
}

// restores the input of the executed launches `rec` (run in place on buf) by their inverses, last
// first: (post . gates . pre)^-1 = pre^-1 (Z_T gates Z_T / 2^nt) post^-1, since (I - iX)^-1 =
// Z (I - iX) Z / 2 and (I - iY)^-1 = Z (I - iY) Z / 2 — the same kernel with other diagonals
void Engine::flip_undo(const std::vector<Executed> &rec, int buf, const HalfProgram &hp) {
  for (size_t i = rec.size(); i-- > 0;) {
    const Executed &e = rec[i];
    Diag zt;
    int nt = 0;
    for (int q = 0; q < 32; ++q)
      if ((e.tp->targets >> q) & 1u) zt.add_Z(q), ++nt;
    const Diag pre = Diag::merge(zt, e.post.inverse());
    Diag post = Diag::merge(e.pre.inverse(), zt);
    post.nhalf += 2 * nt;
    launch_plan(*e.tp, Diag(), true, states_[buf]->ptr, states_[buf]->ptr, hp, -1, nullptr, &pre, &post);
    st_.undo_sweeps++;
  }
}

// The tree of one block with sibling flips (depth-first).  Buffers: the root path runs in buffer 0;
// a level's child-0 state whose source must survive (more siblings to come) goes to a buffer of its
// own ("slot") when one is left, else in place over the source and is undone after its subtree.
// Slots are given buffers by the launches the undo would cost (instances x launches).  false: not
// applicable (a free fork that is a projector, or an in-place slot that could not be inverted).
bool Engine::run_tree_flip(int half, const TreeVariant &v, int lz, const std::vector<int> &pin, int m, void *slice,
                           const uint64_t *dS, int64_t nS, int nbuf) {
  const HalfProgram &hp = v.prog;
  const int F = (int)hp.levels.size() - 1, c = (int)circ_.cuts.size();
  std::vector<int> start(F + 2, 0);
  for (int l = 0; l <= F; ++l) start[l + 1] = start[l] + (int)hp.levels[l].sweeps.size();
  const int Sm = start[F + 1] - lz;
  int M = 0;
  std::vector<int> skip(F + 1, 0);
  for (int l = 0; l <= F; ++l) {
    const int n = (int)hp.levels[l].sweeps.size();
    const int mat = std::max(0, std::min(n, Sm - start[l]));
    if (mat > 0) M = l;
    skip[l] = n - mat;
  }
  std::vector<std::vector<const TilePlan *>> first(F + 1), rest(F + 1);
  for (int l = 0; l <= M; ++l) {
    if ((size_t)skip[l] >= v.plans[l].size()) throw Error(QSIM_EINVAL, "internal: lazy tail longer than the plans");
    for (const TilePlan &tp : v.plans[l][(size_t)skip[l]]) {
      if (!tp.swaps.empty()) return false;
      (tp.sweep == 0 ? first[l] : rest[l]).push_back(&tp);
    }
  }
  std::vector<ChildSet> cs(F + 1);
  for (int l = 1; l <= F; ++l) {
    cs[l] = child_set(hp.levels[l], pin);
    if (l <= M)
      for (int j : cs[l].free)
        if ((hp.levels[l].pmask >> j) & 1u) return false;  // a free projector fork: no sibling flips
  }
  // slots: X(l) = level l's first sweep from a shared parent state (once per parent), D(l) = the
  // rest of level l from the shared child-0 state (once per child)
  struct Slot {
    double cost;
    int level;
    bool d, must;
  };
  std::vector<Slot> slots;
  int fb = 0;
  for (int l = 1; l <= M; ++l) {
    if (fb > 0) {
      const bool proj = hp.fork_diag(l, cs[l].base).pm != 0;  // pinned projector: not invertible
      slots.push_back(Slot{std::ldexp(1.0, fb) * (double)first[l].size(), l, false, proj});
    }
    fb += (int)cs[l].free.size();
    if (!rest[l].empty() && fb > 0) slots.push_back(Slot{std::ldexp(1.0, fb) * (double)rest[l].size(), l, true, false});
  }
  std::sort(slots.begin(), slots.end(), [](const Slot &a, const Slot &b) {
    return a.must != b.must ? a.must : a.cost > b.cost;
  });
  int budget = std::max(0, nbuf - 1);
  if (flip_max_nb_ >= 0) budget = std::min(budget, flip_max_nb_);
  std::vector<char> nbX(F + 1, 0), nbD(F + 1, 0);
  int nb = 0;
  for (const Slot &s : slots) {
    if (nb < budget) {
      (s.d ? nbD : nbX)[s.level] = 1;
      ++nb;
    } else if (s.must) {
      return false;
    }
  }
  ensure_states(half, 1 + nb);
  std::vector<int> freebuf;
  for (int i = nb; i >= 1; --i) freebuf.push_back(i);
  auto alloc = [&]() {
    const int b = freebuf.back();
    freebuf.pop_back();
    return b;
  };
  if (std::getenv("QSIM_DEBUG_TREE")) {
    std::fprintf(stderr, "flip tree half %d m=%d lz=%d M=%d buffers=%d slots:", half, m, lz, M, 1 + nb);
    for (const Slot &s : slots)
      std::fprintf(stderr, " %c%d(%.0f%s)", s.d ? 'D' : 'X', s.level, s.cost,
                   (s.d ? nbD : nbX)[s.level] ? ",own" : ",in place");
    std::fprintf(stderr, "\n");
  }
  // C = T_f X: child f (free fork bits, relative to child 0) of level lev, first sweep s0
  auto sibling = [&](const Level &lev, const ChildSet &cq, uint64_t f, const VState &X) {
    uint64_t zq = 0;
    for (size_t t = 0; t < cq.free.size(); ++t)
      if ((f >> t) & 1u) zq ^= 1ull << lev.cut_bits[cq.free[t]];
    if (!zq) return X;
    const Sweep &s0 = lev.sweeps[0];
    uint64_t tg = 0, sx = 0;
    for (const Gate1 &g : s0.gates) {
      tg |= 1ull << g.bit;
      if (g.kind == 1) sx |= 1ull << g.bit;
    }
    const uint64_t mf = zq & tg;
    Diag phi;
    for (int b = 0; b < 64; ++b) {
      if (!((zq >> b) & 1u)) continue;
      if (!((mf >> b) & 1u)) {
        phi.add_Z(b);  // untargeted: Z commutes with the sweep
      } else if ((sx >> b) & 1u) {
        phi.add_Z(b);  // X^1/2: -Y = flip with phase i (-1)^{x_q}
        phi.ph0 = (phi.ph0 + 2) & 7;
      }
    }
    const Diag post = s0.post.phase_only();
    phi = Diag::merge(phi, Diag::merge(post, post.shift(mf).inverse()));
    VState C;
    C.buf = X.buf;
    C.m = X.m ^ mf;
    C.phi = X.has_phi ? Diag::merge(phi, X.phi.shift(mf)) : phi;
    C.has_phi = true;
    st_.flip_siblings++;
    return C;
  };
  std::function<void(int, const VState &, bool, uint64_t)> node = [&](int l, const VState &V, bool keepV,
                                                                       uint64_t bacc) {
    if (l == M) {
      gather_tree(v, lz, M, pin, states_[V.buf]->ptr, bacc, m, slice, dS, nS, V.m, V.has_phi ? &V.phi : nullptr);
      return;
    }
    const int q = l + 1;
    const Level &lev = hp.levels[q];
    const ChildSet &cq = cs[q];
    const uint64_t nch = 1ull << cq.free.size();
    int xb = V.buf;
    bool xnew = false, xip = false;
    if (keepV) {
      if (nbX[q])
        xb = alloc(), xnew = true;
      else
        xip = true;
    }
    std::vector<Executed> rx;
    flip_exec(first[q], hp.fork_diag(q, cq.base), V, xb, hp, xip ? &rx : nullptr);
    VState X;
    X.buf = xb;
    X.m = V.m;
    for (uint64_t f = 0; f < nch; ++f) {
      const bool keepX = f + 1 < nch || xip;
      const VState C = sibling(lev, cq, f, X);
      const uint64_t bits = bacc | branch_bits(lev, child_of(lev, cq, f), c);
      if (rest[q].empty()) {
        node(q, C, keepX, bits);
        continue;
      }
      int db = xb;
      bool dnew = false, dip = false;
      if (keepX) {
        if (nbD[q])
          db = alloc(), dnew = true;
        else
          dip = true;
      }
      std::vector<Executed> rd;
      flip_exec(rest[q], Diag(), C, db, hp, dip ? &rd : nullptr);
      VState D;
      D.buf = db;
      D.m = C.m;
      node(q, D, dip, bits);
      if (dip) flip_undo(rd, db, hp);
      if (dnew) freebuf.push_back(db);
    }
    if (xip) flip_undo(rx, xb, hp);
    if (xnew) freebuf.push_back(xb);
  };
  VState root;
  root.buf = 0;
  std::vector<const TilePlan *> all0 = first[0];
  all0.insert(all0.end(), rest[0].begin(), rest[0].end());
  flip_exec(all0, Diag(), root, 0, hp, nullptr);
  node(0, root, false, 0);
  return true;
}

// ---------------------------------------------------------------- Pauli frames (tree executor)
// DESIGN.md §5 "Frames".  Every node of the block's tree is a real state (a buffer) seen through a
// frame F = phi . X^m (program.h frame_through): a fork Z^b multiplies the frames of the children,
// and a sweep runs ONCE on the buffer while each node's frame moves through it (F -> G F G^-1).
// Nodes whose frame breaks at a sweep (a T phase met a gate on a flipped qubit) get a buffer of
// their own: the sweep runs conjugated by the frame (flip_exec); nodes whose frame relative to such
// a representative does move through the sweep share it.  The leaves are gathered through their
// frames (x ^ m, phi).  In the App. A.1 circuits a Z inserted after the second cut period mostly
// survives to the last layer, so a 256-branch block needs a handful of real states instead of one
// per branch.  false: not applicable (a free projector fork, a pinned projector after a free fork).
namespace {
struct KeyHash4 {  // FNV-1a over a frame's bit planes and flip (frame basis keys)
  size_t operator()(const std::array<uint64_t, 4> &k) const {
    uint64_t h = 1469598103934665603ull;
    for (uint64_t v : k) h = (h ^ v) * 1099511628211ull;
    return (size_t)h;
  }
};
}  // namespace

bool Engine::run_tree_frames(int half, const TreeVariant &v, const std::vector<int> &pin, int m, void *slice,
                             const uint64_t *dS, int64_t nS, int nbuf) {
  const HalfProgram &hp = v.prog;
  const int F = (int)hp.levels.size() - 1, c = (int)circ_.cuts.size();
  struct Step {
    int level, s;
    std::vector<const TilePlan *> tps;
  };
  std::vector<Step> steps;
  std::vector<int> lstart(F + 1, 0);
  bool free_seen = false;
  for (int l = 0; l <= F; ++l) {
    lstart[l] = (int)steps.size();
    const Level &lev = hp.levels[l];
    const ChildSet cs = child_set(lev, pin);
    for (int j : cs.free)
      if ((lev.pmask >> j) & 1u) return false;  // projector fork: no frames
    if (l >= 1 && free_seen && pinned_diag(lev, pin).pm && !lev.sweeps.empty()) return false;
    if (!cs.free.empty()) free_seen = true;
    if (v.plans[l].empty()) return false;
    const auto &launches = v.plans[l][0];
    for (size_t s = 0; s < lev.sweeps.size(); ++s) {
      Step st;
      st.level = l;
      st.s = (int)s;
      for (const TilePlan &tp : launches) {
        if (!tp.swaps.empty()) return false;
        if (tp.sweep == (int)s) st.tps.push_back(&tp);
      }
      if (st.tps.empty()) return false;
      steps.push_back(st);
    }
  }
  const int nsteps = (int)steps.size();
  struct FNode {  // one term of a leaf: (cr + i ci) F raw
    LinFrame f;
    uint64_t bits = 0;
    double cr = 1.0, ci = 0.0;
    int depth = 0;  // expansions so far
  };
  // a frame that breaks on T / S phases is expanded into a sum of frames (lin_expand_through) while
  // its term has been expanded fewer than expand_depth_ times and the step needs <= 16 terms
  LinFrame xf[16];
  double xc[32];
  // the block's slice rows are accumulated (a leaf may be gathered from several real states)
  check(cudaMemsetAsync(slice, 0, ((size_t)1 << m) * (size_t)nS * amp_, stream_), "zero slice rows");
  std::vector<int> freebuf;  // state buffers beyond the root's, reserved when a split first needs one
  const int extra = std::max(0, std::min(nbuf - 1, flip_max_nb_ >= 0 ? flip_max_nb_ : 64));
  while ((int)states_.size() < 1 + extra) states_.push_back(new DevBuf());
  states_[0]->reserve(state_bytes_);
  for (int i = extra; i >= 1; --i) freebuf.push_back(i);
  const uint64_t rmask = m >= 64 ? ~0ull : ((1ull << m) - 1ull);
  int nreal = 1, nsw = 0;
  auto lin_of = [](const Diag &d, LinFrame &f) {  // f = d . f for a linear diagonal d
    if (d.pm || d.allzero || d.has_cz() || d.nhalf) return false;
    f.add_counts(d.t1, d.t2, d.zm);
    f.ph0 = (f.ph0 + d.ph0) & 7;
    return true;
  };
  std::function<void(int, int, std::vector<FNode> &, bool, Diag)> process = [&](int pos, int raw,
                                                                                std::vector<FNode> &nodes,
                                                                                bool keepRaw, Diag pin_pre) {
    std::vector<Executed> rec;  // in-place sweeps on raw, undone at the end when the caller keeps raw
    Diag tail;  // fixed forks after the last sweep that are no linear frame (a projector): common to the leaves
    for (;; ++pos) {
      for (int l = 1; l <= F; ++l) {
        if (lstart[l] != pos) continue;
        const Level &lev = hp.levels[l];
        const ChildSet cs = child_set(lev, pin);
        const Diag pd = pinned_diag(lev, pin);
        if (!pd.identity()) {
          if (nodes.size() == 1 && nodes[0].f.identity() && pos < nsteps) {
            pin_pre = Diag::merge(pin_pre, pd);  // the real sweep applies it (the root path)
          } else {
            bool lin = true;
            for (FNode &n : nodes) lin = lin_of(pd, n.f) && lin;
            if (!lin) {
              if (pos < nsteps) throw Error(QSIM_EINVAL, "internal: projector fork inside a frame tree");
              tail = Diag::merge(tail, pd);  // after the last sweep: a common factor of the leaves
            }
          }
        }
        const uint64_t bb = branch_bits(lev, cs.base, c);
        for (FNode &n : nodes) n.bits |= bb;
        if (cs.free.empty()) continue;
        std::vector<FNode> out;
        out.reserve(nodes.size() << cs.free.size());
        for (const FNode &n : nodes)
          for (uint64_t f = 0; f < (1ull << cs.free.size()); ++f) {
            FNode x = n;
            for (size_t t = 0; t < cs.free.size(); ++t)
              if ((f >> t) & 1u) x.f.add_Z(lev.cut_bits[cs.free[t]]);
            x.bits |= branch_bits(lev, child_of(lev, cs, f), c) & ~bb;
            out.push_back(x);
          }
        nodes.swap(out);
      }
      if (pos == nsteps) break;
      const Step &st = steps[pos];
      const Sweep &sw = hp.levels[st.level].sweeps[st.s];
      std::vector<FNode> surv, fail;
      surv.reserve(nodes.size());
      for (FNode &n : nodes) {
        if (n.f.identity() || lin_through(sw, n.f)) {
          surv.push_back(n);
          continue;
        }
        const int nt = n.depth < expand_depth_ ? lin_expand_through(sw, n.f, 16, xf, xc) : 0;
        if (nt == 0) {
          fail.push_back(n);
          continue;
        }
        for (int i = 0; i < nt; ++i) {
          FNode x = n;
          x.f = xf[i];
          x.cr = n.cr * xc[2 * i] - n.ci * xc[2 * i + 1];
          x.ci = n.cr * xc[2 * i + 1] + n.ci * xc[2 * i];
          x.depth = n.depth + 1;
          surv.push_back(x);
        }
        nterms_ += nt - 1;
      }
      nodes.clear();
      nodes.shrink_to_fit();
      // classes of the breaking nodes: a member's frame relative to the representative moves through
      struct Cls {
        FNode rep;
        std::vector<FNode> mem;  // frames relative to the representative, moved through the sweep
      };
      std::vector<Cls> cls;
      for (const FNode &n : fail) {
        bool placed = false;
        for (Cls &k : cls) {
          LinFrame rel = lin_compose(n.f, lin_inverse(k.rep.f));
          if (lin_through(sw, rel)) {
            FNode x = n;
            x.f = rel;
            k.mem.push_back(x);
            placed = true;
            break;
          }
        }
        if (!placed) cls.push_back(Cls{n, {}});
      }
      fail.clear();
      if (cls.empty()) {  // every frame moved through: one sweep for all nodes
        VState V;
        V.buf = raw;
        flip_exec(st.tps, pin_pre, V, raw, hp, keepRaw ? &rec : nullptr);
        ++nsw;
        pin_pre = Diag();
        nodes.swap(surv);
        continue;
      }
      // a split: the survivors and every class run the sweep from raw, each into a state of its own.
      // Smaller groups first, into free buffers (else in place, undone afterwards); the largest group
      // (the most splits still to come) last, in place, with the buffers free again for its splits.
      struct Group {
        bool surv;
        LinFrame rep;
        std::vector<FNode> nodes;
      };
      std::vector<Group> groups;
      if (!surv.empty()) groups.push_back(Group{true, LinFrame(), std::move(surv)});
      for (Cls &k : cls) {
        Group g{false, k.rep.f, {}};
        LinFrame flip;
        flip.m = k.rep.f.m;
        g.nodes.reserve(1 + k.mem.size());
        FNode r = k.rep;
        r.f = flip;  // on its new state the representative is X^{m_rep} dst, a member R' X^{m_rep} dst
        g.nodes.push_back(r);
        for (const FNode &x : k.mem) {
          FNode y = x;
          y.f = lin_compose(x.f, flip);
          g.nodes.push_back(y);
        }
        k.mem.clear();
        groups.push_back(std::move(g));
      }
      cls.clear();
      std::stable_sort(groups.begin(), groups.end(),
                       [](const Group &a, const Group &b) { return a.nodes.size() < b.nodes.size(); });
      for (size_t gi = 0; gi < groups.size(); ++gi) {
        Group &g = groups[gi];
        const bool last = gi + 1 == groups.size();
        int dst = raw;
        bool dnew = false, dip = false;
        if (!last) {
          if (!freebuf.empty()) {
            dst = freebuf.back(), freebuf.pop_back(), dnew = true;
            states_[dst]->reserve(state_bytes_);
          } else {
            dip = true;
          }
        } else {
          dip = keepRaw;
        }
        std::vector<Executed> rd;
        VState V;
        V.buf = raw;
        if (!g.surv) {
          V.m = g.rep.m;
          V.phi = g.rep.diag();
          V.has_phi = true;
        }
        flip_exec(st.tps, g.surv ? pin_pre : Diag(), V, dst, hp, dip ? &rd : nullptr);
        if (!g.surv) ++nreal;
        ++nsw;
        process(pos + 1, dst, g.nodes, dip, Diag());
        if (dip) flip_undo(rd, dst, hp);
        if (dnew) freebuf.push_back(dst);
      }
      nodes.clear();
      break;
    }
    if (!nodes.empty()) {  // leaves: batched gathers through their frames, the terms of a leaf summed
      // the distinct flips are gathered once each into rows (coalesced reads for every term after) when
      // they are fewer than the terms and their rows fit; else every term reads the state scattered
      std::unordered_map<uint64_t, uint32_t> fidx;
      std::vector<uint64_t> flips;
      for (const FNode &n : nodes)
        if (fidx.emplace(n.f.m, (uint32_t)flips.size()).second) flips.push_back(n.f.m);
      const size_t rows_bytes = flips.size() * (size_t)nS * amp_;
      size_t free_b = 0, total_b = 0;
      check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
      const bool use_rows = flip_rows_ && flips.size() * 4 <= nodes.size() &&
                            rows_bytes + flips.size() * 8 + ((size_t)1 << 30) <= free_b + flip_rows_buf_.bytes;
      if (std::getenv("QSIM_DEBUG_TREE"))
        std::fprintf(stderr, "frames gather: %zu terms, %zu distinct flips on buffer %d (%s)\n", nodes.size(),
                     flips.size(), raw, use_rows ? "flip rows" : "scattered");
      if (use_rows) {
        flip_rows_buf_.reserve(rows_bytes);
        flip_idx_buf_.reserve(flips.size() * 8);
        upload_async(flip_idx_buf_.ptr, flips.data(), flips.size() * 8);
        check(launch_flip_rows(states_[raw]->ptr, dS, nS, flip_idx_buf_.as<uint64_t>(), (int64_t)flips.size(),
                               flip_rows_buf_.ptr, c128_, stream_),
              "flip rows launch");
        st_.kernel_launches++;
      }
      const DiagDev pend = to_dev(tail);
      std::unordered_map<std::array<uint64_t, 4>, uint32_t, KeyHash4> bidx;  // frame -> basis row
      std::vector<const FNode *> reps;
      if (basis_on_) {  // the distinct frames; more than the basis rows hold: gather the leaves (first point only)
        for (const FNode &n : nodes) {
          if (bidx.emplace(std::array<uint64_t, 4>{n.f.t1, n.f.t2, n.f.zm, n.f.m}, (uint32_t)reps.size()).second)
            reps.push_back(&n);
          if (basis_T_ + (int64_t)reps.size() > basis_cap_) {
            if (basis_points_ > 0) throw BasisAbort();
            basis_on_ = false;
            break;
          }
        }
      }
      if (basis_on_) {
        // basis mode (qsim_evolve_range, DESIGN.md §5 "Frame basis"): every distinct frame (t1, t2, zm, m)
        // becomes ONE gathered row of the basis; each leaf is recorded as its terms' (row, basis, c w^ph0)
        // every gather point (a real state) appends its distinct frames after the rows of the earlier ones
        basis_points_++;
        const int64_t T0 = basis_T_;
        static const double r2 = 0.70710678118654752440;
        static const double W[8][2] = {{1, 0}, {r2, r2}, {0, 1}, {-r2, r2}, {-1, 0}, {-r2, -r2}, {0, -1}, {r2, -r2}};
        basis_entries_.reserve(basis_entries_.size() + nodes.size());
        for (const FNode &n : nodes) {
          const uint32_t tb = bidx.find(std::array<uint64_t, 4>{n.f.t1, n.f.t2, n.f.zm, n.f.m})->second;
          const int ph = n.f.ph0 & 7;
          basis_entries_.push_back(BasisEntry{(uint32_t)(basis_row0_ + (n.bits & rmask)), (uint32_t)(T0 + tb),
                                              n.cr * W[ph][0] - n.ci * W[ph][1], n.cr * W[ph][1] + n.ci * W[ph][0]});
          if (!n.f.identity()) st_.flip_siblings++;
        }
        basis_T_ = T0 + (int64_t)reps.size();
        char *brows = (char *)basis_rows_->ptr + (size_t)T0 * (size_t)nS * amp_;
        check(cudaMemsetAsync(brows, 0, reps.size() * (size_t)nS * amp_, stream_), "zero basis rows");
        FrameBatch fb;
        fb.nleaf = 0;
        fb.off[0] = 0;
        for (size_t t = 0; t < reps.size(); ++t) {
          const FNode &n = *reps[t];
          FrameTerm &T = fb.term[fb.nleaf];
          T.t1 = (uint32_t)n.f.t1;
          T.t2 = (uint32_t)n.f.t2;
          T.zm = (uint32_t)n.f.zm;
          T.m = use_rows ? fidx[n.f.m] : (uint32_t)n.f.m;
          T.ph0 = 0;
          T.pad = 0;
          T.cr = 1.0;
          T.ci = 0.0;
          fb.row[fb.nleaf] = (uint32_t)t;
          fb.off[fb.nleaf + 1] = (uint16_t)(fb.nleaf + 1);
          if (++fb.nleaf == kMaxBatchLeaves || t + 1 == reps.size()) {
            check(launch_frame_gather(use_rows ? flip_rows_buf_.ptr : states_[raw]->ptr, dS, nS, brows, fb, pend, c128_,
                                      stream_, use_rows),
                  "basis gather launch");
            st_.kernel_launches++;
            fb.nleaf = 0;
          }
        }
        if (std::getenv("QSIM_DEBUG_TREE"))
          std::fprintf(stderr, "frame basis: %zu terms over %lld distinct frames\n", nodes.size(), (long long)basis_T_);
        nodes.clear();
      }
      std::stable_sort(nodes.begin(), nodes.end(),
                       [&](const FNode &a, const FNode &b) { return (a.bits & rmask) < (b.bits & rmask); });
      FrameBatch fb;
      fb.nleaf = 0;
      fb.off[0] = 0;
      int nterm = 0;
      auto flush = [&]() {
        if (!fb.nleaf) return;
        check(launch_frame_gather(use_rows ? flip_rows_buf_.ptr : states_[raw]->ptr, dS, nS, slice, fb, pend, c128_,
                                  stream_, use_rows),
              "frame gather launch");
        st_.kernel_launches++;
        fb.nleaf = 0;
        nterm = 0;
      };
      for (size_t a = 0; a < nodes.size();) {
        size_t e = a + 1;
        while (e < nodes.size() && (nodes[e].bits & rmask) == (nodes[a].bits & rmask)) ++e;
        for (size_t s0 = a; s0 < e; s0 += kMaxBatchTerms) {  // a leaf with more terms spans launches
          const size_t s1 = std::min(e, s0 + (size_t)kMaxBatchTerms);
          if (fb.nleaf == kMaxBatchLeaves || nterm + (int)(s1 - s0) > kMaxBatchTerms) flush();
          for (size_t q = s0; q < s1; ++q) {
            const FNode &n = nodes[q];
            if (!n.f.identity()) st_.flip_siblings++;
            FrameTerm &T = fb.term[nterm++];
            T.t1 = (uint32_t)n.f.t1;
            T.t2 = (uint32_t)n.f.t2;
            T.zm = (uint32_t)n.f.zm;
            T.m = use_rows ? fidx[n.f.m] : (uint32_t)n.f.m;
            T.ph0 = n.f.ph0;
            T.pad = 0;
            T.cr = n.cr;
            T.ci = n.ci;
          }
          fb.row[fb.nleaf] = (uint32_t)(nodes[a].bits & rmask);
          fb.off[++fb.nleaf] = (uint16_t)nterm;
        }
        a = e;
      }
      flush();
    }
    if (keepRaw) flip_undo(rec, raw, hp);
  };
  std::vector<FNode> root(1);
  process(0, 0, root, false, Diag());
  if (std::getenv("QSIM_DEBUG_TREE"))
    std::fprintf(stderr, "frames half %d m=%d: %d real states, %d sweeps (+%llu undone), %d steps, %d extra buffers, "
                 "%lld extra terms\n", half, m, nreal, nsw, (unsigned long long)st_.undo_sweeps, nsteps, extra,
                 (long long)nterms_);
  return true;
}

void Engine::run_tree(int half, const TreeVariant &v, int lz, const std::vector<int> &pin, int m, void *slice,
                      const uint64_t *dS, int64_t nS, size_t bfs_avail) {
  (void)half;
  const HalfProgram &hp = v.prog;
  const int F = (int)hp.levels.size() - 1, c = (int)circ_.cuts.size();
  std::vector<int> start(F + 2, 0);
  for (int l = 0; l <= F; ++l) start[l + 1] = start[l] + (int)hp.levels[l].sweeps.size();
  const int Sm = start[F + 1] - lz;
  int M = 0;
  std::vector<int> skip(F + 1, 0);
  for (int l = 0; l <= F; ++l) {
    const int n = (int)hp.levels[l].sweeps.size();
    const int mat = std::max(0, std::min(n, Sm - start[l]));
    if (mat > 0) M = l;
    skip[l] = n - mat;
  }
  for (int l = 0; l <= F; ++l)
    if ((size_t)skip[l] >= v.plans[l].size()) throw Error(QSIM_EINVAL, "internal: lazy tail longer than the plans");
  auto run = [&](int l, const Diag &fork, const void *src, void *dst) {
    const auto &launches = v.plans[l][(size_t)skip[l]];
    for (size_t i = 0; i < launches.size(); ++i)
      launch_plan(launches[i], i == 0 ? fork : Diag(), i == 0, i == 0 ? src : dst, dst, hp, -1, &fork);
  };
  std::function<void(int, int, uint64_t)> node = [&](int l, int bi, uint64_t bacc) {
    if (l == M) {
      gather_tree(v, lz, M, pin, states_[bi]->ptr, bacc, m, slice, dS, nS);
      return;
    }
    if (bfs_avail && bfs_tree(v, lz, M, skip, pin, l, states_[bi]->ptr, bacc, m, slice, dS, nS, bfs_avail)) return;
    const Level &lev = hp.levels[l + 1];
    const ChildSet cs = child_set(lev, pin);
    const int di = cs.free.empty() ? bi : bi + 1;
    for (uint64_t f = 0; f < (1ull << cs.free.size()); ++f) {
      const uint64_t ch = child_of(lev, cs, f);
      run(l + 1, hp.fork_diag(l + 1, ch), states_[bi]->ptr, states_[di]->ptr);
      node(l + 1, di, bacc | branch_bits(lev, ch, c));
    }
  };
  run(0, Diag(), nullptr, states_[0]->ptr);
  node(0, 0, 0);
}

// The leaf of a tree path: the last lz sweeps are evaluated at the sampled indices; the forks of
// the levels that start at a lazy sweep enter that stage's pre diagonal, those of a trailing level
// without sweeps (cuts never targeted again) its post diagonal; one output row per fork value.
void Engine::gather_tree(const TreeVariant &v, int lz, int M, const std::vector<int> &pin, const void *psi,
                         uint64_t bacc, int m, void *slice, const uint64_t *dS, int64_t nS, uint64_t xmask,
                         const Diag *phi) {
  Nvtx nv("leaf gather");
  const HalfProgram &hp = v.prog;
  const int F = (int)hp.levels.size() - 1, c = (int)circ_.cuts.size();
  const uint64_t rmask = m >= 64 ? ~0ull : ((1ull << m) - 1ull);
  auto row = [&](uint64_t b) { return (char *)slice + (size_t)(b & rmask) * (size_t)nS * amp_; };
  const auto st = lazy_stages(hp, lz);
  const int pl = (F > M && hp.levels[F].sweeps.empty()) ? F : -1;
  struct Combo {
    Diag d[2];
    uint64_t bits = 0;
  };
  auto combos = [&](int l0, int l1) {  // fork values of two levels (-1: none)
    std::vector<Combo> out(1);
    const int ls[2] = {l0, l1};
    for (int t = 0; t < 2; ++t) {
      if (ls[t] < 0) continue;
      const Level &lev = hp.levels[ls[t]];
      const ChildSet cs = child_set(lev, pin);
      std::vector<Combo> nx;
      for (const Combo &cb : out)
        for (uint64_t f = 0; f < (1ull << cs.free.size()); ++f) {
          Combo x = cb;
          const uint64_t ch = child_of(lev, cs, f);
          x.d[t] = hp.fork_diag(ls[t], ch);
          x.bits |= branch_bits(lev, ch, c);
          nx.push_back(x);
        }
      out.swap(nx);
    }
    return out;
  };
  auto lazy = [&](const Sweep &sw, const Diag &pre, const Diag &post) {
    LazyLayer ll = lazy_layer(sw, pre);
    ll.post = to_dev(post, true);
    return ll;
  };
  // a sibling-flip state (flip_node): psi read at x ^ xmask, phi joins the first diagonal
  auto with_phi = [&](const Diag &d) { return phi ? Diag::merge(d, *phi) : d; };
  if (lz == 0) {
    for (const Combo &cb : combos(pl, -1)) {
      check(launch_gather(psi, dS, nS, row(bacc | cb.bits), to_dev(with_phi(cb.d[0])), c128_, stream_, ~0ull, 0,
                          xmask),
            "gather launch");
      st_.kernel_launches++;
    }
    return;
  }
  // lz >= 1 stages: index lists deepest first (idx[L-1] = the block; idx[s-1] = the cone of idx[s]
  // over stage s's targets), values of stage s at idx[s] from psi (s = 0) or from stage s-1's values
  // (compact); the forks of a stage's level enter its pre diagonal, the trailing level's its post
  const int L = (int)st.size();
  std::vector<const uint64_t *> idx(L);
  std::vector<int64_t> cnt(L);
  idx[L - 1] = dS;
  cnt[L - 1] = nS;
  // the cone index lists depend only on the stages' target bits and the block: computed once per block
  // (evolve_block invalidates them) and reused by every leaf
  std::vector<uint64_t> key = {(uint64_t)(uintptr_t)dS, (uint64_t)nS, (uint64_t)L};
  for (int s2 = L - 1; s2 >= 1; --s2)
    for (const Gate1 &g : st[s2].first->gates) key.push_back(((uint64_t)s2 << 8) | g.bit);
  const bool reuse = lazy_idx_valid_ && key == lazy_idx_key_;
  for (int s2 = L - 1; s2 >= 1; --s2) {
    const LazyLayer shape = lazy_layer(*st[s2].first, Diag());
    cnt[s2 - 1] = cnt[s2] << shape.k;
    if (!reuse) {
      lazy_idx_[s2 - 1].reserve((size_t)cnt[s2 - 1] * 8);
      check(launch_cone_indices(idx[s2], cnt[s2], shape, lazy_idx_[s2 - 1].as<uint64_t>(), stream_), "cone launch");
      st_.kernel_launches++;
    }
    idx[s2 - 1] = lazy_idx_[s2 - 1].as<uint64_t>();
  }
  lazy_idx_key_ = key;
  lazy_idx_valid_ = true;
  for (int s2 = 0; s2 + 1 < L; ++s2) lazy_val_[s2].reserve((size_t)cnt[s2] * amp_);
  std::function<void(int, uint64_t, const void *)> stage = [&](int s2, uint64_t bits, const void *prev) {
    const Sweep &sw = *st[s2].first;
    const bool last = s2 == L - 1;
    for (const Combo &cb : combos(st[s2].second, last ? pl : -1)) {
      const Diag pre0 = Diag::merge(sw.pre, cb.d[0]);
      LazyLayer ll = lazy(sw, s2 == 0 ? with_phi(pre0) : pre0, last ? Diag::merge(sw.post, cb.d[1]) : sw.post);
      if (s2 == 0) ll.xmask = xmask;
      void *out = last ? (void *)row(bacc | bits | cb.bits) : lazy_val_[s2].ptr;
      if (s2 == 0)
        check(launch_gather_layer(psi, idx[0], cnt[0], out, ll, c128_, stream_), "gather_layer launch");
      else
        check(launch_gather_layer_compact(prev, idx[s2], cnt[s2], out, ll, c128_, stream_),
              "gather_layer_compact launch");
      st_.kernel_launches++;
      if (last)
        st_.lazy_gathers++;
      else
        stage(s2 + 1, bits | cb.bits, lazy_val_[s2].ptr);
    }
  };
  stage(0, 0, nullptr);
}


}  // namespace qsim
