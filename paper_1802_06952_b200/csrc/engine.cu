// Engine: device memory plan, sweep planning and launches, reconstruction, sampling and the NCCL
// reduction of partial blocks; the branch-tree executors are in tree.cu.
#include "engine.h"
#include "engine_internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>

namespace qsim {

// ---------------------------------------------------------------- helpers
void DevBuf::reserve(size_t n) {
  if (n <= bytes && ptr) return;
  release();
  if (n == 0) return;
  cudaError_t e = cudaMalloc(&ptr, n);
  if (e != cudaSuccess) {
    ptr = nullptr;
    bytes = 0;
    (void)cudaGetLastError();
    std::ostringstream m;
    m << "cudaMalloc of " << n << " bytes failed: " << cudaGetErrorString(e);
    throw Error(QSIM_ENOMEM, m.str());
  }
  bytes = n;
}

void DevBuf::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

void Engine::check(cudaError_t e, const char *what) {
  if (e != cudaSuccess) {
    std::ostringstream m;
    m << what << ": " << cudaGetErrorString(e);
    throw Error(e == cudaErrorMemoryAllocation ? QSIM_ENOMEM : QSIM_ECUDA, m.str());
  }
}

DiagDev to_dev(const Diag &d, bool force_active) {
  // the device form holds bits 0..31 (a distributed half's diagonals are restricted to the shard
  // first, Diag::restrict_low); anything above is a planning error, not a result
  if (!d.allzero && !d.below(32)) throw Error(QSIM_EINVAL, "internal: a diagonal above bit 31 reached the device");
  DiagDev o;
  std::memset(&o, 0, sizeof(o));
  o.t1 = (uint32_t)d.t1;
  o.t2 = (uint32_t)d.t2;
  o.zm = (uint32_t)d.zm;
  o.pm = (uint32_t)d.pm;
  o.pv = (uint32_t)(d.pv & d.pm);
  for (int k = 1; k < 32; ++k)
    if (d.cz[k]) {
      o.czd[o.ncz] = (uint8_t)k;
      o.czm[o.ncz++] = (uint32_t)d.cz[k];
    }
  o.ph0 = d.ph0 & 7;
  o.active = (force_active || !d.identity()) ? 1 : 0;
  o.scale = d.scale();
  if (d.allzero) {  // (i & 1) == 2 never holds
    o.pm = 1;
    o.pv = 2;
    o.active = 1;
  }
  return o;
}

// DiagSplit of a diagonal for the register slots at global bit positions regpos
// (slot index bit j <-> regpos[j]); see kernels.h.
static DiagSplit make_split(const Diag &d, const std::vector<int> &regpos) {
  DiagSplit s;
  std::memset(&s, 0, sizeof(s));
  const DiagDev dd = to_dev(d, true);
  uint32_t Rbits = 0;
  for (int p : regpos) Rbits |= 1u << p;
  const int nslots = 1 << regpos.size();
  for (int idx = 0; idx < nslots; ++idx) {
    uint32_t R = 0;
    for (size_t j = 0; j < regpos.size(); ++j)
      if ((idx >> j) & 1) R |= 1u << regpos[j];
    int ph = dd.ph0 + __builtin_popcount(R & dd.t1) + 2 * __builtin_popcount(R & dd.t2) +
             4 * __builtin_popcount(R & dd.zm);
    for (int k = 1; k < 32; ++k) ph += 4 * __builtin_popcount(R & (R >> k) & (uint32_t)d.cz[k]);
    const bool okR = (R & dd.pm & Rbits) == (dd.pv & dd.pm & Rbits);
    s.P[idx] = (uint8_t)((ph & 7) << 3);
    if (!okR) s.notok |= 1u << idx;
  }
  s.has_proj = (dd.pm != 0) ? 1 : 0;
  for (size_t j = 0; j < regpos.size(); ++j) {
    const int p = regpos[j];
    uint32_t N = 0;  // partners of register bit p in CZ pairs
    for (int k = 1; k < 32; ++k) {
      if (((d.cz[k] >> p) & 1u) && p + k < 32) N |= 1u << (p + k);
      if (p >= k && ((d.cz[k] >> (p - k)) & 1u)) N |= 1u << (p - k);
    }
    s.N[j] = N & ~Rbits;
  }
  s.Bpm = dd.pm & ~Rbits;
  s.Bpv = dd.pv & ~Rbits;
  if ((dd.pv & ~dd.pm) & ~Rbits) s.Bpv = dd.pv & ~Rbits;  // allzero encoding: never matches
  return s;
}

static std::vector<int> reg_positions(const TileSweepParams &p, int pass, bool c128) {
  std::vector<int> pos;
  if (!c128) pos.push_back(0);  // the vector bit (c64: 2 amplitudes per 16 bytes)
  for (int s = 0; s < 4; ++s) pos.push_back(p.hb[p.gsel[pass][s]]);
  return pos;
}


// ---------------------------------------------------------------- construction
Engine::Engine(qsim_precision prec, int device) : prec_(prec), device_(device) {
  if (prec != QSIM_C64 && prec != QSIM_C128) throw Error(QSIM_EINVAL, "precision must be QSIM_C64 or QSIM_C128");
  if (device < 0) throw Error(QSIM_EINVAL, "device must be >= 0");
  c128_ = prec == QSIM_C128;
  amp_ = c128_ ? 16 : 8;
  half_.emplace_back();
  half_.emplace_back();
}

Engine::~Engine() {
  for (auto &s : staging_) {
    if (s.ev) cudaEventSynchronize(s.ev), cudaEventDestroy(s.ev);
    if (s.host) cudaFreeHost(s.host);
  }
  staging_.clear();
  if (inited_) {
    cudaSetDevice(device_);
    cudaStreamSynchronize(stream_);
    for (auto &pr : ev_sweep_) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    for (auto &pr : ev_gemm_) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    for (auto e : ev_pool_) cudaEventDestroy(e);
    for (void *p : ipc_opened_) cudaIpcCloseMemHandle(p);
    for (auto *b : states_) delete b;
    states_.clear();
    if (comm_) ncclCommDestroy(comm_);
    if (own_stream_) cudaStreamDestroy(own_stream_);
  }
}

void Engine::upload_async(void *dst, const void *src, size_t bytes) {
  if (!bytes) return;
  Staging *slot = nullptr;
  for (auto &s : staging_)
    if (!s.pending || cudaEventQuery(s.ev) == cudaSuccess) {
      slot = &s;
      break;
    }
  if (!slot) {
    if (staging_.size() < 8) {
      staging_.emplace_back();
      slot = &staging_.back();
      check(cudaEventCreateWithFlags(&slot->ev, cudaEventDisableTiming), "cudaEventCreate");
    } else {
      slot = &staging_.front();
      check(cudaEventSynchronize(slot->ev), "staging wait");
    }
  }
  if (slot->cap < bytes) {
    if (slot->host) cudaFreeHost(slot->host);
    slot->host = nullptr;
    slot->cap = 0;
    check(cudaMallocHost(&slot->host, bytes), "cudaMallocHost");
    slot->cap = bytes;
  }
  std::memcpy(slot->host, src, bytes);
  check(cudaMemcpyAsync(dst, slot->host, bytes, cudaMemcpyHostToDevice, stream_), "upload");
  check(cudaEventRecord(slot->ev, stream_), "cudaEventRecord");
  slot->pending = true;
}

void Engine::ensure_device() {
  if (inited_) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    return;
  }
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    (void)cudaGetLastError();
    throw Error(QSIM_ECUDA, std::string("no CUDA device available: ") +
                                (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
  }
  if (device_ >= n) throw Error(QSIM_EINVAL, "device index out of range");
  check(cudaSetDevice(device_), "cudaSetDevice");
  cudaDeviceProp prop;
  check(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
  if (prop.major != 10) {
    std::ostringstream m;
    m << "this build targets sm_100a (B200); device " << device_ << " is sm_" << prop.major << prop.minor;
    throw Error(QSIM_ECUDA, m.str());
  }
  num_sms_ = prop.multiProcessorCount;
  check(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  if (!stream_) stream_ = own_stream_;
  check(tile_sweep_setup(&occ1_, &occ2_, c128_), "tile sweep setup");
  check(tile_sweep_tma_setup(c128_), "tma sweep setup");
  occ1_ = std::max(occ1_, 1);
  occ2_ = std::max(occ2_, 1);
  inited_ = true;
}

void Engine::set_option(int key, int64_t value) {
  ++plan_gen_;  // compiled multi-part programs depend on the options
  switch (key) {
    case QSIM_OPT_TIME_SWEEPS:
      time_sweeps_ = value != 0;
      return;
    case QSIM_OPT_MODE:
      if (value < 0 || value > 2) throw Error(QSIM_EINVAL, "QSIM_OPT_MODE must be 0, 1 or 2");
      mode_ = (int)value;
      roles_chosen_ = false;
      if (have_circuit_) {
        for (int h = 0; h < 2; ++h) {
          half_[h].uploaded = false;
          compile_plans(half_[h]);
        }
      }
      return;
    case QSIM_OPT_MEM_BUDGET:
      if (value < 0) throw Error(QSIM_EINVAL, "memory budget must be >= 0");
      mem_budget_ = value;
      return;
    case QSIM_OPT_LAZY_LAST:
      if (value < 0 || value > 4) throw Error(QSIM_EINVAL, "QSIM_OPT_LAZY_LAST must be 0 .. 4");
      lazy_depth_ = (int)value;
      return;
    case QSIM_OPT_FUSE_LAYERS:  // multi-layer tiles were compute-bound, never faster: removed
      if (value != 0) throw Error(QSIM_EINVAL, "QSIM_OPT_FUSE_LAYERS: layer fusion was removed; only 0 is accepted");
      return;
    case QSIM_OPT_DISTRIBUTE:
      if (value < 0 || value > 1) throw Error(QSIM_EINVAL, "QSIM_OPT_DISTRIBUTE must be 0 or 1");
      dist_ = value != 0;
      if (have_circuit_) compile_all();
      have_blocks_ = false;  // the sampled indices are relabelled per layout
      return;
    case QSIM_OPT_BFS:
      if (value < 0 || value > 1) throw Error(QSIM_EINVAL, "QSIM_OPT_BFS must be 0 or 1");
      bfs_ = value != 0;
      return;
    case QSIM_OPT_MAX_CTAS:
      if (value < 0 || value > 100000) throw Error(QSIM_EINVAL, "QSIM_OPT_MAX_CTAS must be >= 0");
      max_ctas_ = (int)value;
      return;
    case QSIM_OPT_DEFER:
      if (value < 0 || value > 1) throw Error(QSIM_EINVAL, "QSIM_OPT_DEFER must be 0 or 1");
      deferred_ = value != 0;
      return;
    case QSIM_OPT_FLIP:
      if (value < 0 || value > 1) throw Error(QSIM_EINVAL, "QSIM_OPT_FLIP must be 0 or 1");
      flip_ = value != 0;
      return;
    case QSIM_OPT_FLIP_NB:
      if (value < -1 || value > 64) throw Error(QSIM_EINVAL, "QSIM_OPT_FLIP_NB must be -1 .. 64");
      flip_max_nb_ = (int)value;
      return;
    case QSIM_OPT_SWEEP_KERNEL:
      if (value < 0 || value > 3) throw Error(QSIM_EINVAL, "QSIM_OPT_SWEEP_KERNEL must be 0, 1, 2 or 3");
      sweep_kernel_ = (int)value;
      if (have_circuit_)
        for (int h = 0; h < 2; ++h) compile_plans(half_[h]);
      return;
    default:
      throw Error(QSIM_EINVAL, "unknown option key");
  }
}

void Engine::set_stream(void *s) {
  stream_ = s ? reinterpret_cast<cudaStream_t>(s) : own_stream_;
}

// ---------------------------------------------------------------- circuit
void Engine::load_circuit(uint32_t rows, uint32_t cols, uint32_t depth, const qsim_gate *gates,
                          size_t n_gates, uint32_t cut_row, const uint32_t *cut_layers,
                          size_t n_cut_layers) {
  Circuit c;
  std::string err = build_circuit(rows, cols, depth, gates, n_gates, cut_row, cut_layers, n_cut_layers, c);
  if (!err.empty()) throw Error(QSIM_EINVAL, err);
  circ_ = std::move(c);
  ++plan_gen_;
  compile_all();
  have_circuit_ = true;
  have_blocks_ = false;
  reduced_ = false;
}

void Engine::compile_all() {
  roles_chosen_ = false;
  roles_.clear();
  if (dist_) {
    if (world_ & (world_ - 1) || world_ > 4)
      throw Error(QSIM_EINVAL, "distributed halves need 1, 2 or 4 ranks (qsim_comm_init)");
    gbits_ = world_ == 4 ? 2 : world_ == 2 ? 1 : 0;
  } else {
    gbits_ = 0;
  }
  for (int h = 0; h < 2; ++h) {
    half_[h].prog = compile_half(circ_, h == 0);
    half_[h].uploaded = false;
    compile_plans(half_[h]);
    if (dist_) {
      plan_distributed(half_[h]);
      compile_plans(half_[h]);
    } else if (half_[h].tree && half_[h].prog.h <= 32) {  // relabel qubits to physical bits (choose_perm)
      std::vector<double> lw;
      if (deferred_) lw = deferred_layer_weights(h, perm_ns_[h]);
      // the frame executor gathers the leaves with direct reads (no lazy tail): no gather term
      static const bool frames_w = !(std::getenv("QSIM_PERM_FRAMES") && std::getenv("QSIM_PERM_FRAMES")[0] == '0');
      const bool frame_mode = deferred_ && frames_ && frames_w && flip_half(h);
      const std::vector<int> perm = choose_perm(half_[h], frame_mode ? 0 : perm_ns_[h], deferred_ ? &lw : nullptr);
      bool ident = true;
      for (size_t b = 0; b < perm.size(); ++b) ident = ident && perm[b] == (int)b;
      if (!ident) {
        half_[h].prog = compile_half(circ_, h == 0, perm);
        compile_plans(half_[h]);
      }
    }
  }
}

void Engine::partition(uint32_t *n_cuts, uint64_t *n_branches, qsim_cut *cuts) const {
  if (!have_circuit_) throw Error(QSIM_ESTATE, "no circuit loaded");
  const size_t c = circ_.cuts.size();
  if (c > 63) throw Error(QSIM_EINVAL, "more than 63 cut CZs: 2^c branches do not fit in uint64");
  if (n_cuts) *n_cuts = (uint32_t)c;
  if (n_branches) *n_branches = 1ull << c;
  if (cuts)
    for (size_t g = 0; g < c; ++g) cuts[g] = circ_.cuts[g];
}

// ---------------------------------------------------------------- sweep planning
static void outer_runs(const std::vector<int> &hb, int L, int h, uint8_t *run_start, uint8_t *run_len,
                       int32_t *nruns) {
  int nr = 0;
  for (int b = L; b < h;) {
    if (std::find(hb.begin(), hb.end(), b) != hb.end()) {
      ++b;
      continue;
    }
    int e = b;
    while (e < h && std::find(hb.begin(), hb.end(), e) == hb.end()) ++e;
    run_start[nr] = (uint8_t)b;
    run_len[nr] = (uint8_t)(e - b);
    ++nr;
    b = e;
  }
  *nruns = nr;
}

// The launches of the `n` leading sweeps of a level: one single-layer plan per sweep (a layer wider
// than the tile is split into several launches, legacy_plans).
std::vector<TilePlan> Engine::level_launches(const HalfProgram &hp, const Level &lev, size_t n) {
  std::vector<TilePlan> out;
  for (size_t s = 0; s < n; ++s) {
    auto v = legacy_plans(hp, lev.sweeps[s]);
    for (auto &tp : v) tp.sweep = (int)s;
    out.insert(out.end(), v.begin(), v.end());
  }
  return out;
}

// Tile plans of every level (host only; precision-dependent tile geometry).  The leaf
// level gets one launch list per lazy-tail depth (0, 1, 2 trailing sweeps left out).
void Engine::compile_plans(HalfExec &he) {
  const HalfProgram &hp = he.prog;
  const int L = tile_low_bits(c128_), T = L + kHiBits;
  const bool can_tree = hp.hl >= T, can_small = hp.h <= small_max_h(c128_) && !dist_;
  if (mode_ == 1)
    he.tree = false;
  else if (mode_ == 2)
    he.tree = true;
  else
    he.tree = !can_small || dist_;
  he.plans.clear();
  he.variants.clear();
  he.glayers.clear();
  he.ft.clear();
  if ((he.tree && !can_tree) || (!he.tree && !can_small)) return;  // reported at evolve time
  if (hp.hl > 32) return;  // more than 32 local bits: only the shards of a distributed half are planned
  if (!he.tree) return;
  plan_levels(hp, he.plans, false);
}

void Engine::plan_levels(const HalfProgram &hp, std::vector<std::vector<std::vector<TilePlan>>> &plans,
                         bool all_skips) {
  const size_t F = hp.levels.size() - 1;
  plans.clear();
  plans.resize(hp.levels.size());
  for (size_t l = 0; l <= F; ++l) {
    const Level &lev = hp.levels[l];
    const size_t nskip = (l == F || all_skips) ? 4 : 1;  // lazy tails of up to 3 sweeps
    uint32_t forkmask = 0;
    for (int b : lev.cut_bits) forkmask |= 1u << b;
    for (size_t skip = 0; skip < nskip; ++skip) {
      const size_t n = lev.sweeps.size() - std::min(skip, lev.sweeps.size());
      plans[l].push_back(level_launches(hp, lev, n));
      uint32_t touched = 0;  // a projected fork bit stays fixed until a gate acts on it
      for (TilePlan &tp : plans[l].back()) {
        tp.zfix = forkmask & ~touched;
        touched |= tp.targets;
      }
      if (std::getenv("QSIM_DEBUG_PLANS")) {
        std::fprintf(stderr, "%s level %zu skip %zu: %zu sweeps ->", hp.upper ? "U" : "D", l, skip, n);
        for (auto &tp : plans[l].back())
          std::fprintf(stderr, " [x%d p%d m%d]", tp.layers, tp.npass, tp.p.run_m);
        std::fprintf(stderr, "\n");
      }
    }
  }
}

// Qubit-to-bit relabelling of a tree half (program.h HalfProgram::perm).  A tile sweep is fastest
// when its rows are long: the hi bits of the tile (the layer's targets above the L low bits,
// padded with the lowest free bits) should start at bit L and be consecutive (run of 2^(L+m)
// amplitudes), with few hi targets (> 4 need a second register pass) and few targets on lane
// bits (shuffles).  Speed model from tools/sweep_micro.py on B200 (one layer repeated, GB/s):
// by m = 0..7 about 4940, 5310, 5680, 5930, 5990, 6020, 6040, 6050; a second pass costs ~3 % (c64)
// and, in c128 with 6-7 hi targets, ~30 %; each lane-bit target ~2 % (c64) / 3 % (c128).  The cost
// of a permutation is the sum over the sweeps that run as full passes of (nodes executing the
// sweep) / speed; a seeded local search over transpositions minimises it.
// QSIM_PERM = id | rev | rand | auto (default) for tests.
// Tree nodes running the sweep of each layer in the deferred-fork tree of the whole branch range
// (choose_tree): 2^{#cuts whose fork applies at or before the layer}; 0 for the lazy tail.
std::vector<double> Engine::deferred_layer_weights(int half, int64_t nS) {
  HalfExec &he = half_[half];
  const bool up = half == 0;
  he.glayers = gate_layers(circ_, up ? 0 : circ_.h_u, up ? circ_.h_u : circ_.n);
  he.ft = first_targets(circ_, half_cuts(circ_, up));
  const int c = (int)circ_.cuts.size();
  if (nS <= 0) nS = 4096;
  const int lz = tree_lazy(half, nS);
  // sibling flips: a level's first sweep runs once per parent, its later ones once per child, so the
  // sweep of layer t runs 2^{#forks applied before t} times; else 2^{#forks applied at or before t}
  const bool flip = flip_half(half);
  std::vector<double> w(circ_.depth + 2, 0.0);
  const int S = (int)he.glayers.size();
  static const bool frames_w = !(std::getenv("QSIM_PERM_FRAMES") && std::getenv("QSIM_PERM_FRAMES")[0] == '0');
  if (flip && frames_ && frames_w) {  // the frame executor: every sweep runs once, on the one real state
    for (int i = 0; i < S; ++i) w[he.glayers[i]] = 1.0;
    return w;
  }
  const TreeChoice tc = flip ? flip_choice(half, c) : choose_tree(half, c, lz, nS, 6, true);
  for (int i = 0; i + lz < S; ++i) {
    const int t = he.glayers[i];
    int n = 0;
    for (int g = 0; g < c; ++g) n += flip ? tc.apply[g] < t : tc.apply[g] <= t;
    w[t] = std::ldexp(1.0, n);
  }
  return w;
}

std::vector<int> Engine::choose_perm(const HalfExec &he, int64_t nS, const std::vector<double> *layer_w) const {
  const HalfProgram &hp = he.prog;
  const int h = hp.h, L = tile_low_bits(c128_);
  std::vector<int> perm(h);
  for (int b = 0; b < h; ++b) perm[b] = b;
  const char *mode = std::getenv("QSIM_PERM");
  const std::string m = mode ? mode : "auto";
  if (m == "id") return perm;
  if (m == "rev") {
    for (int b = 0; b < h; ++b) perm[b] = h - 1 - b;
    return perm;
  }
  uint64_t rng = 0x9E3779B97F4A7C15ull ^ (uint64_t)h;
  auto next = [&]() {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return rng;
  };
  if (m == "rand") {
    for (int b = h - 1; b > 0; --b) std::swap(perm[b], perm[(int)(next() % (uint64_t)(b + 1))]);
    return perm;
  }
  // sweeps (target canonical bits) and their execution weights
  struct SW {
    std::vector<int> bits;
    double w;
  };
  std::vector<SW> sws;
  const int F = (int)hp.levels.size() - 1;
  int sbits = 0;
  for (int l = 0; l <= F; ++l) {
    sbits += hp.levels[l].k;
    const auto &sw = hp.levels[l].sweeps;
    const size_t lazy = (l == F && lazy_depth_ > 0) ? std::min<size_t>(2, sw.size() > 0 ? sw.size() - 1 : 0) : 0;
    for (size_t i = 0; i < sw.size(); ++i) {
      if (!layer_w && i + lazy >= sw.size()) continue;
      if (sw[i].gen || sw[i].gates.empty()) continue;
      SW x;
      for (auto &g : sw[i].gates) x.bits.push_back(g.bit);  // identity program: canonical bits
      x.w = layer_w ? (*layer_w)[sw[i].first_layer] : std::ldexp(1.0, sbits);
      if (x.w > 0) sws.push_back(x);
    }
  }
  static const double speed[8] = {4940, 5310, 5680, 5930, 5990, 6020, 6040, 6050};
  const int VB = c128_ ? 0 : 1;
  // lazy-tail gather (nS > 0: the block size is known): per leaf, nS * 2^(k_d) cone points each read
  // the 2^(k_(d-1)) combinations of the earlier lazy layer's targets (depth 2; depth 1: nS points x
  // 2^(k_d)); targets on the bits inside a 32-byte sector share sectors.  Cost in sweep units at ~4400
  // GB/s of random sectors (B200, lazy gather measured in the launch lists).
  int lz = 0;
  std::vector<int> gbits;  // canonical target bits of the gathered layer
  double gpoints = 0.0;
  static const bool gather_term = !(std::getenv("QSIM_PERM_GATHER") && std::getenv("QSIM_PERM_GATHER")[0] == '0');
  if (gather_term && nS > 0 && F >= 1) {
    // the lazy tail (tree_lazy_of: up to three stages, cones of cones): per leaf nS * 2^{sum k_s}
    // reads, at the sampled indices with every lazy target bit varied; a sector serves the reads
    // that differ only in lazy target bits below the sector size
    std::vector<const Sweep *> all;
    for (auto &l : hp.levels)
      for (auto &s : l.sweeps) all.push_back(&s);
    lz = tree_lazy_of(hp, nS);
    if (lz >= 1 && all.size() >= (size_t)lz) {
      int ksum = 0;
      for (size_t s = all.size() - (size_t)lz; s < all.size(); ++s)
        for (auto &x : all[s]->gates) {
          ++ksum;
          if (std::find(gbits.begin(), gbits.end(), (int)x.bit) == gbits.end()) gbits.push_back(x.bit);
        }
      gpoints = (double)nS * std::ldexp(1.0, ksum) * std::ldexp(1.0, sbits);
    }
  }
  const int sector_bits = c128_ ? 1 : 2;
  const double sweep_bytes = 2.0 * std::ldexp(1.0, h) * (double)amp_;
  auto cost = [&](const std::vector<int> &p) {
    double c = 0;
    for (const SW &x : sws) {
      std::vector<int> hi;
      int nlane = 0;
      for (int b : x.bits) {
        if (p[b] >= L)
          hi.push_back(p[b]);
        else if (p[b] >= VB)
          ++nlane;
      }
      std::sort(hi.begin(), hi.end());
      const size_t nch = std::max<size_t>(1, (hi.size() + kHiBits - 1) / kHiBits);
      for (size_t ci = 0; ci < nch; ++ci) {
        std::vector<int> hb;
        for (size_t i = 0; i < hi.size(); ++i)
          if (i * nch / std::max<size_t>(1, hi.size()) == ci) hb.push_back(hi[i]);
        for (int b = L; (int)hb.size() < kHiBits && b < h; ++b)
          if (std::find(hb.begin(), hb.end(), b) == hb.end()) hb.push_back(b);
        int mm = 0;
        while (mm < kHiBits && std::find(hb.begin(), hb.end(), L + mm) != hb.end()) ++mm;
        const size_t k = hi.size() / nch;
        double v = speed[std::min(mm, 7)];
        if (k > 4) v *= c128_ ? (k > 5 ? 0.70 : 0.96) : 0.97;
        if (ci == 0) v *= 1.0 - (c128_ ? 0.03 : 0.02) * nlane;
        c += x.w / v;
      }
    }
    if (!gbits.empty()) {
      int in_sector = 0;
      for (int b : gbits) in_sector += p[b] < sector_bits;
      const double sectors = gpoints * std::ldexp(1.0, -in_sector);
      c += sectors * 32.0 / sweep_bytes / 4400.0;
    }
    return c;
  };
  static const int iters = std::getenv("QSIM_PERM_ITERS") ? std::atoi(std::getenv("QSIM_PERM_ITERS")) : 6000;
  static const int restarts = std::getenv("QSIM_PERM_RESTARTS") ? std::atoi(std::getenv("QSIM_PERM_RESTARTS")) : 1;
  std::vector<int> best = perm;
  double bc = cost(best);
  for (int r = 0; r < std::max(1, restarts); ++r) {
    std::vector<int> cur = perm;
    double cc = cost(cur);
    for (int it = 0; it < iters; ++it) {
      std::vector<int> q = cur;
      const int i = (int)(next() % (uint64_t)h), j = (int)(next() % (uint64_t)h);
      if (i == j) continue;
      std::swap(q[i], q[j]);
      const double c = cost(q);
      if (c <= cc) {
        cur = q;
        cc = c;
      }
    }
    if (cc < bc) best = cur, bc = cc;
  }
  if (std::getenv("QSIM_DEBUG_PERM"))
    std::fprintf(stderr, "choose_perm h=%d nS=%lld cost %.6g (identity %.6g)\n", h, (long long)nS, bc, cost(perm));
  return best;
}

// Layout schedule of a distributed half (§2.3.3).  Physical bits
// hl .. h-1 are global (the rank); a sweep can only target local bits.  Walking the sweeps in
// tree order (every node of a level runs the same sweeps, so the layout sequence is linear),
// a sweep with a target on a global bit gets it swapped, at the output of the previous sweep,
// with a local bit that is not in that sweep's tile (an outer bit of its tiles) and not a target
// of either sweep; the evicted qubit is the one needed again the latest (Belady).  The initial
// layout puts on the global bits qubits not targeted by the first two sweeps.  Every layer is
// then compiled in the layout of the sweep that applies it.
void Engine::plan_distributed(HalfExec &he) {
  const HalfProgram id = he.prog;  // canonical layout: gate bit == canonical bit
  const int h = id.h, g = gbits_, hl = h - g, L = tile_low_bits(c128_), T = L + kHiBits;
  if (hl < T + 2) {
    std::ostringstream m;
    m << "distributed half: a " << h << "-qubit half over " << (1 << g) << " ranks leaves " << hl
      << " local qubits; need >= " << T + 2;
    throw Error(QSIM_EINVAL, m.str());
  }
  struct SQ {
    int level, idx;
    std::vector<int> tq;
    bool gen;
    int first, last;
  };
  std::vector<SQ> seq;
  for (size_t l = 0; l < id.levels.size(); ++l)
    for (size_t i = 0; i < id.levels[l].sweeps.size(); ++i) {
      const Sweep &sw = id.levels[l].sweeps[i];
      SQ x{(int)l, (int)i, {}, sw.gen, sw.first_layer, sw.last_layer};
      for (auto &gt : sw.gates) x.tq.push_back(gt.bit);
      seq.push_back(x);
    }
  const size_t n = seq.size();
  auto is_target = [&](size_t s, int q) { return std::find(seq[s].tq.begin(), seq[s].tq.end(), q) != seq[s].tq.end(); };
  auto next_use = [&](int q, size_t from) {
    for (size_t s = from; s < n; ++s)
      if (is_target(s, q)) return s;
    return n + 1;
  };
  std::vector<int> cur(h), at(h);  // canonical bit -> position, position -> canonical bit
  for (int b = 0; b < h; ++b) cur[b] = at[b] = b;
  auto put = [&](int q, int pos) {  // exchange the positions of qubit q and the qubit at pos
    const int o = at[pos], pq = cur[q];
    cur[q] = pos;
    at[pos] = q;
    cur[o] = pq;
    at[pq] = o;
  };
  // initial global qubits: not targeted by the first two sweeps, latest first use
  {
    std::vector<int> cand;
    for (int q = 0; q < h; ++q)
      if (!(n > 0 && is_target(0, q)) && !(n > 1 && is_target(1, q))) cand.push_back(q);
    // QSIM_DIST_STRESS (tests): the earliest-needed qubits instead, so that swaps happen early
    const bool stress = std::getenv("QSIM_DIST_STRESS") != nullptr;
    std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) {
      return stress ? next_use(a, 0) < next_use(b, 0) : next_use(a, 0) > next_use(b, 0);
    });
    if ((int)cand.size() < g) throw Error(QSIM_EINVAL, "distributed half: no global qubit placement");
    for (int j = 0; j < g; ++j) put(cand[j], hl + j);
  }
  std::vector<std::vector<int>> sperm(n);
  std::vector<std::vector<std::pair<int, int>>> sswap(n);
  for (size_t s = 0; s < n; ++s) {
    std::vector<int> need;
    for (int q : seq[s].tq)
      if (cur[q] >= hl) need.push_back(q);
    if (!need.empty()) {
      if (s == 0 || seq[s - 1].gen) throw Error(QSIM_EINVAL, "distributed half: swap after the generated sweep");
      const size_t pv = s - 1;
      // bits of the previous sweep's tiles: its hi targets and (a superset of) their padding,
      // the lowest free bits >= L; the swapped bit must be an outer bit of those tiles
      std::vector<int> tile;
      for (int q : seq[pv].tq)
        if (cur[q] >= L) tile.push_back(cur[q]);
      for (int pos = L, pad = 0; pos < hl && pad < kHiBits; ++pos)
        if (std::find(tile.begin(), tile.end(), pos) == tile.end()) {
          tile.push_back(pos);
          ++pad;
        }
      std::vector<int> used;
      for (int q : need) {
        const int G = cur[q];
        int best = -1;
        size_t bu = 0;
        for (int pos = L; pos < hl; ++pos) {
          const int v = at[pos];
          if (is_target(pv, v) || is_target(s, v)) continue;
          if (std::find(tile.begin(), tile.end(), pos) != tile.end()) continue;
          if (std::find(used.begin(), used.end(), pos) != used.end()) continue;
          const size_t u = next_use(v, s);
          if (best < 0 || u > bu) {
            best = pos;
            bu = u;
          }
        }
        if (best < 0) throw Error(QSIM_EINVAL, "distributed half: no local qubit to swap out");
        sswap[pv].push_back({best, G - hl});
        used.push_back(best);
        put(q, best);  // q becomes local at `best`, the evicted qubit global at G
      }
    }
    sperm[s] = cur;
  }
  // layouts per layer: the sweep that applies the layer (pending diagonals: the level's first)
  std::vector<std::vector<int>> layer_perm(circ_.depth + 2, sperm.empty() ? cur : sperm[0]);
  for (size_t l = 0; l < id.levels.size(); ++l) {
    const int first = (l == 0) ? 1 : id.levels[l].fork_layer + 1;
    const int last = (l + 1 < id.levels.size()) ? id.levels[l + 1].fork_layer : (int)circ_.depth;
    size_t s0 = n;
    for (size_t s = 0; s < n; ++s)
      if (seq[s].level == (int)l) {
        s0 = s;
        break;
      }
    for (int t = first; t <= last; ++t) {
      size_t sw = s0;
      for (size_t s = s0; s < n && seq[s].level == (int)l; ++s)
        if (seq[s].first <= t && t <= seq[s].last) sw = s;
      if (sw < n) layer_perm[t] = sperm[sw];
    }
    if (first <= (int)circ_.depth + 1 && s0 < n) layer_perm[first] = sperm[s0];
  }
  layer_perm[circ_.depth + 1] = cur;
  HalfProgram hp = compile_half_layers(circ_, id.upper, layer_perm, cur);
  hp.hl = hl;
  if (std::getenv("QSIM_DEBUG_PLANS")) {
    std::fprintf(stderr, "%s distributed h=%d hl=%d:", id.upper ? "U" : "D", h, hl);
    for (size_t k = 0; k < n; ++k)
      if (!sswap[k].empty()) std::fprintf(stderr, " L%d.%d x%zu", seq[k].level, seq[k].idx, sswap[k].size());
    std::fprintf(stderr, " (%zu sweeps)\n", n);
  }
  size_t s = 0;
  for (auto &lev : hp.levels)
    for (auto &sw : lev.sweeps) {
      sw.swaps = sswap[s++];
      for (auto &gt : sw.gates)
        if (gt.bit >= hl) throw Error(QSIM_EINVAL, "distributed half: a target left on a global bit");
    }
  he.prog = hp;
}

// Legacy per-sweep plans (register-only kernel; the generated root sweep).
std::vector<TilePlan> Engine::legacy_plans(const HalfProgram &hp, const Sweep &sw) {
  std::vector<TilePlan> out;
  const int L = tile_low_bits(c128_), T = L + kHiBits;
  {
    {
      std::vector<Gate1> low, high;
      for (auto &g : sw.gates) (g.bit < L ? low : high).push_back(g);
      const int nchunks = std::max<int>(1, (int)((high.size() + kHiBits - 1) / kHiBits));
      std::vector<std::vector<Gate1>> chunks(nchunks);
      for (size_t i = 0; i < high.size(); ++i) chunks[i * nchunks / high.size()].push_back(high[i]);
      for (int ci = 0; ci < nchunks; ++ci) {
        TilePlan tp;
        std::memset(&tp.p, 0, sizeof(tp.p));
        const auto &H = chunks[ci];
        std::vector<int> hb;
        for (auto &g : H) hb.push_back(g.bit);
        for (int b = L; (int)hb.size() < kHiBits && b < hp.hl; ++b)
          if (std::find(hb.begin(), hb.end(), b) == hb.end()) hb.push_back(b);
        std::sort(hb.begin(), hb.end());
        auto idx_of = [&](int bit) { return (int)(std::find(hb.begin(), hb.end(), bit) - hb.begin()); };
        auto kind_of = [&](int bit) {
          for (auto &g : H)
            if (g.bit == bit) return (int)g.kind;
          return 0;
        };
        for (int j = 0; j < kHiBits; ++j) tp.p.hb[j] = (uint8_t)hb[j];
        tp.npass = H.size() <= 4 ? 1 : 2;
        std::vector<int> tgt_idx;
        for (auto &g : H) tgt_idx.push_back(idx_of(g.bit));
        for (int q = 0; q < tp.npass; ++q) {
          std::vector<int> regs;
          const size_t from = q * 4, to = std::min(H.size(), (size_t)(q * 4 + 4));
          for (size_t i = from; i < to; ++i) regs.push_back(tgt_idx[i]);
          const size_t ntgt = regs.size();
          for (int j = 0; j < kHiBits && regs.size() < 4; ++j) {
            const bool is_tgt = std::find(tgt_idx.begin(), tgt_idx.end(), j) != tgt_idx.end();
            if (!is_tgt && std::find(regs.begin(), regs.end(), j) == regs.end()) regs.push_back(j);
          }
          for (int j = 0; j < kHiBits && regs.size() < 4; ++j)
            if (std::find(regs.begin(), regs.end(), j) == regs.end()) regs.push_back(j);
          std::vector<int> warps;
          for (int j = 0; j < kHiBits; ++j)
            if (std::find(regs.begin(), regs.end(), j) == regs.end()) warps.push_back(j);
          for (int s4 = 0; s4 < 4; ++s4) {
            tp.p.gsel[q][s4] = (uint8_t)regs[s4];
            tp.p.gkind[q][s4] = (uint8_t)((size_t)s4 < ntgt ? kind_of(hb[regs[s4]]) : 0);
          }
          for (int s3 = 0; s3 < 3; ++s3) tp.p.wsel[q][s3] = (uint8_t)warps[s3];
        }
        if (ci == 0)
          for (auto &g : low) tp.p.lowkind[g.bit] = g.kind;
        {
          const int VB = c128_ ? 0 : 1;
          for (int b = VB; b < VB + 5; ++b)
            if (tp.p.lowkind[b]) {
              tp.p.lane_bit[tp.p.n_lane] = (uint8_t)(b - VB);
              tp.p.lane_kind[tp.p.n_lane] = tp.p.lowkind[b];
              tp.p.n_lane++;
            }
        }
        // outer runs
        int nr = 0;
        for (int b = L; b < hp.hl;) {
          if (std::find(hb.begin(), hb.end(), b) != hb.end()) {
            ++b;
            continue;
          }
          int e = b;
          while (e < hp.hl && std::find(hb.begin(), hb.end(), e) == hb.end()) ++e;
          tp.p.run_start[nr] = (uint8_t)b;
          tp.p.run_len[nr] = (uint8_t)(e - b);
          ++nr;
          b = e;
        }
        tp.p.nruns = nr;
        tp.p.log2_ntiles = hp.hl - T;
        tp.targets = 0;
        for (auto &g : H) {
          tp.targets |= 1u << g.bit;
          if (g.kind == 2) tp.sy_targets |= 1u << g.bit;
        }
        if (ci == 0)
          for (auto &g : low) {
            tp.targets |= 1u << g.bit;
            if (g.kind == 2) tp.sy_targets |= 1u << g.bit;
          }
        tp.layers = ci == nchunks - 1 ? 1 : 0;
        if (ci == nchunks - 1) tp.swaps = sw.swaps;
        tp.use_pre = ci == 0;
        tp.gen = sw.gen && ci == 0;
        tp.pre = sw.pre;
        Diag post = ci == nchunks - 1 ? sw.post : Diag();
        if (dist_) post = post.restrict_low(hp.hl, (uint64_t)rank_ << hp.hl);  // this rank's shard
        tp.post = post;
        tp.p.post = to_dev(post);
        tp.p.post_s = make_split(post, reg_positions(tp.p, tp.npass - 1, c128_));
        int m = 0;
        while (m < kHiBits && hb[m] == L + m) ++m;
        tp.p.run_m = m;
        out.push_back(tp);
      }
    }
  }
  return out;
}

void Engine::upload_small(HalfExec &he) {
  if (he.uploaded) return;
  const HalfProgram &hp = he.prog;
  std::vector<SmallLevelDev> levs(hp.levels.size());
  std::vector<SmallSweepDev> sws;
  for (size_t l = 0; l < hp.levels.size(); ++l) {
    const Level &lev = hp.levels[l];
    SmallLevelDev d;
    std::memset(&d, 0, sizeof(d));
    d.k = lev.k;
    d.first_sweep = (int)sws.size();
    d.nsweeps = (int)lev.sweeps.size();
    for (int j = 0; j < lev.k; ++j) d.cut_bits[j] = (uint8_t)lev.cut_bits[j];
    d.pmask = lev.pmask;
    levs[l] = d;
    for (auto &sw : lev.sweeps) {
      SmallSweepDev s;
      std::memset(&s, 0, sizeof(s));
      s.pre = to_dev(sw.pre, sw.gen);
      s.post = to_dev(sw.post);
      s.gen = sw.gen ? 1 : 0;
      s.ngates = (int)sw.gates.size();
      for (size_t g = 0; g < sw.gates.size(); ++g) {
        s.bit[g] = sw.gates[g].bit;
        s.kind[g] = sw.gates[g].kind;
      }
      sws.push_back(s);
    }
  }
  he.d_levels.reserve(levs.size() * sizeof(SmallLevelDev));
  he.d_sweeps.reserve(std::max<size_t>(1, sws.size()) * sizeof(SmallSweepDev));
  check(cudaMemcpyAsync(he.d_levels.ptr, levs.data(), levs.size() * sizeof(SmallLevelDev),
                        cudaMemcpyHostToDevice, stream_),
        "upload small program");
  if (!sws.empty())
    check(cudaMemcpyAsync(he.d_sweeps.ptr, sws.data(), sws.size() * sizeof(SmallSweepDev),
                          cudaMemcpyHostToDevice, stream_),
          "upload small program");
  check(cudaStreamSynchronize(stream_), "upload small program");
  he.uploaded = true;
}

// ---------------------------------------------------------------- blocks
static void validate_block(const uint64_t *v, size_t n, uint32_t h, const char *name) {
  if (n == 0 || !v) throw Error(QSIM_EINVAL, std::string(name) + " block is empty");
  std::vector<uint64_t> s(v, v + n);
  const uint64_t lim = h >= 64 ? ~0ull : (1ull << h);
  for (uint64_t x : s)
    if (x >= lim) {
      std::ostringstream m;
      m << name << " block index " << x << " >= 2^" << h;
      throw Error(QSIM_EINVAL, m.str());
    }
  std::sort(s.begin(), s.end());
  if (std::adjacent_find(s.begin(), s.end()) != s.end())
    throw Error(QSIM_EINVAL, std::string(name) + " block has duplicate indices");
}

void Engine::set_blocks(const uint64_t *up, size_t nu, const uint64_t *lo, size_t nl) {
  if (!have_circuit_) throw Error(QSIM_ESTATE, "no circuit loaded");
  validate_block(up, nu, circ_.h_u, "upper");
  validate_block(lo, nl, circ_.h_l, "lower");
  if (!dist_ && (perm_ns_[0] != (int64_t)nu || perm_ns_[1] != (int64_t)nl)) {
    // the relabelling weighs the lazy-tail gathers by the block sizes: re-plan for these sizes
    perm_ns_[0] = (int64_t)nu;
    perm_ns_[1] = (int64_t)nl;
    compile_all();
  }
  ensure_device();
  Su_.assign(up, up + nu);
  Sl_.assign(lo, lo + nl);
  d_Su_.reserve(nu * 8);
  d_Sl_.reserve(nl * 8);
  check(cudaMemcpyAsync(d_Su_.ptr, up, nu * 8, cudaMemcpyHostToDevice, stream_), "upload S_u");
  check(cudaMemcpyAsync(d_Sl_.ptr, lo, nl * 8, cudaMemcpyHostToDevice, stream_), "upload S_l");
  for (int h = 0; h < 2; ++h) {
    const std::vector<uint64_t> &S = h == 0 ? Su_ : Sl_;
    std::vector<uint64_t> P(S.size());
    for (size_t i = 0; i < S.size(); ++i) P[i] = half_[h].prog.phys(S[i]);
    d_Sp_[h].reserve(P.size() * 8);
    check(cudaMemcpyAsync(d_Sp_[h].ptr, P.data(), P.size() * 8, cudaMemcpyHostToDevice, stream_), "upload S");
    check(cudaStreamSynchronize(stream_), "upload S");  // P is a temporary
  }
  roles_chosen_ = false;  // the lazy tail, hence the fork placement, depends on the block sizes
  A_acc_.reserve(nu * nl * 16);
  check(cudaMemsetAsync(A_acc_.ptr, 0, nu * nl * 16, stream_), "zero block");
  check(cudaStreamSynchronize(stream_), "set_blocks");
  have_blocks_ = true;
  reduced_ = false;
}

void Engine::check_blocks(const uint64_t *up, size_t nu, const uint64_t *lo, size_t nl) const {
  if (!have_blocks_) throw Error(QSIM_ESTATE, "no blocks set / evolved");
  if (up && (nu != Su_.size() || !std::equal(Su_.begin(), Su_.end(), up)))
    throw Error(QSIM_ESTATE, "upper block differs from the evolved one");
  if (lo && (nl != Sl_.size() || !std::equal(Sl_.begin(), Sl_.end(), lo)))
    throw Error(QSIM_ESTATE, "lower block differs from the evolved one");
}

void Engine::reset_block() {
  if (!have_blocks_) throw Error(QSIM_ESTATE, "no blocks set");
  ensure_device();
  check(cudaMemsetAsync(A_acc_.ptr, 0, Su_.size() * Sl_.size() * 16, stream_), "zero block");
  reduced_ = false;
}

// ---------------------------------------------------------------- events
cudaEvent_t Engine::get_event() {
  if (!ev_pool_.empty()) {
    cudaEvent_t e = ev_pool_.back();
    ev_pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  check(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

void Engine::resolve_events() {
  auto drain = [&](std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, double &ms, uint64_t *cnt) {
    if (v.empty()) return;
    check(cudaEventSynchronize(v.back().second), "cudaEventSynchronize");
    for (auto &pr : v) {
      float t = 0.f;
      check(cudaEventElapsedTime(&t, pr.first, pr.second), "cudaEventElapsedTime");
      ms += t;
      if (cnt) ++*cnt;
      ev_pool_.push_back(pr.first);
      ev_pool_.push_back(pr.second);
    }
    v.clear();
  };
  drain(ev_sweep_, st_.sweep_ms, &st_.timed_sweeps);
  drain(ev_gemm_, st_.gemm_ms, nullptr);
}

// ---------------------------------------------------------------- executor
// Shared-memory stages of the TMA sweep (QSIM_OPT_SWEEP_KERNEL 0): two 64 KB stages, or three for
// tiles of short runs (< 4 KB: more, smaller requests in flight per byte).  QSIM_TMA_STAGE_RULE
// (A/B only): 0 = always two, 1 = short runs or two passes, 2 = short runs (default), 3 = two passes.
int Engine::tma_stages(const TilePlan &tp) const {
  static const int rule = std::getenv("QSIM_TMA_STAGE_RULE") ? std::atoi(std::getenv("QSIM_TMA_STAGE_RULE")) : 2;
  if (rule == 1) return (tp.p.run_m < 3 || tp.npass == 2) ? 3 : 2;
  if (rule == 2) return tp.p.run_m < 3 ? 3 : 2;
  if (rule == 3) return tp.npass == 2 ? 3 : 2;
  return 2;
}

void Engine::launch_plan(const TilePlan &tp, const Diag &fork, bool first, const void *src, void *dst,
                         const HalfProgram &hp, int out_buf, const Diag *child_fork, const Diag *pre_ov,
                         const Diag *post_ov) {
  const int h = hp.hl;
  int pre_mode = 0;
  Diag pre;
  TileSweepParams p = tp.p;
  // pre_ov / post_ov (sibling-flip executor): the complete pre / post diagonals of this launch
  const bool use_pre = tp.use_pre || pre_ov;
  // a fork bit this launch targets is applied inside its gate (gate kind k + 2 f, sweep_tma.cu)
  // instead of through the pre diagonal: a Z^b or P_b fork then costs no per-element multiply
  uint32_t absorbed_pm = 0, absorbed_pv = 0;
  Diag fk = pre_ov ? *pre_ov : fork;
  if (use_pre && absorb_ && !tp.gen && sweep_kernel_ != 1 && !dist_ && !fk.allzero) {
    const Diag &fork = fk;
    const int L = tile_low_bits(c128_), VB = c128_ ? 0 : 1;
    const uint32_t cand = (uint32_t)((fork.pm ^ fork.zm) & (fork.pm | fork.zm) & tp.targets & ~(fork.t1 | fork.t2));
    for (int q = 0; q < 32; ++q) {
      if (!((cand >> q) & 1u)) continue;
      const uint64_t m = 1ull << q;
      const int f = (fork.pm & m) ? ((fork.pv & m) ? 3 : 2) : 1;
      uint8_t *k = nullptr;
      if (q >= L) {
        for (int j = 0; j < kHiBits && !k; ++j)
          if (p.hb[j] == q)
            for (int ps = 0; ps < tp.npass && !k; ++ps)
              for (int s4 = 0; s4 < 4 && !k; ++s4)
                if (p.gsel[ps][s4] == j && p.gkind[ps][s4]) k = &p.gkind[ps][s4];
      } else if (VB && q == 0) {
        if (p.lowkind[0]) k = &p.lowkind[0];
      } else {
        for (int i = 0; i < p.n_lane && !k; ++i)
          if (p.lane_bit[i] == q - VB) k = &p.lane_kind[i];
      }
      if (!k || *k > 2) continue;
      *k = (uint8_t)(*k + 2 * f);
      if (f == 1) {
        fk.zm &= ~m;
      } else {
        fk.pm &= ~m;
        fk.pv &= ~m;
        absorbed_pm |= (uint32_t)m;
        if (f == 3) absorbed_pv |= (uint32_t)m;
      }
    }
  }
  if (use_pre) {
    pre = pre_ov ? fk : Diag::merge(fk, tp.pre);
    if (dist_) pre = pre.restrict_low(hp.hl, (uint64_t)rank_ << hp.hl);  // this rank's shard
    if (tp.gen)
      pre_mode = 2;
    else if (!pre.identity())
      pre_mode = 1;
  }
  const bool timed = time_sweeps_;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    e0 = get_event();
    e1 = get_event();
    check(cudaEventRecord(e0, stream_), "cudaEventRecord");
  }
  skip_pm_last_ = 0;
  {
    p.no_pskip = pskip_ ? 0 : 1;
    p.pre = to_dev(pre, pre_mode != 0);
    p.ld_pm = (pre_mode == 1 ? p.pre.pm : 0u) | absorbed_pm;
    p.ld_pv = (pre_mode == 1 ? p.pre.pv : 0u) | absorbed_pv;
    p.njobs = 1;
    if (dist_) {
      p.gbase = 0;  // the diagonals were restricted to this rank's shard on the host
      p.rank = (uint32_t)rank_;
      if (!tp.swaps.empty()) {  // fused local/global swap: destination buffers of the ranks
        if (out_buf < 0 || tp.swaps.size() > 2) throw Error(QSIM_EINVAL, "distributed swap plan");
        p.nswap = (int)tp.swaps.size();
        for (size_t j = 0; j < tp.swaps.size(); ++j) {
          p.swap_l[j] = (uint8_t)tp.swaps[j].first;
          p.swap_j[j] = (uint8_t)tp.swaps[j].second;
        }
        for (int d = 0; d < (1 << gbits_); ++d) p.peer[d] = peer_[out_buf][rank_ ^ d];
      }
    }
    p.src[0] = tp.gen ? nullptr : src;
    p.dst[0] = dst;
    p.job_pv[0] = p.pre.pv;
    p.job_zm[0] = p.pre.zm;
    if (child_fork && zero_skip_ && !dist_ && !tp.gen && child_fork->pm && !child_fork->allzero) {
      // tiles outside the fork's projector (on qubits no gate of the level has touched) are zero
      uint32_t outer = (h >= 32 ? ~0u : ((1u << h) - 1u)) & ~((1u << tile_low_bits(c128_)) - 1u);
      for (int j = 0; j < kHiBits; ++j) outer &= ~(1u << p.hb[j]);
      p.skip_pm = (uint32_t)child_fork->pm & tp.zfix & outer;
      p.skip_pv = (uint32_t)child_fork->pv & p.skip_pm;
    }
    skip_pm_last_ = p.skip_pm;
    if (post_ov) {
      p.post = to_dev(*post_ov);
      p.post_s = make_split(*post_ov, reg_positions(p, tp.npass - 1, c128_));
    }
    const uint64_t tiles = 1ull << p.log2_ntiles;
    const bool tma = (sweep_kernel_ != 1 || p.nswap) && (pre_mode != 2 || (gen_tma_ && !dist_));
    if (tma) {
      if (pre_mode >= 1) p.pre_s = make_split(pre, reg_positions(p, 0, c128_));
      const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)grid_ctas());
      const int stages = sweep_kernel_ == 2 ? 2 : sweep_kernel_ == 3 ? 3 : tma_stages(tp);
      check(launch_tile_sweep_tma(p, c128_, pre_mode, tp.npass, grid, stream_, stages),
            "tma sweep launch");
    } else {
      const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)num_sms_ * (tp.npass == 1 ? occ1_ : occ2_));
      check(launch_tile_sweep(p, c128_, pre_mode, tp.npass, grid, stream_), "tile sweep launch");
    }
  }
  if (timed) {
    check(cudaEventRecord(e1, stream_), "cudaEventRecord");
    ev_sweep_.emplace_back(e0, e1);
    if (ev_sweep_.size() > 8192) resolve_events();
  }
  (void)first;
  st_.kernel_launches++;
  st_.sweeps++;
  st_.sweep_states += 1;
  st_.layers_applied += (uint64_t)tp.layers;
  const double state = std::ldexp(1.0, h) * (double)amp_;
  st_.sweep_bytes += (tp.gen ? 1.0 : 2.0) * state;
  // reads of known-zero tiles (a fraction 1 - 2^-popc(skip_pm) of the tiles) are not issued
  const double skipped = tp.gen ? 0.0 : 1.0 - std::ldexp(1.0, -__builtin_popcount(skip_pm_last_));
  st_.sweep_bytes_moved += ((tp.gen ? 1.0 : 2.0) - skipped) * state;
}

// Runs the sweeps of `level` for fork child `child`, all but the last `skip` of them
// (the lazily evaluated tail); returns where the state ended (src when no sweep ran).
const void *Engine::run_level(int half, int level, uint64_t child, const void *src, void *dst, int skip) {
  HalfExec &he = half_[half];
  const Diag fork = he.prog.fork_diag(level, child);
  const auto &launches = he.plans[level][std::min<size_t>((size_t)skip, he.plans[level].size() - 1)];
  const size_t n = launches.size();
  for (size_t i = 0; i < n; ++i)
    launch_plan(launches[i], i == 0 ? fork : Diag(), i == 0, i == 0 ? src : dst, dst, he.prog, -1, &fork);
  return n ? dst : src;
}

LazyLayer lazy_layer(const Sweep &sw, const Diag &pre) {
  LazyLayer ll;
  std::memset(&ll, 0, sizeof(ll));
  ll.k = (int)sw.gates.size();
  for (size_t t = 0; t < sw.gates.size(); ++t) {
    ll.bit[t] = sw.gates[t].bit;
    ll.tmask |= 1u << sw.gates[t].bit;
    (sw.gates[t].kind == 1 ? ll.sxmask : ll.symask) |= 1u << sw.gates[t].bit;
  }
  ll.pre = to_dev(pre);
  if (sw.post.below(32)) ll.post = to_dev(sw.post, true);  // else the caller restricts it (distributed)
  ll.lmask = ~0ull;
  ll.gsel = 0;
  return ll;
}

// Number of the leaf level's trailing sweeps evaluated lazily at the sampled indices
// (0, 1 or 2; at most lazy_depth_).  Cost model in bytes: a sweep moves 2 * 2^h * amp;
// a lazy layer costs ~96 bytes per scattered read (32-byte sector, ~3x random-access
// inefficiency); depth 2 reads n_S * 2^(k_d + k_(d-1)) values.
int Engine::lazy_depth(int half, int64_t nS) const { return lazy_depth_of(half_[half].prog, nS); }

int Engine::lazy_depth_of(const HalfProgram &hp, int64_t nS) const {
  const int F = (int)hp.levels.size() - 1;
  if (full_leaf_ || F < 1 || lazy_depth_ < 1) return 0;
  const auto &sw = hp.levels[F].sweeps;
  if (sw.empty() || sw.back().gates.size() > 12) return 0;
  if (lazy_depth_ < 2 || sw.size() < 2) return 1;
  // distributed half: a skipped sweep must not carry a local/global swap
  if (dist_ && !sw[sw.size() - 2].swaps.empty()) return 1;
  const int kd = (int)sw.back().gates.size(), kd1 = (int)sw[sw.size() - 2].gates.size();
  if (kd + kd1 > 20 || ((double)nS * std::ldexp(1.0, kd)) > (double)(1 << 26)) return 1;
  const double sweep = 2.0 * std::ldexp(1.0, hp.hl) * (double)amp_;
  const double lazy1 = 96.0 * (double)nS * std::ldexp(1.0, kd);
  const double lazy2 = 96.0 * (double)nS * std::ldexp(1.0, kd + kd1) + 2.0 * lazy1;
  if (lazy_depth_ == 3) return 2;  // forced (tests)
  return lazy2 < sweep + lazy1 ? 2 : 1;
}

// Leaf gather.  depth 0: psi is the complete leaf (a pending fork diagonal is applied);
// depth 1: the leaf level's last sweep is evaluated at the sampled indices; depth 2: its
// last two sweeps, the earlier one on the cone of the last one (compact buffer).
void Engine::gather_leaf(int half, uint64_t child_last, const void *psi, const uint64_t *dS, int64_t nS,
                         void *out_row, int depth) {
  HalfExec &he = half_[half];
  const int F = (int)he.prog.levels.size() - 1;
  const Level &lev = he.prog.levels[F];
  if (depth >= 1) {
    const size_t n = lev.sweeps.size();
    auto pre_of = [&](size_t s) {
      return s == 0 ? Diag::merge(he.prog.fork_diag(F, child_last), lev.sweeps[0].pre) : lev.sweeps[s].pre;
    };
    const uint64_t gsel = (uint64_t)rank_ << he.prog.hl;
    auto shard = [&](const Diag &d) { return dist_ ? d.restrict_low(he.prog.hl, gsel) : d; };
    LazyLayer lld = lazy_layer(lev.sweeps[n - 1], shard(pre_of(n - 1)));
    if (dist_) {
      lld.post = to_dev(shard(lev.sweeps[n - 1].post), true);
      lld.lmask = (1ull << he.prog.hl) - 1ull;
      lld.gsel = gsel;
    }
    if (depth == 1) {
      check(launch_gather_layer(psi, dS, nS, out_row, lld, c128_, stream_), "gather_layer launch");
      st_.kernel_launches++;
    } else {
      LazyLayer ll1 = lazy_layer(lev.sweeps[n - 2], shard(pre_of(n - 2)));
      if (dist_) ll1.post = to_dev(shard(lev.sweeps[n - 2].post), true);
      ll1.lmask = lld.lmask;
      ll1.gsel = lld.gsel;
      const int64_t ncone = nS << lld.k;
      cone_idx_.reserve((size_t)ncone * 8);
      cone_val_.reserve((size_t)ncone * amp_);
      check(launch_cone_indices(dS, nS, lld, cone_idx_.as<uint64_t>(), stream_), "cone launch");
      check(launch_gather_layer(psi, cone_idx_.as<uint64_t>(), ncone, cone_val_.ptr, ll1, c128_, stream_),
            "gather_layer launch");
      check(launch_gather_layer_compact(cone_val_.ptr, dS, nS, out_row, lld, c128_, stream_),
            "gather_layer_compact launch");
      st_.kernel_launches += 3;
    }
    st_.lazy_gathers++;
    return;
  }
  Diag pend;
  if (F >= 1 && lev.sweeps.empty()) pend = he.prog.fork_diag(F, child_last);
  const uint64_t lmask = dist_ ? (1ull << he.prog.hl) - 1ull : ~0ull;
  const uint64_t gsel = dist_ ? (uint64_t)rank_ << he.prog.hl : 0ull;
  if (dist_) pend = pend.restrict_low(he.prog.hl, gsel);
  check(launch_gather(psi, dS, nS, out_row, to_dev(pend), c128_, stream_, lmask, gsel), "gather launch");
  st_.kernel_launches++;
}

int Engine::materialized_from(int half, size_t free_bytes, int *nbuf) {
  const HalfProgram &hp = half_[half].prog;
  const int F = (int)hp.levels.size() - 1;
  size_t budget = free_bytes;
  if (mem_budget_ > 0) budget = std::min(budget, (size_t)mem_budget_);
  int m0 = 0;
  while ((size_t)(F + 1 - m0) * state_bytes_ > budget && m0 < F) ++m0;
  if ((size_t)(F + 1 - m0) * state_bytes_ > budget) {
    std::ostringstream m;
    m << "a " << hp.h << "-qubit half state needs " << state_bytes_ << " bytes; only " << budget
      << " bytes available for state buffers";
    throw Error(QSIM_ENOMEM, m.str());
  }
  *nbuf = F + 1 - m0;
  return m0;
}

void Engine::ensure_states(int half, int nbuf) {
  (void)half;
  while ((int)states_.size() < nbuf) states_.push_back(new DevBuf());
  for (int i = 0; i < nbuf; ++i) states_[i]->reserve(state_bytes_);
}

// Distributed half: the shards run the paper's branch tree depth-first.  A level
// state is kept (its own buffer pair) only when more than one of its children lies in [b0, b1);
// other levels continue in the pair of their parent, in place, so a single branch needs one pair.
// A sweep that swaps local and global qubits stores into the peers' copy of the pair's other
// buffer between two stream-ordered barriers (run_level_dist).
void Engine::evolve_half_dist(int half, uint64_t b0, uint64_t b1, void *slice, const uint64_t *dS, int64_t nS) {
  HalfExec &he = half_[half];
  const HalfProgram &hp = he.prog;
  const int c = hp.ncuts, F = (int)hp.levels.size() - 1;
  std::vector<int> sbits(F + 1, 0);
  for (int l = 1; l <= F; ++l) sbits[l] = sbits[l - 1] + hp.levels[l].k;
  // pair[l]: the buffer pair of level l (a new pair after each kept level)
  std::vector<int> pair(F + 1, 0);
  int npair = 1;
  for (int l = 0; l < F; ++l) {
    const int sh = c - sbits[l + 1];
    const bool keep = sbits[l + 1] > sbits[l] && (b0 >> sh) != ((b1 - 1) >> sh);
    pair[l + 1] = keep ? npair++ : pair[l];
  }
  const int hmax = std::max(half_[0].prog.hl, half_[1].prog.hl);
  dist_buffers(((size_t)1 << hmax) * amp_, 2 * std::max(npair, dist_pairs_));
  dist_pairs_ = std::max(npair, dist_pairs_);
  state_bytes_ = ((size_t)1 << hp.hl) * amp_;
  const int lazy = lazy_depth(half, nS);
  auto skip = [&](int l) { return l == F ? lazy : 0; };
  std::function<void(int, uint64_t, int)> node = [&](int l, uint64_t prefix, int idx) {
    if (l == F) {
      const uint64_t b = prefix;
      const uint64_t ch = F >= 1 ? (b & ((1ull << hp.levels[F].k) - 1ull)) : 0;
      gather_leaf(half, ch, states_[idx]->ptr, dS, nS, (char *)slice + (b - b0) * (uint64_t)nS * amp_, lazy);
      return;
    }
    const int k = hp.levels[l + 1].k;
    const int shift = c - sbits[l + 1];
    for (uint64_t ch = 0; ch < (1ull << k); ++ch) {
      const uint64_t cp = (prefix << k) | ch;
      const uint64_t lo = cp << shift, hi = (cp + 1) << shift;
      if (hi <= b0 || lo >= b1) continue;
      node(l + 1, cp, run_level_dist(half, l + 1, ch, idx, pair[l + 1], skip(l + 1)));
    }
  };
  node(0, 0, run_level_dist(half, 0, 0, -1, 0, skip(0)));
}

int Engine::run_level_dist(int half, int level, uint64_t child, int src, int pair, int skip) {
  HalfExec &he = half_[half];
  const Diag fork = he.prog.fork_diag(level, child);
  const auto &launches = he.plans[level][std::min<size_t>((size_t)skip, he.plans[level].size() - 1)];
  int cur = src;
  for (size_t i = 0; i < launches.size(); ++i) {
    const TilePlan &tp = launches[i];
    int out;
    if (i == 0 && (src < 0 || src / 2 != pair))
      out = 2 * pair;  // a fresh pair: out of place from the parent
    else
      out = tp.swaps.empty() ? cur : (cur ^ 1);  // in place, or the pair's other buffer when swapping
    if (!tp.swaps.empty()) dist_barrier();
    launch_plan(tp, i == 0 ? fork : Diag(), i == 0, cur < 0 ? nullptr : states_[cur]->ptr, states_[out]->ptr,
                he.prog, out);
    if (!tp.swaps.empty()) dist_barrier();
    cur = out;
  }
  return cur;
}

void Engine::evolve_half(int half, uint64_t b0, uint64_t b1, void *slice, const uint64_t *dS, int64_t nS) {
  HalfExec &he = half_[half];
  const HalfProgram &hp = he.prog;
  const int c = hp.ncuts;
  if (!he.tree) {
    if (hp.h > small_max_h(c128_))
      throw Error(QSIM_EINVAL, "flat (small-state) mode needs h <= 12");
    upload_small(he);
    SmallParams sp;
    sp.levels = he.d_levels.as<SmallLevelDev>();
    sp.sweeps = he.d_sweeps.as<SmallSweepDev>();
    sp.nlevels = (int)hp.levels.size();
    sp.h = hp.h;
    sp.c = c;
    sp.S = dS;
    sp.nS = nS;
    const uint64_t maxb = 1u << 30;
    for (uint64_t b = b0; b < b1; b += maxb) {
      const uint64_t nb = std::min(maxb, b1 - b);
      sp.b0 = b;
      sp.out = (char *)slice + (b - b0) * (uint64_t)nS * amp_;
      check(launch_small(sp, c128_, nb, stream_), "small kernel launch");
      st_.kernel_launches++;
      st_.sweeps++;
      st_.sweep_states += nb;
    }
    return;
  }
  const int T = tile_low_bits(c128_) + kHiBits;
  if (hp.hl < T) throw Error(QSIM_EINVAL, "tree mode needs h >= tile bits");
  if (dist_) {
    evolve_half_dist(half, b0, b1, slice, dS, nS);
    return;
  }
  state_bytes_ = ((size_t)1 << hp.hl) * amp_;
  size_t free_b = 0, total_b = 0;
  check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  size_t have = 0;
  for (auto *b : states_) have += b->bytes;
  const size_t margin = (size_t)512 << 20;
  const size_t avail = free_b + have > margin ? free_b + have - margin : 0;
  int nbuf = 0;
  const int m0 = dist_ ? 0 : materialized_from(half, avail, &nbuf);
  if (!dist_) ensure_states(half, nbuf);
  const int F = (int)hp.levels.size() - 1;
  std::vector<int> sbits(F + 1, 0);  // cut bits consumed up to and including level l
  for (int l = 1; l <= F; ++l) sbits[l] = sbits[l - 1] + hp.levels[l].k;
  auto buf = [&](int l) { return dist_ ? states_[2 * l]->ptr : states_[std::max(l, m0) - m0]->ptr; };
  // lazy tail: the leaf level's last `lazy` sweeps are evaluated at the sampled indices
  const int lazy = lazy_depth(half, nS);
  auto skip = [&](int l) { return l == F ? lazy : 0; };

  // recompute levels 0..lt along the path of prefix `cp` in place in buf(m0)
  auto recompute_path = [&](int lt, uint64_t cp) {
    void *b = buf(m0);
    run_level(half, 0, 0, nullptr, b, skip(0));
    for (int l = 1; l <= lt; ++l) {
      const uint64_t ch = (cp >> (sbits[lt] - sbits[l])) & ((1ull << hp.levels[l].k) - 1ull);
      run_level(half, l, ch, b, b, skip(l));
    }
  };

  // from level mb down, a node whose whole subtree lies in [b0, b1) runs it level-synchronously
  const int mb = bfs_level(half, m0, avail > (size_t)nbuf * state_bytes_ ? avail - (size_t)nbuf * state_bytes_ : 0);
  if (std::getenv("QSIM_DEBUG_BFS"))
    std::fprintf(stderr, "evolve_half %d [%llu, %llu): h=%d F=%d cuts=%d m0=%d mb=%d state=%zu avail=%zu\n", half,
                 (unsigned long long)b0, (unsigned long long)b1, hp.hl, F, c, m0, mb, state_bytes_, avail);
  std::function<void(int, uint64_t, const void *)> node = [&](int l, uint64_t prefix, const void *state) {
    if (mb >= 0 && l >= mb && l < F && state) {  // deeper levels have smaller subtrees: they fit too
      const uint64_t lo = prefix << (c - sbits[l]), hi = (prefix + 1) << (c - sbits[l]);
      if (lo >= b0 && hi <= b1) {
        bfs_subtree(half, l, state, (char *)slice + (lo - b0) * (uint64_t)nS * amp_, dS, nS);
        return;
      }
    }
    if (l == F) {
      const uint64_t b = prefix;
      const uint64_t ch = F >= 1 ? (b & ((1ull << hp.levels[F].k) - 1ull)) : 0;
      gather_leaf(half, ch, state, dS, nS, (char *)slice + (b - b0) * (uint64_t)nS * amp_, lazy);
      return;
    }
    const int k = hp.levels[l + 1].k;
    const int shift = c - sbits[l + 1];
    for (uint64_t ch = 0; ch < (1ull << k); ++ch) {
      const uint64_t cp = (prefix << k) | ch;
      const uint64_t lo = cp << shift, hi = (cp + 1) << shift;
      if (hi <= b0 || lo >= b1) continue;
      if (l + 1 < m0) {
        node(l + 1, cp, nullptr);
      } else if (l + 1 == m0) {
        recompute_path(m0, cp);
        node(m0, cp, buf(m0));
      } else {
        node(l + 1, cp, run_level(half, l + 1, ch, state, buf(l + 1), skip(l + 1)));
      }
    }
  };
  if (m0 == 0) {
    node(0, 0, run_level(half, 0, 0, nullptr, buf(0), skip(0)));
  } else {
    node(0, 0, nullptr);
  }
}

void Engine::gemm(const void *U, const void *L, int64_t K, int64_t M, int64_t N, double *A) {
  Nvtx nv("branch GEMM");
  const bool timed = time_sweeps_;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    e0 = get_event();
    e1 = get_event();
    check(cudaEventRecord(e0, stream_), "cudaEventRecord");
  }
  check(launch_branch_gemm(U, L, K, M, N, A, c128_, stream_), "branch gemm launch");
  if (timed) {
    check(cudaEventRecord(e1, stream_), "cudaEventRecord");
    ev_gemm_.emplace_back(e0, e1);
  }
  st_.kernel_launches++;
  st_.gemm_flops += 8.0 * (double)M * (double)N * (double)K;
}

// Half pairs (r2, multi-GPU): with the frame executor each half needs one real state for any
// branch range, so ranks 2i and 2i+1 split the two halves instead of both computing both: each evolves one
// half over the pair's joint range, the rows of the partner's range are swapped (ncclSend / ncclRecv), and
// each contracts its own range.  false: not applicable (the range is not this rank's own, an odd world,
// unequal or non-adjacent partner ranges, a half without frames, or the rows do not fit).
bool Engine::evolve_pair(uint64_t b0, uint64_t b1) {
  if (!pairs_ || dist_ || world_ < 2 || (world_ & 1) || !frames_ || !deferred_) return false;
  if (!flip_half(0) || !flip_half(1)) return false;
  uint64_t r0 = 0, r1 = 0, p0 = 0, p1 = 0;
  rank_range_of(rank_, &r0, &r1);
  rank_range_of(rank_ ^ 1, &p0, &p1);
  if (r0 != b0 || r1 != b1 || p1 - p0 != b1 - b0 || (p1 != b0 && p0 != b1)) return false;
  const int h = rank_ & 1;  // even ranks: the upper half, odd ranks: the lower half
  const uint64_t lo = std::min(b0, p0), hi = std::max(b1, p1), K = b1 - b0;
  const int64_t nu = (int64_t)Su_.size(), nl = (int64_t)Sl_.size();
  const int64_t nh = h == 0 ? nu : nl, no = h == 0 ? nl : nu;
  const size_t mine = (size_t)(hi - lo) * (size_t)nh * amp_, theirs = (size_t)K * (size_t)no * amp_;
  size_t free_b = 0, total_b = 0;
  check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  size_t have = U_.bytes + L_.bytes;
  for (auto *b : states_) have += b->bytes;
  const size_t st = ((size_t)1 << half_[h].prog.hl) * amp_;
  if (mine + theirs + 2 * st + ((size_t)3 << 30) > free_b + have) return false;
  DevBuf &P = h == 0 ? U_ : L_, &Q = h == 0 ? L_ : U_;
  if (P.bytes < mine || Q.bytes < theirs) {
    for (auto *b : states_) b->release();
    U_.release();
    L_.release();
  }
  P.reserve(mine);
  Q.reserve(theirs);
  const bool zz = flip_half(0);
  // the frame basis over the pair range (the lower rank builds it): the Walsh-Hadamard rows
  // then go to the upper side whatever the lower rank's outcome, since sum_a V_a (H L)_a = sum_b (H V)_b L_b
  const uint64_t plen = hi - lo;
  const bool use_basis = basis_enabled_ && zz && (plen & (plen - 1)) == 0 && (lo & (plen - 1)) == 0;
  bool basis_ok = false;
  if (h == 1 && use_basis) {
    basis_on_ = true;
    basis_rows_ = &P;
    basis_cap_ = (int64_t)plen;
    basis_entries_.clear();
    basis_T_ = 0;
    basis_points_ = 0;
    bool aborted = false;
    try {
      evolve_tree(h, lo, hi, P.ptr, d_Sp_[h].as<uint64_t>(), nh, false, true, zz);
    } catch (const BasisAbort &) {
      aborted = true;
    }
    basis_on_ = false;
    basis_ok = !aborted && basis_points_ >= 1 && basis_T_ >= 2;
    if (aborted) evolve_tree(h, lo, hi, P.ptr, d_Sp_[h].as<uint64_t>(), nh, false, true, zz);
  } else {
    evolve_tree(h, lo, hi, P.ptr, d_Sp_[h].as<uint64_t>(), nh, false, true, zz);
  }
  if (zz && h == (use_basis ? 0 : 1)) {  // the same aligned blocks as evolve_tree
    const int c = (int)circ_.cuts.size();
    for (uint64_t a = lo; a < hi;) {
      int m = 0;
      while (m < c && ((a >> m) & 1u) == 0 && a + (2ull << m) <= hi) ++m;
      check(launch_wht_rows((char *)P.ptr + (size_t)(a - lo) * (size_t)nh * amp_, c128_, m, nh, stream_),
            "wht launch");
      st_.kernel_launches += (uint64_t)((m + 7) / 8);
      a += 1ull << m;
    }
  }
  ensure_comm();
  const ncclDataType_t dt = c128_ ? ncclDouble : ncclFloat;
  auto nccl_ok = [&](ncclResult_t r, const char *what) {
    if (r != ncclSuccess) throw Error(QSIM_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
  };
  if (use_basis) {
    // header lower -> upper: basis used, T, terms of the upper's share of the basis rows
    int64_t hdr[4] = {0, 0, 0, 0};
    std::vector<uint32_t> off_lo, src_lo, off_hi, src_hi;
    std::vector<double> coef_lo, coef_hi;
    int64_t T = 0, th = 0;
    if (h == 1 && basis_ok) {
      T = basis_T_;
      th = T / 2;  // the lower rank contracts basis rows [0, th), the upper one [th, T)
      off_lo.assign((size_t)th + 1, 0);
      off_hi.assign((size_t)(T - th) + 1, 0);
      for (const BasisEntry &x : basis_entries_) (x.t < th ? off_lo[x.t + 1] : off_hi[x.t - th + 1])++;
      for (int64_t t = 0; t < th; ++t) off_lo[t + 1] += off_lo[t];
      for (int64_t t = 0; t < T - th; ++t) off_hi[t + 1] += off_hi[t];
      src_lo.resize(off_lo.back());
      coef_lo.resize(2 * (size_t)off_lo.back());
      src_hi.resize(off_hi.back());
      coef_hi.resize(2 * (size_t)off_hi.back());
      std::vector<uint32_t> plo(off_lo.begin(), off_lo.end() - 1), phi(off_hi.begin(), off_hi.end() - 1);
      for (const BasisEntry &x : basis_entries_) {
        const bool lw = x.t < th;
        const uint32_t q = lw ? plo[x.t]++ : phi[x.t - th]++;
        (lw ? src_lo : src_hi)[q] = x.row;
        (lw ? coef_lo : coef_hi)[2 * q] = x.cr;
        (lw ? coef_lo : coef_hi)[2 * q + 1] = x.ci;
      }
      hdr[0] = 1;
      hdr[1] = T;
      hdr[2] = (int64_t)off_hi.back();
    }
    basis_hdr_.reserve(32);
    if (h == 1) check(cudaMemcpyAsync(basis_hdr_.ptr, hdr, 32, cudaMemcpyHostToDevice, stream_), "pair header");
    nccl_ok(h == 1 ? ncclSend(basis_hdr_.ptr, 4, ncclInt64, rank_ ^ 1, comm_, stream_)
                   : ncclRecv(basis_hdr_.ptr, 4, ncclInt64, rank_ ^ 1, comm_, stream_),
            "pair header");
    if (h == 0) {
      check(cudaMemcpyAsync(hdr, basis_hdr_.ptr, 32, cudaMemcpyDeviceToHost, stream_), "pair header");
      check(cudaStreamSynchronize(stream_), "pair header");
      T = hdr[1];
      th = T / 2;
    }
    if (hdr[0] == 1) {
      const int64_t nnz_hi = hdr[2];
      // the lower rank: its CSR of [0, th) local, the upper's sent; the upper rank: all H V rows sent
      DevBuf &hv = h == 0 ? U_ : Q;  // the (H V) rows of the pair range on each rank
      if (h == 1) Q.reserve((size_t)plen * (size_t)nu * amp_);
      if (h == 0) Q.reserve((size_t)(T - th) * (size_t)nl * amp_);
      const int64_t Tm = h == 0 ? T - th : th;
      basis_off_.reserve((size_t)(Tm + 1) * 4);
      basis_src_.reserve((size_t)std::max<int64_t>(1, h == 0 ? nnz_hi : (int64_t)src_lo.size()) * 4);
      basis_coef_.reserve((size_t)std::max<int64_t>(1, h == 0 ? nnz_hi : (int64_t)src_lo.size()) * 16);
      if (h == 1) {
        check(cudaMemcpyAsync(basis_off_.ptr, off_lo.data(), off_lo.size() * 4, cudaMemcpyHostToDevice, stream_), "csr");
        check(cudaMemcpyAsync(basis_src_.ptr, src_lo.data(), src_lo.size() * 4, cudaMemcpyHostToDevice, stream_), "csr");
        check(cudaMemcpyAsync(basis_coef_.ptr, coef_lo.data(), coef_lo.size() * 8, cudaMemcpyHostToDevice, stream_),
              "csr");
        basis_xoff_.reserve(off_hi.size() * 4);
        basis_xsrc_.reserve(std::max<size_t>(1, src_hi.size()) * 4);
        basis_xcoef_.reserve(std::max<size_t>(1, src_hi.size()) * 16);
        check(cudaMemcpyAsync(basis_xoff_.ptr, off_hi.data(), off_hi.size() * 4, cudaMemcpyHostToDevice, stream_), "csr");
        check(cudaMemcpyAsync(basis_xsrc_.ptr, src_hi.data(), src_hi.size() * 4, cudaMemcpyHostToDevice, stream_), "csr");
        check(cudaMemcpyAsync(basis_xcoef_.ptr, coef_hi.data(), coef_hi.size() * 8, cudaMemcpyHostToDevice, stream_),
              "csr");
      }
      ncclGroupStart();
      if (h == 1) {
        nccl_ok(ncclSend((const char *)P.ptr + (size_t)th * (size_t)nl * amp_, (size_t)(T - th) * (size_t)nl * 2, dt,
                         rank_ ^ 1, comm_, stream_), "basis rows");
        nccl_ok(ncclSend(basis_xoff_.ptr, (size_t)(T - th) + 1, ncclUint32, rank_ ^ 1, comm_, stream_), "basis csr");
        if (nnz_hi) {
          nccl_ok(ncclSend(basis_xsrc_.ptr, (size_t)nnz_hi, ncclUint32, rank_ ^ 1, comm_, stream_), "basis csr");
          nccl_ok(ncclSend(basis_xcoef_.ptr, 2 * (size_t)nnz_hi, ncclDouble, rank_ ^ 1, comm_, stream_), "basis csr");
        }
        nccl_ok(ncclRecv(hv.ptr, (size_t)plen * (size_t)nu * 2, dt, rank_ ^ 1, comm_, stream_), "H V rows");
      } else {
        nccl_ok(ncclSend(U_.ptr, (size_t)plen * (size_t)nu * 2, dt, rank_ ^ 1, comm_, stream_), "H V rows");
        nccl_ok(ncclRecv(Q.ptr, (size_t)(T - th) * (size_t)nl * 2, dt, rank_ ^ 1, comm_, stream_), "basis rows");
        nccl_ok(ncclRecv(basis_off_.ptr, (size_t)(T - th) + 1, ncclUint32, rank_ ^ 1, comm_, stream_), "basis csr");
        if (nnz_hi) {
          nccl_ok(ncclRecv(basis_src_.ptr, (size_t)nnz_hi, ncclUint32, rank_ ^ 1, comm_, stream_), "basis csr");
          nccl_ok(ncclRecv(basis_coef_.ptr, 2 * (size_t)nnz_hi, ncclDouble, rank_ ^ 1, comm_, stream_), "basis csr");
        }
      }
      nccl_ok(ncclGroupEnd(), "pair basis exchange");
      // U' of this rank's basis rows in the idle state buffer, then the GEMM over them
      const size_t ub = (size_t)Tm * (size_t)nu * amp_;
      DevBuf *scratch = (!states_.empty() && states_[0]->bytes >= ub) ? states_[0] : &tmp_;
      if (scratch == &tmp_) tmp_.reserve(ub);
      check(launch_combine_rows(hv.ptr, nu, basis_off_.as<uint32_t>(), basis_src_.as<uint32_t>(), basis_coef_.ptr, Tm,
                                scratch->ptr, c128_, stream_),
            "combine rows launch");
      st_.kernel_launches++;
      check(cudaStreamSynchronize(stream_), "pair basis");  // host CSR temporaries
      const void *brows = h == 0 ? Q.ptr : P.ptr;  // the upper received rows [th, T); the lower keeps [0, th)
      gemm(scratch->ptr, brows, Tm, nu, nl, A_acc_.as<double>());
      st_.branches_evolved += K;
      check(cudaGetLastError(), "evolve");
      reduced_ = false;
      return true;
    }
  }
  ncclGroupStart();
  ncclResult_t r1s = ncclSend((const char *)P.ptr + (size_t)(p0 - lo) * (size_t)nh * amp_, (size_t)K * (size_t)nh * 2,
                              dt, rank_ ^ 1, comm_, stream_);
  ncclResult_t r2s = ncclRecv(Q.ptr, (size_t)K * (size_t)no * 2, dt, rank_ ^ 1, comm_, stream_);
  ncclResult_t r3s = ncclGroupEnd();
  if (r1s != ncclSuccess || r2s != ncclSuccess || r3s != ncclSuccess)
    throw Error(QSIM_ENCCL, std::string("pair row exchange: ") + ncclGetErrorString(r3s != ncclSuccess ? r3s : r1s));
  const void *own = (const char *)P.ptr + (size_t)(b0 - lo) * (size_t)nh * amp_;
  gemm(h == 0 ? own : Q.ptr, h == 0 ? Q.ptr : own, (int64_t)K, nu, nl, A_acc_.as<double>());
  st_.branches_evolved += K;
  check(cudaGetLastError(), "evolve");
  reduced_ = false;
  return true;
}

void Engine::evolve_range(uint64_t b0, uint64_t b1) {
  Nvtx nv("qsim_evolve_range");
  if (!have_circuit_) throw Error(QSIM_ESTATE, "no circuit loaded");
  if (!have_blocks_) throw Error(QSIM_ESTATE, "no blocks set (qsim_set_blocks)");
  const int c = (int)circ_.cuts.size();
  if (c > 62) throw Error(QSIM_EINVAL, "too many cuts");
  const uint64_t B = 1ull << c;
  if (b0 >= b1 || b1 > B) throw Error(QSIM_EINVAL, "bad branch range");
  ensure_device();
  for (int h = 0; h < 2; ++h) {
    const HalfExec &he = half_[h];
    const int T = tile_low_bits(c128_) + kHiBits;
    if (he.prog.hl > 32) {
      std::ostringstream m;
      m << "a " << he.prog.h << "-qubit half needs QSIM_OPT_DISTRIBUTE over at least " << (1 << (he.prog.h - 32))
        << " ranks (at most 32 qubits per shard)";
      throw Error(QSIM_EINVAL, m.str());
    }
    if (he.tree && he.prog.h < T) throw Error(QSIM_EINVAL, "tree mode needs h >= 13 (c64) / 12 (c128)");
    if (!he.tree && he.prog.h > small_max_h(c128_)) throw Error(QSIM_EINVAL, "flat mode needs h <= 12");
  }
  if (!roles_chosen_ && deferred_) choose_roles();
  // shared basis (ranks <= QSIM_SHARED_BASIS_MAX, default 2): every rank evolves both halves
  // over the union of the ranks' ranges (the frame executor needs one state per half for any range) and
  // contracts its share of the frame basis; no data exchange.  Else half pairs, else the own range.
  uint64_t own0 = b0, own1 = b1;
  int share_r = 0, share_n = 1;
  if (world_ >= 2 && world_ <= shared_basis_max_ && !dist_ && frames_ && basis_enabled_ && deferred_ &&
      flip_half(0) && flip_half(1)) {
    uint64_t r0 = 0, r1 = 0, g0 = 0, g1 = 0, x0 = 0, x1 = 0;
    rank_range_of(rank_, &r0, &r1);
    rank_range_of(0, &g0, &x0);
    rank_range_of(world_ - 1, &x1, &g1);
    const uint64_t len = g1 - g0;
    if (r0 == b0 && r1 == b1 && (len & (len - 1)) == 0 && (g0 & (len - 1)) == 0) {
      b0 = g0;
      b1 = g1;
      share_r = rank_;
      share_n = world_;
    }
  }
  if (share_n == 1 && evolve_pair(b0, b1)) return;
  const int64_t nu = (int64_t)Su_.size(), nl = (int64_t)Sl_.size();
  // slices for a chunk of branches (bounded at 1 GiB per half)
  const uint64_t per_branch = (uint64_t)std::max(nu, nl) * amp_;
  uint64_t chunk = std::max<uint64_t>(1, ((uint64_t)1 << 30) / per_branch);
  if (frames_ && (flip_half(0) || flip_half(1))) {
    // Pauli frames share real states across every branch of a block, so one block should span the
    // range: slices as large as the memory left beside two state buffers of the larger half allows
    size_t free_b = 0, total_b = 0;
    check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    size_t have = U_.bytes + L_.bytes;
    for (auto *b : states_) have += b->bytes;
    const size_t st = ((size_t)1 << std::max(half_[0].prog.hl, half_[1].prog.hl)) * amp_;
    const size_t reserve = 2 * st + ((size_t)3 << 30);
    const size_t room = free_b + have > reserve ? free_b + have - reserve : 0;
    const uint64_t both = (uint64_t)(nu + nl) * amp_;
    const uint64_t fit = room / both;
    if (fit > chunk) {
      chunk = fit;
      const uint64_t want = std::min<uint64_t>(chunk, b1 - b0) * both;
      if (U_.bytes + L_.bytes < want) {  // the state buffers are re-reserved by the executor
        for (auto *b : states_) b->release();
        U_.release();
        L_.release();
      }
    }
  }
  // align the chunk to a power of two so that chunks are whole subtrees
  uint64_t p2 = 1;
  while (p2 * 2 <= chunk) p2 *= 2;
  chunk = std::min<uint64_t>(p2, b1 - b0);
  U_.reserve(chunk * nu * amp_);
  L_.reserve(chunk * nl * amp_);
  if (!roles_chosen_ && deferred_) choose_roles();
  for (uint64_t s = b0; s < b1;) {
    uint64_t e = std::min(b1, (s / p2 + 1) * p2);
    e = std::min(e, s + chunk);
    // sibling flips need Z^b forks: in the upper half (P_b canonically) the blocks' free cuts then
    // take Z^b on both endpoints and the lower slices the Walsh-Hadamard transform (R-zz)
    const bool zz = flip_half(0) && deferred_;
    // frame basis for the lower half (one rank, frame executor): the Walsh-Hadamard transform then goes to the
    // upper rows (sum_a V_a (H L)_a = sum_b (H V)_b L_b, H symmetric) so that L stays a sparse combination
    const uint64_t len = e - s;
    const bool one_block = (len & (len - 1)) == 0 && (s & (len - 1)) == 0;  // evolve_tree runs it as one block
    const bool basis = basis_enabled_ && zz && (world_ == 1 || share_n > 1) && !dist_ && frames_ && flip_half(1) &&
                       half_[1].tree && one_block;
    bool basis_ok = false;
    for (int h = 0; h < 2; ++h) {
      void *sl = h == 0 ? U_.ptr : L_.ptr;
      const int64_t ns = h == 0 ? nu : nl;
      if (h == 1 && basis) {
        basis_on_ = true;
        basis_rows_ = &L_;
        basis_cap_ = (int64_t)(e - s);
        basis_entries_.clear();
        basis_T_ = 0;
        basis_points_ = 0;
        bool aborted = false;
        try {
          evolve_tree(h, s, e, sl, d_Sp_[h].as<uint64_t>(), ns, false, true, zz);
        } catch (const BasisAbort &) {
          aborted = true;
        }
        basis_on_ = false;
        basis_ok = !aborted && basis_points_ >= 1;
        // basis_points_ == 0: another executor ran the block and wrote the leaf rows as usual
        if (!aborted) continue;
      }
      if (deferred_ && !dist_ && half_[h].tree)
        evolve_tree(h, s, e, sl, d_Sp_[h].as<uint64_t>(), ns, false, flip_half(h), zz);
      else
        evolve_half(h, s, e, sl, d_Sp_[h].as<uint64_t>(), ns);
    }
    if (zz) {  // the same aligned blocks as evolve_tree
      DevBuf &W = basis ? U_ : L_;
      const int64_t nw = basis ? nu : nl;
      for (uint64_t a = s; a < e;) {
        int m = 0;
        while (m < c && ((a >> m) & 1u) == 0 && a + (2ull << m) <= e) ++m;
        check(launch_wht_rows((char *)W.ptr + (size_t)(a - s) * (size_t)nw * amp_, c128_, m, nw, stream_),
              "wht launch");
        st_.kernel_launches += (uint64_t)((m + 7) / 8);
        a += 1ull << m;
      }
    }
    if (basis_ok && basis_T_ > 0 && share_n == 1 && basis_T_ >= (int64_t)(e - s)) {
      // as many distinct frames as branches: no gain from the basis, the leaf rows L = C B are formed instead
      const int64_t K = (int64_t)(e - s);
      std::vector<uint32_t> off((size_t)K + 1, 0), src(basis_entries_.size());
      std::vector<double> coef(2 * basis_entries_.size());
      for (const BasisEntry &x : basis_entries_) off[x.row + 1]++;
      for (int64_t r = 0; r < K; ++r) off[r + 1] += off[r];
      std::vector<uint32_t> pos(off.begin(), off.end() - 1);
      for (const BasisEntry &x : basis_entries_) {
        const uint32_t q = pos[x.row]++;
        src[q] = x.t;
        coef[2 * q] = x.cr;
        coef[2 * q + 1] = x.ci;
      }
      basis_off_.reserve(off.size() * 4);
      basis_src_.reserve(src.size() * 4);
      basis_coef_.reserve(coef.size() * 8);
      upload_async(basis_off_.ptr, off.data(), off.size() * 4);
      upload_async(basis_src_.ptr, src.data(), src.size() * 4);
      upload_async(basis_coef_.ptr, coef.data(), coef.size() * 8);
      const size_t lb = (size_t)K * (size_t)nl * amp_;
      DevBuf *scratch = (!states_.empty() && states_[0]->bytes >= lb) ? states_[0] : &tmp_;
      if (scratch == &tmp_) tmp_.reserve(lb);
      check(launch_combine_rows(L_.ptr, nl, basis_off_.as<uint32_t>(), basis_src_.as<uint32_t>(), basis_coef_.ptr, K,
                                scratch->ptr, c128_, stream_),
            "combine rows launch");
      st_.kernel_launches++;
      gemm(U_.ptr, scratch->ptr, K, nu, nl, A_acc_.as<double>());
      st_.branches_evolved += e - s;
      s = e;
      continue;
    }
    if (basis_ok && basis_T_ > 0) {
      // A += (C^T (H V))^T B: U'[t] = sum over the terms (b, t, c) of c (H V)_b, then the GEMM over the basis;
      // with a shared basis this rank takes the basis rows [t0, t1)
      const int64_t Tall = basis_T_;
      const int64_t t0 = Tall * share_r / share_n, t1 = Tall * (share_r + 1) / share_n, T = t1 - t0;
      std::vector<uint32_t> off((size_t)T + 1, 0), src(basis_entries_.size());
      std::vector<double> coef(2 * basis_entries_.size());
      for (BasisEntry &x : basis_entries_) x.t = (x.t >= t0 && x.t < t1) ? (uint32_t)(x.t - t0) : ~0u;
      basis_entries_.erase(std::remove_if(basis_entries_.begin(), basis_entries_.end(),
                                          [](const BasisEntry &x) { return x.t == ~0u; }),
                           basis_entries_.end());
      src.resize(basis_entries_.size());
      coef.resize(2 * basis_entries_.size());
      for (const BasisEntry &x : basis_entries_) off[x.t + 1]++;
      for (int64_t t = 0; t < T; ++t) off[t + 1] += off[t];
      std::vector<uint32_t> pos(off.begin(), off.end() - 1);
      for (const BasisEntry &x : basis_entries_) {
        const uint32_t q = pos[x.t]++;
        src[q] = x.row;
        coef[2 * q] = x.cr;
        coef[2 * q + 1] = x.ci;
      }
      basis_off_.reserve(off.size() * 4);
      basis_src_.reserve(src.size() * 4);
      basis_coef_.reserve(coef.size() * 8);
      upload_async(basis_off_.ptr, off.data(), off.size() * 4);
      upload_async(basis_src_.ptr, src.data(), src.size() * 4);
      upload_async(basis_coef_.ptr, coef.data(), coef.size() * 8);
      // U' in the (now idle) state buffer of the lower half when it is large enough
      const size_t ub = (size_t)T * (size_t)nu * amp_;
      DevBuf *scratch = (!states_.empty() && states_[0]->bytes >= ub) ? states_[0] : &tmp_;
      if (scratch == &tmp_) tmp_.reserve(ub);
      check(launch_combine_rows(U_.ptr, nu, basis_off_.as<uint32_t>(), basis_src_.as<uint32_t>(), basis_coef_.ptr, T,
                                scratch->ptr, c128_, stream_),
            "combine rows launch");
      st_.kernel_launches++;
      gemm(scratch->ptr, (const char *)L_.ptr + (size_t)t0 * (size_t)nl * amp_, T, nu, nl, A_acc_.as<double>());
      st_.branches_evolved += e - s;
      s = e;
      continue;
    }
    if (share_n > 1) {  // the basis was not applicable: this rank contracts its own branch range only
      const uint64_t a0 = std::max(s, own0), a1 = std::min(e, own1);
      if (a1 > a0)
        gemm((const char *)U_.ptr + (size_t)(a0 - s) * (size_t)nu * amp_,
             (const char *)L_.ptr + (size_t)(a0 - s) * (size_t)nl * amp_, (int64_t)(a1 - a0), nu, nl,
             A_acc_.as<double>());
      st_.branches_evolved += a1 > a0 ? a1 - a0 : 0;
      s = e;
      continue;
    }
    if (dist_ && world_ > 1) {
      // §2.3.3: each rank gathered the sampled entries it owns (zeros elsewhere).  The lower
      // slices are summed on every rank; the upper ones stay partial, so the GEMM gives this
      // rank's rows of A, and the final block reduction adds the ranks' rows.
      ensure_comm();
      const size_t cnt = (size_t)(e - s) * (size_t)nl * 2;
      ncclResult_t r = ncclAllReduce(L_.ptr, L_.ptr, cnt, c128_ ? ncclDouble : ncclFloat, ncclSum, comm_, stream_);
      if (r != ncclSuccess) throw Error(QSIM_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
    }
    gemm(U_.ptr, L_.ptr, (int64_t)(e - s), nu, nl, A_acc_.as<double>());
    st_.branches_evolved += e - s;
    s = e;
  }
  check(cudaGetLastError(), "evolve");
  reduced_ = false;
}

// ---------------------------------------------------------------- reduction / outputs
double *Engine::reduced_block() {
  Nvtx nv("block reduction");
  const size_t n = Su_.size() * Sl_.size();
  if (world_ == 1) return A_acc_.as<double>();
  if (!reduced_) {
    ensure_comm();
    if (rank_ == 0) A_tot_.reserve(n * 16);
    ncclResult_t r = ncclReduce(A_acc_.ptr, rank_ == 0 ? A_tot_.ptr : nullptr, 2 * n, ncclDouble, ncclSum,
                                0, comm_, stream_);
    if (r != ncclSuccess) throw Error(QSIM_ENCCL, std::string("ncclReduce: ") + ncclGetErrorString(r));
    reduced_ = true;
  }
  return rank_ == 0 ? A_tot_.as<double>() : nullptr;
}

void Engine::amplitudes(void *amps) {
  Nvtx nv("qsim_amplitudes");
  if (!have_blocks_) throw Error(QSIM_ESTATE, "no blocks evolved");
  ensure_device();
  double *A = reduced_block();
  const size_t n = Su_.size() * Sl_.size();
  if (A && amps) {
    if (c128_) {
      check(cudaMemcpyAsync(amps, A, n * 16, cudaMemcpyDeviceToHost, stream_), "D2H amplitudes");
    } else {
      tmp_.reserve(n * 8);
      check(launch_cast_c128_to_c64(A, (int64_t)(2 * n), tmp_.as<float>(), stream_), "cast");
      st_.kernel_launches++;
      check(cudaMemcpyAsync(amps, tmp_.ptr, n * 8, cudaMemcpyDeviceToHost, stream_), "D2H amplitudes");
    }
  }
  check(cudaStreamSynchronize(stream_), "amplitudes");
}

// a8 on rows [row0, row0 + nrows) of an M x N block: p = |a|^2 fused into
// the row scan when A is given (else p is the caller's), row prefixes C and row masses r of the own
// rows; with `collective` the ranks' row masses are all-gathered (one broadcast per rank), every
// rank forms the same R = sequential prefix of r and W = R[M-1], draws the same Philox stream and
// resolves the draws whose row it owns; the draws are summed to rank 0 (unowned ones are 0).
void Engine::run_sampler(const double *A, const double *p, int64_t M, int64_t N, int64_t row0, int64_t nrows,
                         bool collective, const uint64_t *dSu, const uint64_t *dSl, uint32_t hl, uint64_t seed,
                         size_t n, uint64_t *out, double *mass) {
  C_.reserve((size_t)std::max<int64_t>(nrows, 1) * N * 8);
  r_.reserve((size_t)M * 8);
  R_.reserve((size_t)M * 8);
  W_.reserve(8);
  if (A) {
    p_.reserve((size_t)std::max<int64_t>(nrows, 1) * N * 8);
    p = p_.as<double>();
  }
  if (nrows > 0) {
    if (A)
      check(launch_row_scan_abs2(A, nrows, N, p_.as<double>(), C_.as<double>(), r_.as<double>() + row0, stream_),
            "row scan");
    else
      check(launch_row_scan(p, nrows, N, C_.as<double>(), r_.as<double>() + row0, stream_), "row scan");
    st_.kernel_launches++;
  }
  if (collective && world_ > 1) {
    ncclGroupStart();
    for (int q = 0; q < world_; ++q) {
      const int64_t q0 = M * q / world_, q1 = M * (q + 1) / world_;
      if (q1 > q0)
        ncclBroadcast(r_.as<double>() + q0, r_.as<double>() + q0, (size_t)(q1 - q0), ncclDouble, q, comm_, stream_);
    }
    const ncclResult_t rr = ncclGroupEnd();
    if (rr != ncclSuccess) throw Error(QSIM_ENCCL, std::string("row-mass all-gather: ") + ncclGetErrorString(rr));
  }
  check(launch_row_prefix(r_.as<double>(), M, R_.as<double>(), W_.as<double>(), stream_), "row prefix");
  st_.kernel_launches++;
  if (out || mass) {
    double W = 0;
    check(cudaMemcpyAsync(&W, W_.ptr, 8, cudaMemcpyDeviceToHost, stream_), "D2H block mass");
    check(cudaStreamSynchronize(stream_), "sample");
    if (!(W > 0.0)) throw Error(QSIM_ENUMERIC, "block has zero total probability mass");
    if (mass) *mass = W;
  }
  if (n > 0) {
    draws_.reserve(n * 8);
    check(launch_draws(p, C_.as<double>(), r_.as<double>(), R_.as<double>(), W_.as<double>(), M, N, dSu, dSl, hl,
                       seed, (int64_t)n, draws_.as<uint64_t>(), stream_, row0, nrows),
          "draws");
    st_.kernel_launches++;
    if (collective && world_ > 1) {
      const ncclResult_t r = ncclReduce(draws_.ptr, draws_.ptr, n, ncclUint64, ncclSum, 0, comm_, stream_);
      if (r != ncclSuccess) throw Error(QSIM_ENCCL, std::string("ncclReduce (draws): ") + ncclGetErrorString(r));
    }
    if (out && (!collective || rank_ == 0)) {
      check(cudaMemcpyAsync(out, draws_.ptr, n * 8, cudaMemcpyDeviceToHost, stream_), "D2H draws");
      check(cudaStreamSynchronize(stream_), "sample");
    }
  }
}

void Engine::sample(uint64_t seed, size_t n, uint64_t *out, double *mass) {
  Nvtx nv("qsim_sample");
  if (!have_blocks_) throw Error(QSIM_ESTATE, "no blocks evolved");
  if (circ_.n > 64) throw Error(QSIM_EINVAL, "outcomes of more than 64 qubits do not fit a 64-bit draw (qsim_amplitudes)");
  ensure_device();
  const int64_t M = (int64_t)Su_.size(), N = (int64_t)Sl_.size();
  if (world_ == 1) {
    run_sampler(A_acc_.as<double>(), nullptr, M, N, 0, M, false, d_Su_.as<uint64_t>(), d_Sl_.as<uint64_t>(),
                circ_.h_l, seed, n, out, mass);
    return;
  }
  // a7 as SURVEY §8(e): the partial blocks reduce-scattered by rows (one ncclReduce per row shard),
  // then a8 on the own rows with the row masses all-gathered ("the components they possess are
  // calculated and then added")
  ensure_comm();
  const int64_t r0 = M * rank_ / world_, r1 = M * (rank_ + 1) / world_;
  A_part_.reserve((size_t)std::max<int64_t>(r1 - r0, 1) * N * 16);
  {
    Nvtx nv2("block reduce-scatter");
    ncclGroupStart();
    for (int q = 0; q < world_; ++q) {
      const int64_t q0 = M * q / world_, q1 = M * (q + 1) / world_;
      if (q1 > q0)
        ncclReduce(A_acc_.as<double>() + 2 * q0 * N, q == rank_ ? A_part_.ptr : nullptr, (size_t)(2 * (q1 - q0) * N),
                   ncclDouble, ncclSum, q, comm_, stream_);
    }
    const ncclResult_t rr = ncclGroupEnd();
    if (rr != ncclSuccess) throw Error(QSIM_ENCCL, std::string("block reduce-scatter: ") + ncclGetErrorString(rr));
  }
  run_sampler(A_part_.as<double>(), nullptr, M, N, r0, r1 - r0, true, d_Su_.as<uint64_t>(), d_Sl_.as<uint64_t>(),
              circ_.h_l, seed, n, out, mass);
}

void Engine::sample_probs(const double *p, const uint64_t *up, size_t nu, const uint64_t *lo, size_t nl,
                          uint32_t hl, uint64_t seed, size_t n, uint64_t *out, double *mass) {
  if (!p || !up || !lo || nu == 0 || nl == 0) throw Error(QSIM_EINVAL, "empty probability block");
  if (hl > 63) throw Error(QSIM_EINVAL, "h_lower must be < 64");
  for (size_t i = 0; i < nu * nl; ++i)
    if (!(p[i] >= 0.0)) throw Error(QSIM_EINVAL, "probabilities must be >= 0");
  ensure_device();
  p_.reserve(nu * nl * 8);
  tmp_.reserve((nu + nl) * 8);
  check(cudaMemcpyAsync(p_.ptr, p, nu * nl * 8, cudaMemcpyHostToDevice, stream_), "upload p");
  uint64_t *dsu = tmp_.as<uint64_t>(), *dsl = dsu + nu;
  check(cudaMemcpyAsync(dsu, up, nu * 8, cudaMemcpyHostToDevice, stream_), "upload S_u");
  check(cudaMemcpyAsync(dsl, lo, nl * 8, cudaMemcpyHostToDevice, stream_), "upload S_l");
  double W = 0;
  run_sampler(nullptr, p_.as<double>(), (int64_t)nu, (int64_t)nl, 0, (int64_t)nu, false, dsu, dsl, hl, seed, n, out,
              mass ? mass : &W);
}

void Engine::porter_thomas(const double *p, size_t n, uint32_t nq, double z_lo, double z_hi, uint32_t nb,
                           uint64_t *hist, double *expected, qsim_pt_t *out) {
  if (!out) throw Error(QSIM_EINVAL, "null output");
  if (nb < 1 || nb > (uint32_t)PT_MAX_Z_BINS) throw Error(QSIM_EINVAL, "n_bins must be in 1..8192");
  if (!(z_hi > z_lo) || !std::isfinite(z_lo) || !std::isfinite(z_hi)) throw Error(QSIM_EINVAL, "bad z range");
  if (nq == 0) {
    if (!have_circuit_) throw Error(QSIM_EINVAL, "n_qubits = 0 needs a loaded circuit");
    nq = circ_.n;
  }
  if (nq > 1000) throw Error(QSIM_EINVAL, "n_qubits too large");
  if (p) {
    if (n == 0 || n >= (1ull << 32)) throw Error(QSIM_EINVAL, "n must be in 1..2^32-1");
    for (size_t i = 0; i < n; ++i)
      if (!(p[i] >= 0.0)) throw Error(QSIM_EINVAL, "probabilities must be >= 0");
  } else if (!have_blocks_) {
    throw Error(QSIM_ESTATE, "no blocks evolved");
  }
  ensure_device();
  const void *in = nullptr;
  if (p) {
    p_.reserve(n * 8);
    check(cudaMemcpyAsync(p_.ptr, p, n * 8, cudaMemcpyHostToDevice, stream_), "upload p");
    in = p_.ptr;
  } else {
    in = reduced_block();
    n = Su_.size() * Sl_.size();
    if (!in) {  // not rank 0: the reduction is done, nothing to analyse here
      check(cudaStreamSynchronize(stream_), "porter_thomas");
      std::memset(out, 0, sizeof(*out));
      return;
    }
    if (n >= (1ull << 32)) throw Error(QSIM_EINVAL, "block larger than 2^32-1 entries");
  }
  pt_.reserve(PtScratch::bytes((int)nb));
  check(launch_porter_thomas(in, p == nullptr, (int64_t)n, (int)nq, z_lo, z_hi, (int)nb, pt_.ptr, stream_),
        "porter_thomas");
  st_.kernel_launches += 2;
  PtResult r;
  std::vector<unsigned> zh(nb);
  check(cudaMemcpyAsync(&r, pt_result(pt_.ptr), sizeof(r), cudaMemcpyDeviceToHost, stream_), "D2H pt");
  check(cudaMemcpyAsync(zh.data(), pt_zhist(pt_.ptr), nb * 4, cudaMemcpyDeviceToHost, stream_), "D2H hist");
  check(cudaStreamSynchronize(stream_), "porter_thomas");
  const double cnt = (double)n, npos = (double)(n - r.zeros);
  out->count = cnt;
  out->zeros = (double)r.zeros;
  out->mean_Np = r.s1 / cnt;
  out->var_Np = r.s2 / cnt - out->mean_Np * out->mean_Np;
  out->ks_lo = r.ks_lo;
  out->ks_hi = r.ks_hi;
  out->below = (double)r.below;
  out->above = (double)r.above;
  out->n_qubits = nq;
  out->n_bins = nb;
  if (hist)
    for (uint32_t k = 0; k < nb; ++k) hist[k] = zh[k];
  if (expected) {  // Eq. 7 with alpha = 1: F(z) = 1 - exp(-e^z)
    const double w = (z_hi - z_lo) / nb;
    double F0 = -std::expm1(-std::exp(z_lo));
    for (uint32_t k = 0; k < nb; ++k) {
      const double F1 = -std::expm1(-std::exp(z_lo + (k + 1) * w));
      expected[k] = npos * (F1 - F0);
      F0 = F1;
    }
  }
}

void Engine::branch_sum(const void *U, const void *L, size_t nb, size_t nu, size_t nl, void *A) {
  if (!U || !L || !A || nb == 0 || nu == 0 || nl == 0) throw Error(QSIM_EINVAL, "empty slices");
  ensure_device();
  U_.reserve(nb * nu * amp_);
  L_.reserve(nb * nl * amp_);
  A_tot_.reserve(nu * nl * 16);
  check(cudaMemcpyAsync(U_.ptr, U, nb * nu * amp_, cudaMemcpyHostToDevice, stream_), "upload U");
  check(cudaMemcpyAsync(L_.ptr, L, nb * nl * amp_, cudaMemcpyHostToDevice, stream_), "upload L");
  check(cudaMemsetAsync(A_tot_.ptr, 0, nu * nl * 16, stream_), "zero A");
  gemm(U_.ptr, L_.ptr, (int64_t)nb, (int64_t)nu, (int64_t)nl, A_tot_.as<double>());
  check(cudaMemcpyAsync(A, A_tot_.ptr, nu * nl * 16, cudaMemcpyDeviceToHost, stream_), "D2H A");
  check(cudaStreamSynchronize(stream_), "branch_sum");
  reduced_ = false;
}

void Engine::branch_state(int half, uint64_t b, void *out) {
  if (!have_circuit_) throw Error(QSIM_ESTATE, "no circuit loaded");
  if (half != 0 && half != 1) throw Error(QSIM_EINVAL, "half must be 0 (upper) or 1 (lower)");
  const int c = (int)circ_.cuts.size();
  if (c > 62 || b >= (1ull << c)) throw Error(QSIM_EINVAL, "branch out of range");
  if (!out) throw Error(QSIM_EINVAL, "out is NULL");
  ensure_device();
  HalfExec &he = half_[half];
  const int h = he.prog.h;
  const size_t n = (size_t)1 << h;
  // gather every index of the leaf: the same executor, S = 0 .. 2^h - 1
  tmp_.reserve(n * 8);
  std::vector<uint64_t> all(n);
  for (size_t i = 0; i < n; ++i) all[i] = he.prog.phys(i);  // canonical order out
  check(cudaMemcpyAsync(tmp_.ptr, all.data(), n * 8, cudaMemcpyHostToDevice, stream_), "upload S");
  DevBuf slice;
  slice.reserve(n * amp_);
  full_leaf_ = true;
  try {
    if (deferred_ && !dist_ && he.tree)
      evolve_tree(half, b, b + 1, slice.ptr, tmp_.as<uint64_t>(), (int64_t)n, true);
    else
      evolve_half(half, b, b + 1, slice.ptr, tmp_.as<uint64_t>(), (int64_t)n);
  } catch (...) {
    full_leaf_ = false;
    throw;
  }
  full_leaf_ = false;
  if (dist_ && world_ > 1) {  // every rank gathered its shard's entries: sum them
    ensure_comm();
    ncclResult_t r = ncclAllReduce(slice.ptr, slice.ptr, n * 2, c128_ ? ncclDouble : ncclFloat, ncclSum, comm_,
                                   stream_);
    if (r != ncclSuccess) throw Error(QSIM_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  }
  check(cudaMemcpyAsync(out, slice.ptr, n * amp_, cudaMemcpyDeviceToHost, stream_), "D2H state");
  check(cudaStreamSynchronize(stream_), "branch_state");
}

void Engine::branch_values(int half, uint64_t b, const uint64_t *idx, size_t n, void *out) {
  if (!have_circuit_) throw Error(QSIM_ESTATE, "no circuit loaded");
  if (half != 0 && half != 1) throw Error(QSIM_EINVAL, "half must be 0 (upper) or 1 (lower)");
  const int c = (int)circ_.cuts.size();
  if (c > 62 || b >= (1ull << c)) throw Error(QSIM_EINVAL, "branch out of range");
  if (!out || !idx || n == 0) throw Error(QSIM_EINVAL, "empty index list");
  HalfExec &he = half_[half];
  const int h = he.prog.h;
  std::vector<uint64_t> P(n);
  for (size_t i = 0; i < n; ++i) {
    if (idx[i] >> h) throw Error(QSIM_EINVAL, "index >= 2^h");
    P[i] = he.prog.phys(idx[i]);
  }
  ensure_device();
  DevBuf dS, slice;
  dS.reserve(n * 8);
  slice.reserve(n * amp_);
  check(cudaMemcpyAsync(dS.ptr, P.data(), n * 8, cudaMemcpyHostToDevice, stream_), "upload idx");
  if (deferred_ && !dist_ && he.tree)
    evolve_tree(half, b, b + 1, slice.ptr, dS.as<uint64_t>(), (int64_t)n, true);
  else
    evolve_half(half, b, b + 1, slice.ptr, dS.as<uint64_t>(), (int64_t)n);
  if (dist_ && world_ > 1) {
    ensure_comm();
    ncclResult_t r = ncclAllReduce(slice.ptr, slice.ptr, n * 2, c128_ ? ncclDouble : ncclFloat, ncclSum, comm_,
                                   stream_);
    if (r != ncclSuccess) throw Error(QSIM_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  }
  check(cudaMemcpyAsync(out, slice.ptr, n * amp_, cudaMemcpyDeviceToHost, stream_), "D2H values");
  check(cudaStreamSynchronize(stream_), "branch_values");
}

void Engine::info(qsim_info_t *out) const {
  std::memset(out, 0, sizeof(*out));
  out->precision = (uint32_t)prec_;
  out->have_circuit = have_circuit_ ? 1u : 0u;
  if (have_circuit_) {
    out->h_upper = circ_.h_u;
    out->h_lower = circ_.h_l;
    out->n_cuts = (uint32_t)circ_.cuts.size();
  }
  if (have_blocks_) {
    out->n_upper = Su_.size();
    out->n_lower = Sl_.size();
  }
  out->device = device_;
}

// ---------------------------------------------------------------- distributed half (f3)
// Level buffers for sharded half states, and every rank's device pointers to them (CUDA IPC
// handles exchanged with an NCCL all-gather), for the sweeps that store into a peer's shard.
void Engine::dist_buffers(size_t bytes, int nbuf) {
  if (dist_bytes_ >= bytes && (int)peer_.size() >= nbuf && (int)peer_[0].size() == world_) return;
  for (void *p : ipc_opened_) cudaIpcCloseMemHandle(p);
  ipc_opened_.clear();
  peer_.clear();
  size_t free_b = 0, total_b = 0;
  check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  size_t have = 0;
  for (auto *b : states_) have += b->bytes;
  const size_t margin = (size_t)512 << 20;
  if ((size_t)nbuf * bytes + margin > free_b + have) {
    std::ostringstream m;
    m << "distributed half: " << nbuf << " shard buffers of " << bytes << " bytes do not fit";
    throw Error(QSIM_ENOMEM, m.str());
  }
  while ((int)states_.size() < nbuf) states_.push_back(new DevBuf());
  for (int i = 0; i < nbuf; ++i) states_[i]->reserve(bytes);
  dist_bytes_ = bytes;
  peer_.assign(nbuf, std::vector<void *>(world_, nullptr));
  for (int i = 0; i < nbuf; ++i) peer_[i][rank_] = states_[i]->ptr;
  if (world_ == 1) return;
  ensure_comm();
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  std::vector<cudaIpcMemHandle_t> mine(nbuf), all((size_t)nbuf * world_);
  for (int i = 0; i < nbuf; ++i) check(cudaIpcGetMemHandle(&mine[i], states_[i]->ptr), "cudaIpcGetMemHandle");
  DevBuf dev;
  dev.reserve(hb * nbuf * (world_ + 1));
  char *send = dev.as<char>() + hb * nbuf * world_;
  check(cudaMemcpyAsync(send, mine.data(), hb * nbuf, cudaMemcpyHostToDevice, stream_), "upload IPC handles");
  ncclResult_t r = ncclAllGather(send, dev.ptr, hb * nbuf, ncclUint8, comm_, stream_);
  if (r != ncclSuccess) throw Error(QSIM_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
  check(cudaMemcpyAsync(all.data(), dev.ptr, hb * nbuf * world_, cudaMemcpyDeviceToHost, stream_), "IPC handles");
  check(cudaStreamSynchronize(stream_), "IPC handles");
  for (int q = 0; q < world_; ++q) {
    if (q == rank_) continue;
    for (int i = 0; i < nbuf; ++i) {
      void *p = nullptr;
      check(cudaIpcOpenMemHandle(&p, all[(size_t)q * nbuf + i], cudaIpcMemLazyEnablePeerAccess),
            "cudaIpcOpenMemHandle");
      peer_[i][q] = p;
      ipc_opened_.push_back(p);
    }
  }
}

// Stream-ordered barrier: an all-reduce of one word completes on every rank only after every
// rank's earlier work on its stream (the sweeps that read or write peer shards) has completed.
void Engine::dist_barrier() {
  if (world_ == 1) return;
  ensure_comm();
  dbar_.reserve(16);
  ncclResult_t r = ncclAllReduce(dbar_.ptr, dbar_.ptr, 1, ncclInt32, ncclSum, comm_, stream_);
  if (r != ncclSuccess) throw Error(QSIM_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
}

// ---------------------------------------------------------------- multi-GPU
// Records rank / world / id; the communicator itself is created at the first collective
// (ensure_comm), so the sharding logic works without a GPU.
void Engine::comm_init(int rank, int world, const void *id) {
  if (world < 1 || rank < 0 || rank >= world || !id) throw Error(QSIM_EINVAL, "bad rank / world / id");
  if (comm_) {
    ncclCommDestroy(comm_);
    comm_ = nullptr;
  }
  std::memcpy(uid_, id, sizeof(uid_));
  rank_ = rank;
  world_ = world;
  reduced_ = false;
  if (dist_ && have_circuit_) {
    compile_all();
    have_blocks_ = false;
  }
}

void Engine::ensure_comm() {
  if (comm_ || world_ == 1) return;
  ensure_device();
  ncclUniqueId uid;
  static_assert(sizeof(uid) == sizeof(uid_), "ncclUniqueId size");
  std::memcpy(&uid, uid_, sizeof(uid));
  ncclResult_t r = ncclCommInitRank(&comm_, world_, uid, rank_);
  if (r != ncclSuccess) throw Error(QSIM_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
}

void Engine::rank_range(uint64_t *b0, uint64_t *b1) const { rank_range_of(rank_, b0, b1); }

void Engine::rank_range_of(int rank, uint64_t *b0, uint64_t *b1) const {
  if (!have_circuit_) throw Error(QSIM_ESTATE, "no circuit loaded");
  const int c = (int)circ_.cuts.size();
  if (c > 62) throw Error(QSIM_EINVAL, "too many cuts");
  const unsigned __int128 B = (unsigned __int128)1 << c;
  if (dist_) {  // distributed halves: every rank runs every branch on its shard
    *b0 = 0;
    *b1 = (uint64_t)B;
    return;
  }
  // prefix groups: the branches sharing the cuts of the first two cut layers (bench.py's steps)
  int gbits = 0;
  for (size_t i = 0; i < circ_.fork_layers.size() && i < 2; ++i) gbits += circ_.fork_k[i];
  const uint64_t G = 1ull << gbits, per = (uint64_t)(B >> gbits);
  if ((uint64_t)world_ <= G) {
    *b0 = G * (uint64_t)rank / (uint64_t)world_ * per;
    *b1 = G * (uint64_t)(rank + 1) / (uint64_t)world_ * per;
    return;
  }
  *b0 = (uint64_t)(B * (unsigned)rank / (unsigned)world_);
  *b1 = (uint64_t)(B * (unsigned)(rank + 1) / (unsigned)world_);
}

// ---------------------------------------------------------------- cost model
void Engine::cost_model(uint64_t nu, uint64_t nl, double hbm_gbps, qsim_cost_t *out) {
  if (!have_circuit_) throw Error(QSIM_ESTATE, "no circuit loaded");
  if (!(hbm_gbps > 0.0)) throw Error(QSIM_EINVAL, "hbm_gbps must be > 0");
  if (!out) throw Error(QSIM_EINVAL, "null output");
  qsim_cost_t c;
  std::memset(&c, 0, sizeof(c));
  const int ncut = (int)circ_.cuts.size();
  c.n_qubits = circ_.n;
  c.h_upper = circ_.h_u;
  c.h_lower = circ_.h_l;
  c.n_cuts = (uint32_t)ncut;
  c.n_branches = std::ldexp(1.0, ncut);
  c.half_circuits = std::ldexp(1.0, ncut + 1);
  c.N_e = std::max(circ_.h_u, circ_.h_l) + (uint32_t)ncut + 1;
  double mem = (double)(183359ull << 20);  // B200 (nvidia-smi) when no device is attached yet
  if (inited_) {
    size_t f = 0, t = 0;
    if (cudaMemGetInfo(&f, &t) == cudaSuccess) mem = (double)t;
  }
  c.N_m = (uint32_t)std::floor(std::log2(mem / (double)amp_));
  c.regime = c.N_e <= c.N_m ? 0 : (c.N_e < c.n_qubits ? 1 : 2);
  c.flat_layer_evolutions = c.n_branches * 2.0 * circ_.depth;
  for (int h = 0; h < 2; ++h) {
    const HalfExec &he = half_[h];
    const HalfProgram &hp = he.prog;
    const int F = (int)hp.levels.size() - 1;
    if (!he.tree || he.plans.empty()) continue;  // small states: everything stays in shared memory
    const int lazy = lazy_depth(h, (int64_t)(h == 0 ? nu : nl));
    const double state = std::ldexp(1.0, hp.h) * (double)amp_;
    int m0 = 0;  // levels above m0 are recomputed for every level-m0 node (memory plan)
    while ((double)(F + 1 - m0) * state > mem - (512.0 * (1 << 20)) && m0 < F) ++m0;
    std::vector<int> sbits(F + 1, 0);
    for (int l = 1; l <= F; ++l) sbits[l] = sbits[l - 1] + hp.levels[l].k;
    for (int l = 0; l <= F; ++l) {
      const auto &launches = he.plans[l][l == F ? std::min<size_t>(lazy, he.plans[l].size() - 1) : 0];
      const double nodes = std::ldexp(1.0, sbits[std::max(l, m0)]);
      for (const TilePlan &tp : launches) {
        c.tree_sweeps += nodes;
        c.sweep_bytes += nodes * state * (tp.gen ? 1.0 : 2.0);
      }
    }
    if (lazy > 0) c.lazy_gathers += c.n_branches;
  }
  c.predicted_s = c.sweep_bytes / (hbm_gbps * 1e9);
  *out = c;
}

// ---------------------------------------------------------------- stats
void Engine::stats(qsim_stats_t *out) {
  if (inited_) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    resolve_events();
  }
  *out = st_;
}

void Engine::stats_reset() {
  if (inited_) resolve_events();
  st_ = qsim_stats_t{};
}

void Engine::synchronize() {
  if (!inited_) return;
  check(cudaSetDevice(device_), "cudaSetDevice");
  check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
}

// ---------------------------------------------------------------- level-synchronous tree (BFS)
// Node-batched launch of one planned sweep over 2^log2_nodes states (TMA kernel only).
void Engine::launch_nodes(const TilePlan &tp, const void *src, void *dst, int log2_nodes, int shift,
                          const ForkDev &fork, const HalfProgram &hp, bool apply_fork, uint32_t proj_bits,
                          const Diag *extra_pre) {
  if (tp.gen || !tp.swaps.empty()) throw Error(QSIM_EINVAL, "node-batched sweep of an unsupported plan");
  const int h = hp.hl;
  int pre_mode = 0;
  Diag pre;
  if (tp.use_pre) pre = tp.pre;
  if (extra_pre && apply_fork) pre = Diag::merge(pre, *extra_pre);
  if (!pre.identity()) pre_mode = 1;
  const bool timed = time_sweeps_;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    e0 = get_event();
    e1 = get_event();
    check(cudaEventRecord(e0, stream_), "cudaEventRecord");
  }
  TileSweepParams p = tp.p;
  p.no_pskip = pskip_ ? 0 : 1;
  p.pre = to_dev(pre, pre_mode != 0);
  p.ld_pm = pre_mode == 1 ? p.pre.pm : 0u;
  p.ld_pv = pre_mode == 1 ? p.pre.pv : 0u;
  p.njobs = 1;
  p.src[0] = src;
  p.dst[0] = dst;
  p.job_pv[0] = p.pre.pv;
  p.job_zm[0] = p.pre.zm;
  p.log2_nodes = log2_nodes;
  p.node_src_shift = shift;
  p.node_stride = (uint64_t)1 << h;
  p.fork = fork;
  p.fork_apply = apply_fork ? 1 : 0;
  if (zero_skip_ && proj_bits) {  // projected fork bits not yet touched in the level, outside the tile
    uint32_t outer = (h >= 32 ? ~0u : ((1u << h) - 1u)) & ~((1u << tile_low_bits(c128_)) - 1u);
    for (int j = 0; j < kHiBits; ++j) outer &= ~(1u << p.hb[j]);
    p.nb_skip = proj_bits & tp.zfix & outer;
  }
  if (pre_mode == 1) p.pre_s = make_split(pre, reg_positions(p, 0, c128_));
  const uint64_t tiles = 1ull << (p.log2_ntiles + log2_nodes);
  const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)grid_ctas());
  const int stages = sweep_kernel_ == 2 ? 2 : sweep_kernel_ == 3 ? 3 : tma_stages(tp);
  check(launch_tile_sweep_tma(p, c128_, pre_mode, tp.npass, grid, stream_, stages), "node-batched sweep launch");
  if (timed) {
    check(cudaEventRecord(e1, stream_), "cudaEventRecord");
    ev_sweep_.emplace_back(e0, e1);
    if (ev_sweep_.size() > 8192) resolve_events();
  }
  const double nodes = std::ldexp(1.0, log2_nodes);
  st_.kernel_launches++;
  st_.sweeps++;
  st_.sweep_states += (uint64_t)nodes;
  st_.layers_applied += (uint64_t)tp.layers * (uint64_t)nodes;
  st_.sweep_bytes += 2.0 * nodes * std::ldexp(1.0, h) * (double)amp_;
  st_.sweep_bytes_moved += (2.0 - (1.0 - std::ldexp(1.0, -__builtin_popcount(p.nb_skip)))) * nodes *
                           std::ldexp(1.0, h) * (double)amp_;
}

static ForkDev fork_dev(const Level &lev) {
  ForkDev f;
  std::memset(&f, 0, sizeof(f));
  f.n = lev.k;
  f.pmask = lev.pmask;
  for (int j = 0; j < lev.k; ++j) f.bit[j] = (uint8_t)lev.cut_bits[j];
  return f;
}

// Level at which the depth-first executor hands a whole subtree to the level-synchronous one
// (-1: never).  Worth it for small states, where one launch per node and sweep is launch-bound;
// the subtree's two largest levels must fit next to the depth-first buffers.
int Engine::bfs_level(int half, int m0, size_t avail) const {
  const HalfExec &he = half_[half];
  const HalfProgram &hp = he.prog;
  if (!bfs_ || dist_ || sweep_kernel_ == 1 || !he.tree || he.plans.empty()) return -1;
  if (state_bytes_ > ((size_t)256 << 20)) return -1;
  const int F = (int)hp.levels.size() - 1;
  if (F < 1) return -1;
  for (int l = 1; l <= F; ++l) {
    if (l < F && he.plans[l][0].empty()) return -1;  // only the leaf level may defer its fork
    for (const auto &v : he.plans[l])
      for (const TilePlan &tp : v)
        if (tp.gen || !tp.swaps.empty()) return -1;
  }
  std::vector<int> sbits(F + 1, 0);
  for (int l = 1; l <= F; ++l) sbits[l] = sbits[l - 1] + hp.levels[l].k;
  const size_t have = bfs_buf_[0].bytes + bfs_buf_[1].bytes;
  for (int l = m0; l < F; ++l) {
    if (sbits[F] - sbits[l] > 40) continue;
    double need = std::ldexp((double)state_bytes_, sbits[F] - sbits[l]);
    if (F - 1 > l) need += std::ldexp((double)state_bytes_, sbits[F - 1] - sbits[l]);
    if (need + (double)(256u << 20) <= (double)(avail + have)) return sbits[F] > sbits[l] ? l : -1;
  }
  return -1;
}

// The subtree below one level-m node (its state given), level by level: the first sweep of
// level l reads the parents (node >> k_l) and applies the fork per node, the others run in
// place, each as ONE node-batched launch; leaf rows go to out[leaf * nS].
void Engine::bfs_subtree(int half, int m, const void *state, void *out, const uint64_t *dS, int64_t nS) {
  HalfExec &he = half_[half];
  const HalfProgram &hp = he.prog;
  const int F = (int)hp.levels.size() - 1;
  int rel = 0;
  for (int l = m + 1; l <= F; ++l) rel += hp.levels[l].k;
  const int64_t nleaves = (int64_t)1 << rel;
  const int kF = hp.levels[F].k;
  // lazy tails: node-batched when they do not carry the fork, else one gather per leaf (few leaves)
  int lazy = nleaves <= 4096 ? lazy_depth(half, nS) : 0;
  // a lazy tail that covers the leaf level's first sweep carries the per-leaf fork: it cannot be
  // node-batched, and one launch per leaf costs more than the full batched pass it saves
  if (lazy > 0 && hp.levels[F].sweeps.size() <= (size_t)lazy && nleaves > 16) lazy = 0;
  bfs_buf_[F & 1].reserve(state_bytes_ << rel);
  if (F - 1 > m) bfs_buf_[(F & 1) ^ 1].reserve(state_bytes_ << (rel - kF));
  const void *src = state;
  int sb = 0;
  bool pending = false;
  for (int l = m + 1; l <= F; ++l) {
    const Level &lev = hp.levels[l];
    const auto &launches = he.plans[l][l == F ? std::min<size_t>((size_t)lazy, he.plans[l].size() - 1) : 0];
    if (launches.empty()) {  // leaf level without full passes: its fork is applied in the gather
      pending = true;
      break;
    }
    sb += lev.k;
    void *dst = bfs_buf_[l & 1].ptr;
    const ForkDev f = fork_dev(lev);
    uint32_t proj = 0;  // P-role cut bits (a P_b child is zero off its branch bits)
    for (int j = 0; j < lev.k; ++j)
      if ((lev.pmask >> j) & 1u) proj |= 1u << lev.cut_bits[j];
    for (size_t i = 0; i < launches.size(); ++i)
      launch_nodes(launches[i], i == 0 ? src : dst, dst, sb, i == 0 ? lev.k : 0, f, hp, i == 0, proj);
    src = dst;
  }
  if (lazy == 0) {
    ForkDev f;
    std::memset(&f, 0, sizeof(f));
    if (pending) f = fork_dev(hp.levels[F]);
    check(launch_gather_nodes(src, (uint64_t)1 << hp.hl, pending ? kF : 0, nleaves, dS, nS, out, f, c128_, stream_),
          "gather nodes launch");
    st_.kernel_launches++;
    return;
  }
  const Level &levF = hp.levels[F];
  static const bool batch_lazy = !(std::getenv("QSIM_BATCH_LAZY") && std::getenv("QSIM_BATCH_LAZY")[0] == '0');
  if (batch_lazy && !pending && levF.sweeps.size() > (size_t)lazy) {
    // the lazy layers do not carry the fork: one node-batched launch per lazy stage for all leaves
    const size_t n = levF.sweeps.size();
    LazyLayer lld = lazy_layer(levF.sweeps[n - 1], levF.sweeps[n - 1].pre);
    lld.node_stride = (uint64_t)1 << hp.hl;
    lld.nper = nS;
    if (lazy == 1) {
      check(launch_gather_layer(src, dS, nS * nleaves, out, lld, c128_, stream_), "gather_layer launch");
      st_.kernel_launches++;
    } else {
      LazyLayer ll1 = lazy_layer(levF.sweeps[n - 2], levF.sweeps[n - 2].pre);
      const int64_t ncone = nS << lld.k;
      ll1.node_stride = (uint64_t)1 << hp.hl;
      ll1.nper = ncone;
      cone_idx_.reserve((size_t)ncone * 8);
      cone_val_.reserve((size_t)ncone * (size_t)nleaves * amp_);
      check(launch_cone_indices(dS, nS, lld, cone_idx_.as<uint64_t>(), stream_), "cone launch");
      check(launch_gather_layer(src, cone_idx_.as<uint64_t>(), ncone * nleaves, cone_val_.ptr, ll1, c128_, stream_),
            "gather_layer launch");
      check(launch_gather_layer_compact(cone_val_.ptr, dS, nS * nleaves, out, lld, c128_, stream_),
            "gather_layer_compact launch");
      st_.kernel_launches += 3;
    }
    st_.lazy_gathers += (uint64_t)nleaves;
    return;
  }
  for (int64_t leaf = 0; leaf < nleaves; ++leaf) {
    const uint64_t child = (uint64_t)leaf & ((1ull << kF) - 1ull);
    const char *psi = (const char *)src + (size_t)(pending ? (leaf >> kF) : leaf) * state_bytes_;
    gather_leaf(half, child, psi, dS, nS, (char *)out + (size_t)leaf * (size_t)nS * amp_, lazy);
  }
}

// ---------------------------------------------------------------- multi-part partitions (f4)
// SURVEY §8(f) f4; PAPER.md P:114 ("dividing the circuit into three or four parts is more
// effective if the circuit depth is small") and Fig. 3.  Parts are bands of rows
// [r_k, r_{k+1}); Eq. 1 is applied to every CZ crossing a boundary (upper endpoint P_b,
// lower endpoint I / Z, as the bipartition does; DESIGN.md R-f4).  Part k depends only on the
// bits of its two boundaries, so it is one branch tree over those cuts (prefix-shared like a
// half), and the amplitudes of sampled blocks are the chain contraction
//   A[i_0, .., i_{t-1}] = sum_{beta_0..beta_{t-2}} X_0[beta_0, i_0] X_1[beta_0, beta_1, i_1] ...
//                                                    X_{t-1}[beta_{t-2}, i_{t-1}],
// evaluated right to left as batched fp64 GEMMs (branch_gemm_kernel with a batch index).
Engine::MultiPart Engine::multipart_layout(uint32_t t, const uint32_t *row_cuts) const {
  if (!have_circuit_) throw Error(QSIM_ESTATE, "no circuit loaded");
  if (t < 2 || t > 8) throw Error(QSIM_EINVAL, "n_parts must be in 2..8");
  if (!row_cuts) throw Error(QSIM_EINVAL, "row_cuts is NULL");
  MultiPart mp;
  mp.bounds.push_back(0);
  for (uint32_t j = 0; j + 1 < t; ++j) mp.bounds.push_back(row_cuts[j]);
  mp.bounds.push_back(circ_.rows);
  for (uint32_t k = 0; k < t; ++k) {
    if (mp.bounds[k] >= mp.bounds[k + 1])
      throw Error(QSIM_EINVAL, "row_cuts must be strictly increasing inside (0, rows)");
    if ((mp.bounds[k + 1] - mp.bounds[k]) * circ_.cols > 32)
      throw Error(QSIM_EINVAL, "each part must have at most 32 qubits");
  }
  auto part_of = [&](uint32_t q) {
    const uint32_t r = q / circ_.cols;
    uint32_t k = 0;
    while (r >= mp.bounds[k + 1]) ++k;
    return (int)k;
  };
  struct XC {
    int layer;
    uint32_t qu, ql;
    int j;
  };
  std::vector<XC> xs;
  for (const qsim_gate &g : circ_.gates) {
    if (g.kind != QSIM_CZ) continue;
    const int pa = part_of(g.q0), pb = part_of(g.q1);
    if (pa == pb) continue;
    xs.push_back(XC{(int)g.layer, std::min(g.q0, g.q1), std::max(g.q0, g.q1), std::min(pa, pb)});
  }
  std::sort(xs.begin(), xs.end(),
            [](const XC &a, const XC &b) { return a.layer != b.layer ? a.layer < b.layer : a.qu < b.qu; });
  mp.c.assign(t - 1, 0);
  mp.cuts.resize(t);
  mp.bits.resize(t);
  for (const XC &x : xs) {
    const int idx = mp.c[x.j]++;
    mp.cuts[x.j].push_back(PartCut{x.layer, x.qu, true});  // part above the boundary: P_b
    mp.bits[x.j].push_back({x.j, idx});
    mp.cuts[x.j + 1].push_back(PartCut{x.layer, x.ql, false});  // part below: Z^b
    mp.bits[x.j + 1].push_back({x.j, idx});
  }
  return mp;
}

void Engine::multipart_plan(uint32_t t, const uint32_t *row_cuts, uint32_t *part_qubits, uint32_t *boundary_cuts,
                            double *log2_states) {
  const MultiPart mp = multipart_layout(t, row_cuts);
  double states = 0.0;
  for (uint32_t k = 0; k < t; ++k) {
    const uint32_t nq = (mp.bounds[k + 1] - mp.bounds[k]) * circ_.cols;
    if (part_qubits) part_qubits[k] = nq;
    states += std::ldexp(1.0, (int)nq + (int)mp.cuts[k].size());
  }
  for (uint32_t j = 0; j + 1 < t; ++j)
    if (boundary_cuts) boundary_cuts[j] = (uint32_t)mp.c[j];
  if (log2_states) *log2_states = std::log2(states);
}

void Engine::multipart_amplitudes(uint32_t t, const uint32_t *row_cuts, const uint64_t *blocks, const size_t *n_block,
                                  void *amps) {
  if (dist_) throw Error(QSIM_EINVAL, "multi-part partitions do not combine with distributed halves");
  if (!blocks || !n_block) throw Error(QSIM_EINVAL, "blocks / n_block is NULL");
  const MultiPart mp = multipart_layout(t, row_cuts);
  std::vector<int> nq(t);
  std::vector<int64_t> ns(t);
  std::vector<size_t> off(t + 1, 0);
  double total = 1.0;
  for (uint32_t k = 0; k < t; ++k) {
    nq[k] = (int)((mp.bounds[k + 1] - mp.bounds[k]) * circ_.cols);
    ns[k] = (int64_t)n_block[k];
    validate_block(blocks + off[k], n_block[k], (uint32_t)nq[k], "part");
    off[k + 1] = off[k] + n_block[k];
    total *= (double)ns[k];
    if ((int)mp.cuts[k].size() > 30) throw Error(QSIM_EINVAL, "a part has more than 30 cut bits");
  }
  if (total * 16.0 > std::ldexp(1.0, 36)) throw Error(QSIM_EINVAL, "amplitude block larger than 64 GiB");

  // compile the part programs (branch trees over each part's cuts) into half_[2 + k]; reused while
  // the circuit, the options and the row cuts are unchanged (the relabelling search is not free)
  const bool cached = mp_gen_ == plan_gen_ && mp_key_ == mp.bounds && half_.size() == 2 + (size_t)t;
  if (!cached) {
    while (half_.size() > 2) half_.pop_back();
    mp_key_ = mp.bounds;
    mp_gen_ = plan_gen_;
  }
  for (uint32_t k = 0; k < t && !cached; ++k) {
    half_.emplace_back();
    HalfExec &he = half_.back();
    std::vector<int> id(nq[k]);
    for (int b = 0; b < nq[k]; ++b) id[b] = b;
    const uint32_t lo = mp.bounds[k] * circ_.cols, hi = mp.bounds[k + 1] * circ_.cols;
    he.prog = compile_part(circ_, lo, hi, k + 1 < t, mp.cuts[k], std::vector<std::vector<int>>(circ_.depth + 2, id), id);
    compile_plans(he);
    if (he.tree) {
      const std::vector<int> perm = choose_perm(he, ns[k]);
      bool ident = true;
      for (size_t b = 0; b < perm.size(); ++b) ident = ident && perm[b] == (int)b;
      if (!ident) {
        he.prog = compile_part(circ_, lo, hi, k + 1 < t, mp.cuts[k],
                               std::vector<std::vector<int>>(circ_.depth + 2, perm), perm);
        compile_plans(he);
      }
    }
  }

  ensure_device();
  // evolve every part's branches; X_k[(beta_{k-1} << c_k) | beta_k, i] in fp64
  while (mp_X_.size() < t) mp_X_.emplace_back(new DevBuf());
  for (uint32_t k = 0; k < t; ++k) {
    const int hidx = 2 + (int)k;
    const HalfProgram &hp = half_[hidx].prog;
    const int cp = hp.ncuts;
    const int64_t nrows = (int64_t)1 << cp;
    const int c_up = k > 0 ? mp.c[k - 1] : 0, c_dn = k + 1 < t ? mp.c[k] : 0;
    std::vector<uint64_t> P((size_t)ns[k]);
    for (int64_t i = 0; i < ns[k]; ++i) P[i] = hp.phys(blocks[off[k] + i]);
    std::vector<uint32_t> rm((size_t)nrows);
    for (int64_t r = 0; r < nrows; ++r) {
      uint32_t up = 0, dn = 0;
      for (int j = 0; j < cp; ++j) {
        const uint32_t bit = (uint32_t)(r >> (cp - 1 - j)) & 1u;
        const auto &bj = mp.bits[k][j];
        if (bj.first + 1 == (int)k)
          up |= bit << (c_up - 1 - bj.second);
        else
          dn |= bit << (c_dn - 1 - bj.second);
      }
      rm[r] = (up << c_dn) | dn;
    }
    mp_dS_.reserve((size_t)ns[k] * 8);
    mp_rowmap_.reserve((size_t)nrows * 4);
    mp_slice_.reserve((size_t)nrows * ns[k] * amp_);
    check(cudaMemcpyAsync(mp_dS_.ptr, P.data(), P.size() * 8, cudaMemcpyHostToDevice, stream_), "upload part block");
    check(cudaMemcpyAsync(mp_rowmap_.ptr, rm.data(), rm.size() * 4, cudaMemcpyHostToDevice, stream_),
          "upload rowmap");
    evolve_half(hidx, 0, (uint64_t)nrows, mp_slice_.ptr, mp_dS_.as<uint64_t>(), ns[k]);
    mp_X_[k]->reserve((size_t)nrows * ns[k] * 16);
    check(launch_permute_rows(mp_slice_.ptr, c128_, mp_rowmap_.as<uint32_t>(), nrows, ns[k], mp_X_[k]->as<double>(),
                              stream_),
          "permute rows");
    st_.kernel_launches++;
    st_.branches_evolved += (uint64_t)nrows;
    check(cudaStreamSynchronize(stream_), "multi-part evolve");  // P, rm are host temporaries
  }

  // chain contraction split at boundary js: left product L_js[beta_js, (i_0..i_js)] (left to right,
  // GEMM outputs laid out [beta_k][i_0..i_{k-1}][i_k]), right product R[beta_js, (i_{js+1}..)]
  // (right to left, batched over beta_{k-1}), then one GEMM over beta_js.  js minimises the flops.
  auto C2 = [&](int j) { return std::ldexp(1.0, mp.c[j]); };
  int js = 0;
  double best = -1.0;
  for (int j = 0; j + 1 < (int)t; ++j) {
    double P = (double)ns[0], fl = 0.0;
    for (int k = 1; k <= j; ++k) {
      fl += 8.0 * P * C2(k) * (double)ns[k] * C2(k - 1);
      P *= (double)ns[k];
    }
    double Qr = (double)ns[t - 1];
    for (int k = (int)t - 2; k > j; --k) {
      fl += 8.0 * C2(k - 1) * (double)ns[k] * Qr * C2(k);
      Qr *= (double)ns[k];
    }
    fl += 8.0 * P * Qr * C2(j);
    if (best < 0.0 || fl < best) best = fl, js = j;
  }
  auto gemm_timed = [&](const double *U, const double *L, int64_t K, int64_t M, int64_t N, DevBuf &out, int64_t batch,
                        int64_t N2) {
    const size_t bytes = (size_t)batch * (size_t)M * (size_t)N * 16;
    out.reserve(bytes);
    check(cudaMemsetAsync(out.ptr, 0, bytes, stream_), "zero contraction");
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (time_sweeps_) {
      e0 = get_event();
      e1 = get_event();
      check(cudaEventRecord(e0, stream_), "cudaEventRecord");
    }
    check(launch_branch_gemm_batched(U, L, K, M, N, out.as<double>(), batch, stream_, N2), "contraction gemm");
    if (time_sweeps_) {
      check(cudaEventRecord(e1, stream_), "cudaEventRecord");
      ev_gemm_.emplace_back(e0, e1);
    }
    st_.kernel_launches++;
    st_.gemm_flops += 8.0 * (double)batch * (double)M * (double)N * (double)K;
  };
  // left: L_0 = X_0 [beta_0, i_0]
  const double *Lp = mp_X_[0]->as<double>();
  int64_t P = ns[0];
  for (int k = 1; k <= js; ++k) {
    DevBuf &out = mp_T_[k & 1];
    gemm_timed(Lp, mp_X_[k]->as<double>(), (int64_t)1 << mp.c[k - 1], P, ((int64_t)1 << mp.c[k]) * ns[k], out, 1,
               ns[k]);
    Lp = out.as<double>();
    P *= ns[k];
  }
  // right: R_{t-1} = X_{t-1} [beta_{t-2}, i_{t-1}]
  const double *T = mp_X_[t - 1]->as<double>();
  int64_t Nrest = ns[t - 1];
  for (int k = (int)t - 2; k > js; --k) {
    DevBuf &out = mp_T_[2 + (k & 1)];
    gemm_timed(mp_X_[k]->as<double>(), T, (int64_t)1 << mp.c[k], ns[k], Nrest, out, (int64_t)1 << mp.c[k - 1], 0);
    T = out.as<double>();
    Nrest *= ns[k];
  }
  gemm_timed(Lp, T, (int64_t)1 << mp.c[js], P, Nrest, mp_A_, 1, 0);
  const DevBuf &Aout = mp_A_;
  const size_t n = (size_t)P * (size_t)Nrest;
  if (amps) {
    if (c128_) {
      check(cudaMemcpyAsync(amps, Aout.ptr, n * 16, cudaMemcpyDeviceToHost, stream_), "D2H amplitudes");
    } else {
      tmp_.reserve(n * 8);
      check(launch_cast_c128_to_c64(Aout.as<double>(), (int64_t)(2 * n), tmp_.as<float>(), stream_), "cast");
      st_.kernel_launches++;
      check(cudaMemcpyAsync(amps, tmp_.ptr, n * 8, cudaMemcpyDeviceToHost, stream_), "D2H amplitudes");
    }
  }
  check(cudaStreamSynchronize(stream_), "multi-part amplitudes");
}

}  // namespace qsim

