// Per-context engine: device memory plan, branch-tree executor, reconstruction,
// sampling, NCCL reduction of partial amplitude blocks.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <deque>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/qsim.h"
#include "kernels.h"
#include "program.h"

namespace qsim {

struct Error : std::runtime_error {
  qsim_status code;
  Error(qsim_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};

struct DevBuf {
  void *ptr = nullptr;
  size_t bytes = 0;
  void reserve(size_t n);  // grows (re-allocates without preserving contents)
  void release();
  template <typename T>
  T *as() const { return reinterpret_cast<T *>(ptr); }
  ~DevBuf() { release(); }
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
};

// One planned sweep launch of one layer (TileSweepParams): the TMA-pipelined sweep (default) or
// the register-only one (QSIM_OPT_SWEEP_KERNEL 1).  A layer wider than the tile is split into
// several launches.
struct TilePlan {
  std::vector<std::pair<int, int>> swaps;  // distributed half: (local bit, global bit index) after it
  TileSweepParams p;   // src/dst/job fields filled at launch
  int npass = 1;
  int layers = 1;        // gate layers completed by this launch
  bool use_pre = false;  // the launch applies its pre diagonal (fork diagonal merged at launch)
  bool gen = false;
  Diag pre;
  std::vector<int> pass0_regs;  // global bits of the pass-0 register slots (pre DiagSplit)
  uint32_t targets = ~0u;  // bits this launch applies gates on (all: unknown)
  uint32_t zfix = 0;       // fork bits of the level not targeted by an earlier launch of the level
  // host forms for the sibling-flip executor (Engine::flip_node): the post diagonal (identity
  // except on the last launch of a sweep), the Y^1/2 targets, the sweep's index in its level
  Diag post;
  uint32_t sy_targets = 0;
  int sweep = 0;
};


// The branch tree of one half for one placement of its forks (Engine::choose_tree): the
// program (levels = the distinct fork-apply layers) and its tile plans [level][lazy skip 0..2].
struct TreeVariant {
  HalfProgram prog;
  std::vector<std::vector<std::vector<TilePlan>>> plans;
};

// Fork placement chosen for one aligned block of branches: apply[g] = layer at whose input cut
// g's P_b / Z^b is applied; qmask = cuts pinned in addition to the block's fixed top bits (the
// executor loops over their values); cost in full-sweep units; points = branching levels.
struct TreeChoice {
  std::vector<int> apply;
  std::vector<int> qlist;
  double cost = 0;
  int points = 0;
};

struct HalfExec {
  HalfProgram prog;
  // deferred-fork trees (non-distributed tree halves): gate layers of the half, first target
  // layer of every cut, compiled variants by apply vector
  std::vector<int> glayers, ft;
  std::map<std::vector<int>, std::unique_ptr<TreeVariant>> variants;
  bool tree = false;                                // tile sweeps (true) or the small kernel
  std::vector<std::vector<std::vector<TilePlan>>> plans;  // [level][lazy skip] -> launches
  // small kernel program on the device
  DevBuf d_levels, d_sweeps;
  bool uploaded = false;
};

class Engine {
 public:
  Engine(qsim_precision prec, int device);
  ~Engine();

  std::string last_error;

  void set_option(int key, int64_t value);
  void set_stream(void *s);
  void load_circuit(uint32_t rows, uint32_t cols, uint32_t depth, const qsim_gate *gates,
                    size_t n_gates, uint32_t cut_row, const uint32_t *cut_layers, size_t n_cut_layers);
  void partition(uint32_t *n_cuts, uint64_t *n_branches, qsim_cut *cuts) const;
  void set_blocks(const uint64_t *up, size_t nu, const uint64_t *lo, size_t nl);
  void check_blocks(const uint64_t *up, size_t nu, const uint64_t *lo, size_t nl) const;
  void evolve_range(uint64_t b0, uint64_t b1);
  void reset_block();
  void amplitudes(void *amps);
  void sample(uint64_t seed, size_t n, uint64_t *out, double *mass);
  void sample_probs(const double *p, const uint64_t *up, size_t nu, const uint64_t *lo, size_t nl,
                    uint32_t hl, uint64_t seed, size_t n, uint64_t *out, double *mass);
  void porter_thomas(const double *p, size_t n, uint32_t n_qubits, double z_lo, double z_hi, uint32_t n_bins,
                     uint64_t *hist, double *expected, qsim_pt_t *out);
  void branch_sum(const void *U, const void *L, size_t nb, size_t nu, size_t nl, void *A);
  void branch_state(int half, uint64_t b, void *out);
  void branch_values(int half, uint64_t b, const uint64_t *idx, size_t n, void *out);
  void info(qsim_info_t *out) const;
  void comm_init(int rank, int world, const void *id);
  void rank_range(uint64_t *b0, uint64_t *b1) const;
  void rank_range_of(int rank, uint64_t *b0, uint64_t *b1) const;
  void cost_model(uint64_t nu, uint64_t nl, double hbm_gbps, qsim_cost_t *out);
  // multi-part partitions (Fig. 3)
  void multipart_plan(uint32_t n_parts, const uint32_t *row_cuts, uint32_t *part_qubits, uint32_t *boundary_cuts,
                      double *log2_states);
  void multipart_amplitudes(uint32_t n_parts, const uint32_t *row_cuts, const uint64_t *blocks,
                            const size_t *n_block, void *amps);
  void stats(qsim_stats_t *out);
  void stats_reset();
  void synchronize();

  bool have_circuit() const { return have_circuit_; }

 private:
  qsim_precision prec_;
  bool c128_;
  size_t amp_;  // bytes per amplitude
  int device_;
  bool inited_ = false;
  cudaStream_t stream_ = nullptr;
  cudaStream_t own_stream_ = nullptr;
  int num_sms_ = 148;
  int occ1_ = 2, occ2_ = 2;
  int mode_ = 0;
  int64_t mem_budget_ = 0;
  int sweep_kernel_ = 0;  // 0: TMA sweep (auto stages), 1: register-only, 2 / 3: TMA with 2 / 3 stages
  int lazy_depth_ = 2;      // up to this many trailing leaf sweeps evaluated at the sampled indices
  bool full_leaf_ = false; // qsim_branch_state: materialise the complete leaf
  bool time_sweeps_ = false;
  // distributed half (§2.3.3): every half state is sharded over the
  // communicator's ranks by its top gbits_ physical bits; all ranks run every branch
  bool dist_ = false;
  int gbits_ = 0;
  std::vector<std::vector<void *>> peer_;  // [level buffer][rank]: device pointers (CUDA IPC)
  std::vector<void *> ipc_opened_;
  size_t dist_bytes_ = 0;
  DevBuf dbar_;
  DevBuf bfs_buf_[2];
  std::vector<std::unique_ptr<DevBuf>> mp_X_;  // multi-part contraction operands (kept between calls)
  DevBuf mp_dS_, mp_slice_, mp_rowmap_, mp_T_[4], mp_A_;
  std::vector<uint32_t> mp_key_;  // row bounds of the compiled parts in half_[2..]
  uint64_t plan_gen_ = 0, mp_gen_ = ~0ull;

  bool have_circuit_ = false;
  Circuit circ_;
  std::deque<HalfExec> half_;  // [0] upper, [1] lower half; [2 + k] part k of a multi-part partition (f4)

  bool have_blocks_ = false;
  std::vector<uint64_t> Su_, Sl_;
  DevBuf d_Su_, d_Sl_;
  DevBuf d_Sp_[2];  // the blocks in each half's physical bit order (gathers)
  DevBuf A_acc_;  // double2 [nu, nl]
  DevBuf A_tot_;  // reduced block (rank 0 with a communicator)
  bool reduced_ = false;
  DevBuf U_, L_;  // slices
  DevBuf cone_idx_, cone_val_;  // two-layer lazy tail
  std::vector<DevBuf *> states_;
  size_t state_bytes_ = 0;
  // sampler
  DevBuf p_, C_, r_, R_, W_, draws_, tmp_;
  DevBuf pt_;  // Porter-Thomas analyzer scratch

  // comm
  ncclComm_t comm_ = nullptr;
  int rank_ = 0, world_ = 1;
  unsigned char uid_[128] = {};
  void ensure_comm();

  // stats
  qsim_stats_t st_{};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_sweep_, ev_gemm_;
  std::vector<cudaEvent_t> ev_pool_;

  // small H2D uploads without a stream sync: the data is copied into a pinned staging slot whose copy is
  // fenced by an event; a slot is reused only once that event completed (the host keeps running ahead)
  struct Staging {
    void *host = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
  };
  std::vector<Staging> staging_;
  void upload_async(void *dst, const void *src, size_t bytes);
  void ensure_device();
  void check(cudaError_t e, const char *what);
  void compile_plans(HalfExec &he);
  void compile_all();                       // both halves for the current options / world
  void plan_distributed(HalfExec &he);      // layout schedule with fused local/global swaps
  void dist_buffers(size_t bytes, int nbuf);  // level buffers + IPC peer pointers
  void dist_barrier();                      // stream-ordered barrier over the ranks
  std::vector<int> choose_perm(const HalfExec &he, int64_t nS = 0, const std::vector<double> *layer_w = nullptr) const;
  std::vector<double> deferred_layer_weights(int half, int64_t nS);
  int lazy_depth_of(const HalfProgram &hp, int64_t nS) const;
  int64_t perm_ns_[2] = {0, 0};  // block sizes the relabelling of each half was chosen for
  std::vector<TilePlan> level_launches(const HalfProgram &hp, const Level &lev, size_t n);
  std::vector<TilePlan> legacy_plans(const HalfProgram &hp, const Sweep &sw);
  void upload_small(HalfExec &he);
  void ensure_states(int half, int nbuf);
  int materialized_from(int half, size_t free_bytes, int *nbuf);

  // deferred-fork tree executor (non-distributed tree halves)
  void plan_levels(const HalfProgram &hp, std::vector<std::vector<std::vector<TilePlan>>> &plans, bool all_skips);
  int tree_lazy(int half, int64_t nS) const;
  int tree_lazy_of(const HalfProgram &hp, int64_t nS) const;
  TreeChoice choose_tree(int half, int m, int lz, int64_t nS, int nbuf, bool allow_gather) const;
  TreeVariant &variant(int half, const std::vector<int> &apply, const std::vector<char> &roles);
  // canonical: P_b on the upper endpoint of every cut (the branch states of qsim_branch_state /
  // qsim_branch_values); else the per-cut roles_ of the reconstruction (choose_roles)
  // flip: the sibling-flip executor may run the blocks (flip_node); zz: Z^b forks on the upper
  // endpoints of the blocks' free cuts (the lower slices then take the Walsh-Hadamard transform)
  void evolve_tree(int half, uint64_t b0, uint64_t b1, void *slice, const uint64_t *dS, int64_t nS,
                   bool canonical = false, bool flip = false, bool zz = false);
  void evolve_block(int half, uint64_t b0, int m, void *slice, const uint64_t *dS, int64_t nS,
                    const std::vector<char> &roles, bool flip = false);
  // ---- sibling-flip executor (DESIGN.md §5 "Sibling flips").  A node state is a buffer seen
  // through a bit flip and a diagonal: V(x) = phi(x) * buf[x ^ m].
  struct VState {
    int buf = 0;
    uint64_t m = 0;
    Diag phi;
    bool has_phi = false;
  };
  struct Executed {  // a launch as run (pre / post as passed to launch_plan), for its inverse
    const TilePlan *tp;
    Diag pre, post;
  };
  bool flip_half(int half) const;
  bool run_tree_frames(int half, const TreeVariant &v, const std::vector<int> &pin, int m, void *slice,
                       const uint64_t *dS, int64_t nS, int nbuf);
  bool frames_ = !(std::getenv("QSIM_FRAMES") && std::getenv("QSIM_FRAMES")[0] == '0');
  // expansions of a breaking frame into a sum of frames per term (QSIM_FRAME_EXPAND; 0: real splits only)
  int expand_depth_ = std::getenv("QSIM_FRAME_EXPAND") ? std::atoi(std::getenv("QSIM_FRAME_EXPAND")) : 6;
  long long nterms_ = 0;
  // frame basis (qsim_evolve_range, world 1): the lower half's leaves as sparse combinations of the rows of
  // its distinct frames; the GEMM then contracts over those rows (QSIM_FRAME_BASIS=0: off, A/B)
  struct BasisEntry {
    uint32_t row, t;
    double cr, ci;
  };
  struct BasisAbort {};
  bool basis_enabled_ = !(std::getenv("QSIM_FRAME_BASIS") && std::getenv("QSIM_FRAME_BASIS")[0] == '0');
  // shared basis for up to this many ranks (0: off; half pairs with a split basis measured faster at N = 2)
  int shared_basis_max_ = std::getenv("QSIM_SHARED_BASIS_MAX") ? std::atoi(std::getenv("QSIM_SHARED_BASIS_MAX")) : 0;
  bool basis_on_ = false;
  DevBuf *basis_rows_ = nullptr;
  int64_t basis_cap_ = 0, basis_T_ = 0;
  uint64_t basis_row0_ = 0;
  int basis_points_ = 0;
  std::vector<BasisEntry> basis_entries_;
  DevBuf basis_off_, basis_src_, basis_coef_;
  DevBuf basis_xoff_, basis_xsrc_, basis_xcoef_, basis_hdr_;  // half pairs: the partner's share
  // frame gathers through pre-gathered rows of the distinct flips (QSIM_FLIP_ROWS=0: scattered, A/B)
  bool flip_rows_ = !(std::getenv("QSIM_FLIP_ROWS") && std::getenv("QSIM_FLIP_ROWS")[0] == '0');
  DevBuf flip_rows_buf_, flip_idx_buf_;
  TreeChoice flip_choice(int half, int m) const;
  bool run_tree_flip(int half, const TreeVariant &v, int lz, const std::vector<int> &pin, int m, void *slice,
                     const uint64_t *dS, int64_t nS, int nbuf);
  void flip_exec(const std::vector<const TilePlan *> &tps, const Diag &fork, const VState &in, int dst,
                 const HalfProgram &hp, std::vector<Executed> *rec);
  void flip_undo(const std::vector<Executed> &rec, int buf, const HalfProgram &hp);
  bool flip_ = !(std::getenv("QSIM_FLIP") && std::getenv("QSIM_FLIP")[0] == '0');
  int flip_max_nb_ = -1;  // QSIM_OPT_FLIP_NB (tests): at most this many extra buffers (in-place + undo beyond)
  void choose_roles();
  std::vector<char> roles_;  // per cut: 1 = P on the upper endpoint (empty: all 1)
  bool roles_chosen_ = false;
  // off by default: same-box A/B within noise (C5 +0.9 %, C4 -2 %); QSIM_ROLES=1 on
  bool roles_auto_ = std::getenv("QSIM_ROLES") && std::getenv("QSIM_ROLES")[0] == '1';
  void run_tree(int half, const TreeVariant &v, int lz, const std::vector<int> &pin, int m, void *slice,
                const uint64_t *dS, int64_t nS, size_t bfs_avail);
  void gather_tree(const TreeVariant &v, int lz, int M, const std::vector<int> &pin, const void *psi,
                   uint64_t bacc, int m, void *slice, const uint64_t *dS, int64_t nS, uint64_t xmask = 0,
                   const Diag *phi = nullptr);
  // level-synchronous subtree of a tree path below level l (node-batched sweeps; small states)
  bool bfs_tree(const TreeVariant &v, int lz, int M, const std::vector<int> &skip, const std::vector<int> &pin,
                int l, const void *state, uint64_t bacc, int m, void *slice, const uint64_t *dS, int64_t nS,
                size_t avail);
  DevBuf rowmap_;
  DevBuf lazy_idx_[2], lazy_val_[2];  // cone index lists / stage values of the lazy tail (<= 3 stages)
  std::vector<uint64_t> lazy_idx_key_;  // what lazy_idx_ holds (gather_tree), valid within one evolve_block
  bool lazy_idx_valid_ = false;
  bool deferred_ = !(std::getenv("QSIM_DEFER") && std::getenv("QSIM_DEFER")[0] == '0');
  int max_ctas_ = 0;  // QSIM_OPT_MAX_CTAS (tests)
  // deferred forks on a bit the sweep targets are folded into that gate (QSIM_ABSORB=0: off, A/B)
  bool absorb_ = !(std::getenv("QSIM_ABSORB") && std::getenv("QSIM_ABSORB")[0] == '0');
  // rows / tiles the pre projector zeroes are not loaded (QSIM_PSKIP=0: off, A/B only)
  bool pskip_ = !(std::getenv("QSIM_PSKIP") && std::getenv("QSIM_PSKIP")[0] == '0');
  uint32_t skip_pm_last_ = 0;  // known-zero tile mask of the last planned launch (stats)
  int grid_ctas() const { return max_ctas_ > 0 ? std::min(max_ctas_, num_sms_) : num_sms_; }

  // distributed halves (f3): depth-first over the shards, buffer pairs only for kept levels
  void evolve_half_dist(int half, uint64_t b0, uint64_t b1, void *slice, const uint64_t *dS, int64_t nS);
  int run_level_dist(int half, int level, uint64_t child, int src, int pair, int skip);
  int dist_pairs_ = 0;

  // executor
  void evolve_half(int half, uint64_t b0, uint64_t b1, void *slice, const uint64_t *dS, int64_t nS);
  // half pairs over two ranks (multi-GPU with the frame executor; QSIM_PAIRS=0: off, A/B)
  bool evolve_pair(uint64_t b0, uint64_t b1);
  bool pairs_ = !(std::getenv("QSIM_PAIRS") && std::getenv("QSIM_PAIRS")[0] == '0');
  // level-synchronous (BFS) variant for a whole tree whose two largest consecutive levels fit:
  // every sweep of level l runs once over all 2^{sbits_l} node states (node-batched TMA launch)
  int bfs_level(int half, int m0, size_t avail) const;
  void bfs_subtree(int half, int m, const void *state, void *out, const uint64_t *dS, int64_t nS);
  void launch_nodes(const TilePlan &tp, const void *src, void *dst, int log2_nodes, int shift, const ForkDev &fork,
                    const HalfProgram &hp, bool apply_fork = true, uint32_t proj_bits = 0,
                    const Diag *extra_pre = nullptr);
  bool bfs_ = true;  // QSIM_OPT_BFS: level-synchronous subtrees for small states
  // generated (write-only) sweeps through the TMA kernel's PRE = 2 variant (QSIM_GEN_TMA=0: the
  // register kernel, A/B only)
  bool gen_tma_ = !(std::getenv("QSIM_GEN_TMA") && std::getenv("QSIM_GEN_TMA")[0] == '0');
  // known-zero tiles of projected fork children are not read (QSIM_ZERO_SKIP=0: off, A/B only)
  bool zero_skip_ = !(std::getenv("QSIM_ZERO_SKIP") && std::getenv("QSIM_ZERO_SKIP")[0] == '0');
  const void *run_level(int half, int level, uint64_t child, const void *src, void *dst, int skip);
  int lazy_depth(int half, int64_t nS) const;
  int tma_stages(const TilePlan &tp) const;
  void launch_plan(const TilePlan &tp, const Diag &fork, bool first_chunk_of_level, const void *src,
                   void *dst, const HalfProgram &hp, int out_buf = -1, const Diag *child_fork = nullptr,
                   const Diag *pre_ov = nullptr, const Diag *post_ov = nullptr);
  void gather_leaf(int half, uint64_t child_last, const void *psi, const uint64_t *dS, int64_t nS,
                   void *out_row, int depth);
  void gemm(const void *U, const void *L, int64_t K, int64_t M, int64_t N, double *A);
  double *reduced_block();
  void run_sampler(const double *A, const double *p, int64_t M, int64_t N, int64_t row0, int64_t nrows,
                   bool collective, const uint64_t *dSu, const uint64_t *dSl, uint32_t hl, uint64_t seed,
                   size_t n, uint64_t *out, double *mass);
  DevBuf A_part_;  // this rank's rows of the reduced block (multi-GPU sampling)

  struct MultiPart {
    std::vector<uint32_t> bounds;                        // row bounds r_0 = 0 < ... < r_t = rows
    std::vector<int> c;                                  // cuts per boundary j (t - 1)
    std::vector<std::vector<PartCut>> cuts;              // per part, ordered by (layer, upper qubit)
    std::vector<std::vector<std::pair<int, int>>> bits;  // per part: branch bit j -> (boundary, index in it)
  };
  MultiPart multipart_layout(uint32_t n_parts, const uint32_t *row_cuts) const;

  cudaEvent_t get_event();
  void resolve_events();
};

}  // namespace qsim
