// Device parameter blocks and host launch wrappers of the sm_100a kernels.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace qsim {

// Device form of a fused diagonal (program.h Diag):
//   D(i) = scale * w^{(ph0 + popc(i&t1) + 2popc(i&t2) + 4(popc(i&zm)
//          + sum_k popc(i & i>>czd[k] & czm[k]))) & 7} * [(i & pm) == pv]
// czd / czm: the distinct CZ pair distances of the diagonal and their low-bit masks.
constexpr int kMaxCz = 31;
struct DiagDev {
  uint32_t t1, t2, zm, pm, pv;
  int32_t ph0;
  int32_t active;  // 0: identity, skip
  int32_t ncz;
  uint32_t czm[kMaxCz];
  uint8_t czd[kMaxCz];
  double scale;
};

// ---------------------------------------------------------------- tile sweep
// One launch = one memory pass over `njobs` half states of 2^h amplitudes.
// Tile = 2^T amplitudes: the L low bits (contiguous 512-byte rows) + 7 "hi" bits
// (the layer's high target bits, padded with the lowest free bits); the other bits
// are the outer bits enumerated by the tile index.  256 threads hold the tile in
// registers (16 register slots per thread x 16-byte vectors); targets on register
// bits are butterflies in registers, on lane bits warp shuffles, and a second pass
// through shared memory re-maps 4 other hi bits to registers when > 4 hi targets.
constexpr int kMaxJobs = 16;
constexpr int kHiBits = 7;

// Phase decomposition used by the TMA sweep (host precomputed).  For an element
// i = B | R_r, where B holds the thread / tile bits and R_r the register-slot bits,
//   ph(i) = ph_B(B) + P[r] + 4 * sum_j r_j * (popc(B & N[j]) & 1)        (mod 8)
//   ok(i) = ((B & Bpm) == Bpv) && !(P[r] & 8)
// ph_B is the full phase formula on B without ph0; P[r] carries ph0, every term of R_r
// alone and bit 3 = "projector fails on the register bits"; N[j] are the B-side
// partner bits of the CZ pairs of register bit j.
struct DiagSplit {
  uint8_t P[32];      // phase of R_r (+ph0) mod 8, times 8 (byte offset into a float2 table)
  uint32_t N[5];
  uint32_t Bpm, Bpv;
  uint32_t notok;     // bit r: the projector fails on the register bits of slot r
  int32_t has_proj;   // any projector at all (else the zeroing is skipped)
};

// Fork of a branch-tree level applied per node of a node-batched launch (multi-part BFS
// levels): node index = (parent << n) | child; cut j (child bit n-1-j) at local bit bit[j]
// is P_b (zero where the bit != b) when pmask bit j is set, else Z^b (negate where bit & b).
struct ForkDev {
  int32_t n;
  uint32_t pmask;
  uint8_t bit[32];
};

struct TileSweepParams {
  const void *src[kMaxJobs];
  void *dst[kMaxJobs];
  uint32_t job_pv[kMaxJobs];  // per-job projector value of the pre diagonal
  uint32_t job_zm[kMaxJobs];  // per-job Z mask of the pre diagonal
  int32_t njobs;
  int32_t log2_ntiles;  // tiles per job = 2^(h - T)
  int32_t nruns;
  uint8_t run_start[32], run_len[32];  // outer bit runs, ascending
  uint8_t hb[kHiBits];                 // hi tile bit positions, ascending
  uint8_t gsel[2][4];                  // pass p: hb indices held in registers
  uint8_t wsel[2][3];                  // pass p: hb indices mapped to the 3 warp bits
  // gate kinds: 0 none, 1 SX', 2 SY'; the TMA sweep also takes k + 2 f with a deferred fork on the
  // gate's own bit applied just before it (f = 1 Z^1, 2 P0, 3 P1; sweep_tma.cu reg_gates)
  uint8_t gkind[2][4];                 // gate kind per register bit
  uint8_t lowkind[6];                  // gate kind per low bit (lane / vector bits), pass 0
  DiagDev pre, post;
  DiagSplit pre_s, post_s;  // TMA sweep: pre uses the pass-0 registers, post the last pass's
  int32_t run_m;            // hb[0..run_m-1] == L..L+run_m-1: contiguous run of 2^(L+m) amps
  int32_t n_lane;           // TMA sweep: compact list of the lane-bit targets (pass 0)
  uint8_t lane_bit[5], lane_kind[5];
  // distributed half (f3): this rank's shard holds the amplitudes whose global bits (positions
  // h_local ..) equal `rank`; gbase = those bits, ORed into indices for the diagonals only.
  // nswap > 0: the sweep's output exchanges local bit swap_l[j] with global bit j' = swap_j[j]:
  // a tile whose outer bit swap_l[j] differs from the rank's bit j' goes to rank ^ (1 << j')
  // (peer[rank delta] = that rank's destination buffer) with bit swap_l[j] set to the rank's bit.
  uint32_t gbase;
  uint32_t rank;
  int32_t nswap;
  uint8_t swap_l[2], swap_j[2];
  void *peer[4];
  // node batching (TMA sweep only): 2^log2_nodes states of node_stride amplitudes, tile index
  // t = (node << log2_ntiles) | tile; node reads state node >> node_src_shift of src[0] (the
  // parent of a fork child) and writes state node of dst[0]; fork applied per node at pass 0
  int32_t log2_nodes;
  int32_t node_src_shift;
  uint64_t node_stride;
  ForkDev fork;
  // known-zero tiles (TMA sweep, NB = 0): a tile whose outer bits satisfy (outer & skip_pm) !=
  // skip_pv holds only zeros (a fork projector P_b on a qubit no gate of the level has touched
  // yet); it is not loaded, and zeros are stored
  uint32_t skip_pm, skip_pv;
  // node-batched variant: fork_apply = apply p.fork at pass 0 (the level's first launch); nb_skip =
  // the projected fork bits (outer bits of the tile, untouched so far in the level): a tile whose
  // bits there differ from the node's branch bits is zero (not loaded)
  int32_t fork_apply;
  uint32_t nb_skip;
  // the projector of this sweep's input (pre diagonal + the P forks folded into gate kinds): rows /
  // tiles it zeroes are not loaded; no_pskip = 1 loads them anyway (A/B)
  uint32_t ld_pm, ld_pv;
  int32_t no_pskip;
};

// pre_mode: 0 none, 1 apply pre diagonal to loaded values, 2 generate (no load)
// c128: amplitudes are double2, else float2.
cudaError_t launch_tile_sweep(const TileSweepParams &p, bool c128, int pre_mode, int npass,
                              int grid, cudaStream_t s);

// TMA-pipelined sweep (sweep_tma.cu, the default): one CTA per SM, `stages` (2 or 3) shared-memory
// tile stages filled by cp.async.bulk / cp.async under mbarriers, 1 producer warp + two ping-pong
// groups of 8 consumer warps (each group owns alternate tiles); one layer (TileSweepParams).
cudaError_t launch_tile_sweep_tma(const TileSweepParams &p, bool c128, int pre_mode, int npass, int grid,
                                  cudaStream_t s, int stages);
cudaError_t tile_sweep_tma_setup(bool c128);
constexpr int kTileBytes = 65536;
int tile_low_bits(bool c128);  // L: 6 (c64) or 5 (c128); tile T = L + 7
cudaError_t tile_sweep_setup(int *blocks_per_sm_1pass, int *blocks_per_sm_2pass, bool c128);

// ---------------------------------------------------------------- small states (h <= 12)
// Whole half state in shared memory; one CTA per branch; every level and sweep of the
// half program in one launch; the leaf is gathered straight into the slice row.
struct SmallSweepDev {
  DiagDev pre, post;
  int32_t ngates;
  int32_t gen;
  uint8_t bit[32];
  uint8_t kind[32];
};
struct SmallLevelDev {
  int32_t k;
  int32_t first_sweep;
  int32_t nsweeps;
  uint32_t pmask;  // bit j: cut j is P_b (upper endpoint), else Z^b
  uint8_t cut_bits[32];
};
struct SmallParams {
  const SmallLevelDev *levels;
  const SmallSweepDev *sweeps;
  int32_t nlevels;
  int32_t h;
  int32_t c;                 // cut bits of the branch index (the program's ncuts)
  uint64_t b0;               // first branch of this launch (blockIdx.x = b - b0)
  const uint64_t *S;         // sampled indices of this half
  int64_t nS;
  void *out;                 // slice [nb, nS] complex
};
cudaError_t launch_small(const SmallParams &p, bool c128, uint64_t nb, cudaStream_t s);
int small_max_h(bool c128);

// ---------------------------------------------------------------- gather / reconstruction
// out[j] = pend(S[j]) psi[(S[j] ^ xmask) & lmask] if (S[j] & ~lmask) == gsel (the shard owns it),
// else 0; xmask: the state is a sibling flip of the buffer (Engine::flip_node)
cudaError_t launch_gather(const void *psi, const uint64_t *S, int64_t n, void *out,
                          const DiagDev &pend, bool c128, cudaStream_t s, uint64_t lmask = ~0ull,
                          uint64_t gsel = 0, uint64_t xmask = 0);

// Leaves of a node-batched level: out[row(node) * n + j] = pend(S[j]) fork(node, S[j]) *
// psi[(node >> shift) * stride + S[j]], row(node) = rowmap ? rowmap[node] : node
cudaError_t launch_gather_nodes(const void *psi, uint64_t stride, int shift, int64_t nnodes, const uint64_t *S,
                                int64_t n, void *out, const ForkDev &fork, bool c128, cudaStream_t s,
                                const DiagDev *pend = nullptr, const uint32_t *rowmap = nullptr);
// Leaves seen through linear Pauli frames (Engine::run_tree_frames): each leaf is a sum of terms
// c_k w^{ph0_k + popc(x&t1_k) + 2 popc(x&t2_k) + 4 popc(x&zm_k)} psi[x ^ m_k]; for leaf i and x = S[j]
//   out[row_i * n + j] += pend(x) * sum over the leaf's terms k in [off[i], off[i+1])
struct FrameTerm {
  uint32_t t1, t2, zm, m;
  int32_t ph0, pad;
  double cr, ci;
};
constexpr int kMaxBatchLeaves = 256, kMaxBatchTerms = 512;
struct FrameBatch {
  int32_t nleaf;
  uint16_t off[kMaxBatchLeaves + 1];
  uint32_t row[kMaxBatchLeaves];
  FrameTerm term[kMaxBatchTerms];
};
// from_rows: psi is a [flip][n] table of pre-gathered rows (launch_flip_rows) and FrameTerm::m a row index
cudaError_t launch_frame_gather(const void *psi, const uint64_t *S, int64_t n, void *out, const FrameBatch &b,
                                const DiagDev &pend, bool c128, cudaStream_t s, bool from_rows = false);
// g[i * n + j] = psi[S[j] ^ flips[i]] for the nf distinct flips of a gather (one scattered pass per flip)
cudaError_t launch_flip_rows(const void *psi, const uint64_t *S, int64_t n, const uint64_t *flips, int64_t nf, void *g,
                             bool c128, cudaStream_t s);
// Output rows of node-batched leaves: out[N] = base | sum_t ((N >> t) & 1) << pos[t]
struct RowMapDev {
  int32_t nbits;
  uint32_t base;
  uint8_t pos[32];
};
cudaError_t launch_rowmap(uint32_t *out, int64_t n, const RowMapDev &rm, cudaStream_t s);
// out[r][j] = sum_{e in [off[r], off[r+1])} coef[e] * in[src[e]][j] for r < nrows (complex rows of n entries of
// the ctx precision, coef double2, fp64 sums): the frame basis' sparse combinations (Engine::evolve_range)
cudaError_t launch_combine_rows(const void *in, int64_t n, const uint32_t *off, const uint32_t *src, const void *coef,
                                int64_t nrows, void *out, bool c128, cudaStream_t s);
// rows [0, 2^m) of a slice (ncols entries each, ctx precision): Walsh-Hadamard transform over the m
// row-index bits with 1/2 per bit (m launches)
cudaError_t launch_wht_rows(void *A, bool c128, int m, int64_t ncols, cudaStream_t s);
// Lazy last layer: the leaf's final sweep evaluated only at the sampled indices,
//   out[j] = post(x) * sum_y  prod_t M'_t[x_t, y_t] * pre(y) * psi[y],   x = S[j],
// y ranging over the 2^k values of the sweep's target bits (others equal to x).
struct LazyLayer {
  int32_t k;
  uint8_t bit[24];
  uint32_t sxmask, symask, tmask;
  DiagDev pre, post;
  // distributed half: the shard holds the indices with (i & ~lmask) == gsel, at i & lmask (the
  // layer's targets are local, so every term of an owned index is in the shard); others give 0
  uint64_t lmask, gsel;
  // node batching (level-synchronous leaves): node_stride > 0 -> output j covers node j / nper of
  // states psi + node * node_stride at index S[j % nper]; its output row is rowmap[node] (when set)
  uint64_t node_stride;
  int64_t nper;
  const uint32_t *rowmap;
  // psi read at y ^ xmask (launch_gather_layer only): the state is a sibling flip of the buffer
  uint64_t xmask;
};
cudaError_t launch_gather_layer(const void *psi, const uint64_t *S, int64_t n, void *out,
                                const LazyLayer &ll, bool c128, cudaStream_t s);
// Two lazy layers: the cone of the last layer, cone[j * 2^k + m] = (S[j] & ~tmask) | deposit(m),
// is where layer d-1 is needed; launch_gather_layer(psi, cone) evaluates it there, and the
// compact variant applies layer d reading V[j * 2^k + m] instead of psi[y].
cudaError_t launch_cone_indices(const uint64_t *S, int64_t n, const LazyLayer &ll, uint64_t *cone,
                                cudaStream_t s);
cudaError_t launch_gather_layer_compact(const void *V, const uint64_t *S, int64_t n, void *out,
                                        const LazyLayer &ll, bool c128, cudaStream_t s);
// A[m, n] += sum_k U[k, m] * L[k, n]   (complex; U, L of the ctx precision, A double2)
cudaError_t launch_branch_gemm(const void *U, const void *L, int64_t K, int64_t M, int64_t N,
                               double *A, bool c128, cudaStream_t s);
// Multi-part contraction: for z in [0, batch),
//   A_z[m, n] += sum_k U_z[k, m] * L[k, n],  U_z = U + z*K*M, A_z = A + z*M*N  (all double2);
// N2 > 0: n = n1 * N2 + n2 and A_z is laid out [n1][m][n2] (the left chain's next operand)
cudaError_t launch_branch_gemm_batched(const double *U, const double *L, int64_t K, int64_t M, int64_t N,
                                       double *A, int64_t batch, cudaStream_t s, int64_t N2 = 0);
// dst[rowmap[r], :] = src[r, :] converted to double2 (src of the ctx precision)
cudaError_t launch_permute_rows(const void *src, bool c128, const uint32_t *rowmap, int64_t nrows, int64_t ncols,
                                double *dst, cudaStream_t s);
// p[i] = fma(re, re, im*im)
cudaError_t launch_abs2(const double *A, int64_t n, double *p, cudaStream_t s);
// C[i, :] = sequential inclusive prefix of p[i, :]; r[i] = C[i, N-1]
cudaError_t launch_row_scan(const double *p, int64_t M, int64_t N, double *C, double *r,
                            cudaStream_t s);
// the same with p = fma(re, re, im*im) of the complex block A computed in the scan (and stored to p)
cudaError_t launch_row_scan_abs2(const double *A, int64_t M, int64_t N, double *p, double *C, double *r,
                                 cudaStream_t s);
// R = sequential inclusive prefix of r; W = R[M-1] (written to *W)
cudaError_t launch_row_prefix(const double *r, int64_t M, double *R, double *W, cudaStream_t s);
// draws k in [0, n): Philox4x32-10 uniforms, inverse CDF, x = (Su[i] << hl) | Sl[j]; p / C hold
// rows [row0, row0 + nrows) (nrows < 0: all M), r / R all rows; a draw in another rank's rows gives 0
cudaError_t launch_draws(const double *p, const double *C, const double *r, const double *R,
                         const double *W, int64_t M, int64_t N, const uint64_t *Su,
                         const uint64_t *Sl, uint32_t hl, uint64_t seed, int64_t n,
                         uint64_t *out, cudaStream_t s, int64_t row0 = 0, int64_t nrows = -1);
cudaError_t launch_cast_c128_to_c64(const double *A, int64_t n, float *out, cudaStream_t s);

// Porter-Thomas analyzer (stats.cu).  Input: complex block A (double2, p = fma(re,re,im*im))
// when `complex_in`, else probabilities.  Scratch (device, PtScratch::bytes): z / u histograms,
// per-CTA moment partials; result: PtResult on the device.
constexpr int PT_U_BINS = 1 << 20;
constexpr int PT_MAX_Z_BINS = 8192;
constexpr int PT_CTAS = 148 * 4;
struct PtResult {
  unsigned long long zeros, below, above;
  double s1, s2;      // sum x, sum x^2 (fixed order over CTA partials)
  double ks_lo, ks_hi;
};
struct PtScratch {
  static size_t bytes(int n_bins) {
    return (size_t)PT_U_BINS * 4 + (size_t)PT_MAX_Z_BINS * 4 + (size_t)PT_CTAS * 2 * 8 + sizeof(PtResult) + 64;
  }
};
cudaError_t launch_porter_thomas(const void *in, bool complex_in, int64_t n, int n_qubits, double z_lo,
                                 double z_hi, int n_bins, void *scratch, cudaStream_t s);
// device pointers into the scratch block
unsigned *pt_zhist(void *scratch);
const PtResult *pt_result(void *scratch);

}  // namespace qsim
