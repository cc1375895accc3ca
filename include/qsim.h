/*
 * qsim.h — C-ABI of the B200-native hot path of the partitioned simulator of
 * arXiv:1802.06952 ("64-qubit quantum circuit simulation", Chen et al. 2018).
 *
 * Method (§2.1, Supp. A Eqs. 1-8): every CZ that
 * crosses the horizontal cut of a rows x cols grid circuit is rewritten as
 * CZ = P0 (x) I + P1 (x) Z (Eq. 1), splitting the circuit into 2^c
 * branches ("copies") whose upper and lower half-circuits are independent.
 * Sampled amplitudes are reconstructed as
 *     a(x_u, x_l) = sum_b U_b[x_u] * L_b[x_l]
 * then p = |a|^2 and outcomes are drawn (north-star extension).
 *
 * Conventions (bit-exact contract):
 *  - qubit k = row*cols + col; the full bitstring has qubit 0 as its MSB.
 *  - upper half = rows [0, cut_row): h_u = cut_row*cols qubits, x_u = top h_u bits;
 *    lower half = the rest: h_l = n - h_u, x_l = bottom h_l bits; x = (x_u << h_l) | x_l.
 *  - layer 0 (H on every qubit) is implicit; gate layers are 1..depth.
 *  - cuts are ordered by (layer, upper qubit); branch b takes bit (b >> (c-1-g)) & 1
 *    for cut g (first cut = MSB); bit 0 -> P0 on the upper endpoint / I on the lower,
 *    bit 1 -> P1 / Z (Supp. Eq. 7).
 *  - gates: SX = X^1/2, SY = Y^1/2 (principal roots), T = diag(1, (1+i)/sqrt2),
 *    CZ = diag(1,1,1,-1).
 *
 * Threading / ownership: one host thread per ctx.  Every input array is a
 * caller-owned HOST array, read during the call only.  Every output array is a
 * caller-allocated HOST buffer.  The ctx owns all device memory, events and the
 * NCCL communicator; qsim_destroy frees them.  One process drives one GPU; for
 * several GPUs run one process per GPU and join them with qsim_comm_init.
 *
 * Errors: every call returns a qsim_status; qsim_last_error() gives a message
 * that stays valid until the next call on the same ctx.  No C++ exception
 * crosses the ABI.  Status codes 2/3/4 mirror the exit codes of SPEC S:477.
 */
#ifndef QSIM_H
#define QSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qsim_ctx qsim_ctx;

typedef enum {
  QSIM_OK = 0,
  QSIM_EINVAL = 2,   /* invalid argument / circuit / block                       */
  QSIM_ENOMEM = 3,   /* device (or host) memory does not fit the plan            */
  QSIM_ENUMERIC = 4, /* numeric sanity failure (e.g. zero block mass)            */
  QSIM_ECUDA = 5,    /* CUDA runtime error (includes "no CUDA device")           */
  QSIM_ENCCL = 6,    /* NCCL error                                               */
  QSIM_ESTATE = 7    /* call out of order (no circuit, no blocks, not evolved)   */
} qsim_status;

typedef enum { QSIM_C64 = 0, QSIM_C128 = 1 } qsim_precision;

typedef enum { QSIM_SX = 1, QSIM_SY = 2, QSIM_T = 3, QSIM_CZ = 4 } qsim_kind;

#define QSIM_NO_QUBIT 0xFFFFFFFFu

/* One gate: layer in 1..depth; q1 = QSIM_NO_QUBIT unless kind == QSIM_CZ. */
typedef struct { uint32_t layer, kind, q0, q1; } qsim_gate;

/* One cut CZ (E_int,t member, Supp. A P:305). */
typedef struct { uint32_t layer, q_upper, q_lower; } qsim_cut;

/* Counters of the ctx (cumulative since creation or the last qsim_stats_reset). */
typedef struct {
  uint64_t kernel_launches;  /* every kernel this library launched                       */
  uint64_t sweeps;           /* gate-sweep kernel launches (one state pass each)          */
  uint64_t sweep_states;     /* state passes done by those launches (>= sweeps if batched) */
  double sweep_bytes;        /* algorithmic bytes of the sweeps: (reads + writes) * amp size */
  double sweep_ms;           /* summed CUDA-event time of sweep launches (QSIM_OPT_TIME_SWEEPS) */
  uint64_t timed_sweeps;     /* sweep launches included in sweep_ms                      */
  double gemm_flops;         /* 8*M*N*K of the reconstruction GEMMs                      */
  double gemm_ms;            /* CUDA-event time of GEMM launches (QSIM_OPT_TIME_SWEEPS)  */
  uint64_t branches_evolved; /* branch pairs whose slices were gathered                  */
  uint64_t lazy_gathers;     /* leaves whose last sweep was evaluated at the sampled indices only */
  uint64_t layers_applied;   /* gate layers completed by the sweeps (> sweeps when layers are fused) */
  double sweep_bytes_moved;  /* bytes the sweeps actually read + wrote: sweep_bytes minus the reads of
                                known-zero tiles that were skipped               */
  uint64_t flip_siblings;    /* tree children reached as sibling flips of child 0 (no sweep of their own) */
  uint64_t undo_sweeps;      /* inverse sweeps that restored a state overwritten in place (included in sweeps) */
} qsim_stats_t;

typedef enum {
  QSIM_OPT_TIME_SWEEPS = 1, /* 1: bracket each sweep/GEMM launch with CUDA events (default 0) */
  QSIM_OPT_MODE = 2,        /* 0: auto, 1: flat in-shared-memory per-branch kernel (h <= 12),
                               2: prefix-shared branch tree of tile sweeps (h >= 13)          */
  QSIM_OPT_MEM_BUDGET = 3,  /* cap in bytes on device memory for half-state buffers (0 = free memory) */
  QSIM_OPT_SWEEP_KERNEL = 4, /* 0: TMA-pipelined sweep (default); 1: register-only one-layer sweep
                                (comparison); 2 / 3: the TMA sweep with 2 / 3 shared-memory stages      */
  QSIM_OPT_LAZY_LAST = 5     /* lazy tail of each leaf, evaluated only at the sampled indices during the
                                gather instead of full 2^h passes: 0 off, 1 the last sweep, 2 (default)
                                the last one to three by a cost model (cones of cones), 3 / 4 always
                                two / three when possible (tests)                                     */,
  QSIM_OPT_FUSE_LAYERS = 6,  /* reserved: multi-layer tiles were removed (compute-bound, never faster than
                                one pass per layer); only 0 is accepted             */
  QSIM_OPT_DISTRIBUTE = 7    /* 1: distributed half (§2.3.3): every half state
                                is sharded over the ranks of qsim_comm_init (1, 2 or 4, by its top
                                physical bits); every rank runs every branch on its shard; a gate on a
                                global qubit is preceded by a local/global qubit swap fused into the
                                previous sweep (its tiles are stored straight into the peer's HBM over
                                NVLink); sampled slices are summed over the ranks before the GEMM.
                                Needs >= tile bits + 2 qubits per shard; lazy tail off. 0: default */,
  QSIM_OPT_BFS = 8           /* 1 (default): for half / part states of at most 256 MiB, the depth-first
                                executor hands whole subtrees (the largest whose two deepest levels fit
                                in device memory) to a level-synchronous one: each sweep of a level is
                                ONE node-batched launch over every state of the level (the fork's P / Z
                                applied per node inside the sweep), leaves gathered in one launch (or
                                per leaf with the lazy tail when the subtree has <= 4096 leaves);
                                0: one launch per node and sweep                                      */,
  QSIM_OPT_MAX_CTAS = 9,     /* test only: cap on the persistent grid of the TMA sweeps (0 = one CTA per
                                SM, the default), so that small states run many tiles per CTA (mbarrier
                                phase wrap, stage rotation) in the parity tests                       */
  QSIM_OPT_DEFER = 10        /* 1 (default): deferred forks — each cut's P_b / Z^b is applied at the first
                                layer that targets its qubit (branches share their state until then,
                                DESIGN.md §5); 0: at the layer after the cut (A/B and tests)          */,
  QSIM_OPT_FLIP = 11,        /* 1 (default): sibling flips in qsim_evolve_range for half states above
                                256 MiB — the 2^k children of a Z^b fork are one state seen through a bit
                                flip and a diagonal, so only child 0 runs the fork's sweep; the free cuts
                                of a block take Z^b on both endpoints (CZ = sum_ab H_ab Z^a (x) Z^b, the
                                lower slices Walsh-Hadamard transformed); DESIGN.md §5. 0: off (A/B)  */
  QSIM_OPT_FLIP_NB = 12      /* test only: at most this many state buffers beyond the first for the
                                sibling-flip executor; further states run in place and are restored by
                                inverse sweeps (-1, the default: as many as fit)                      */
} qsim_option;

/* Create a context bound to CUDA device `device` (no device call is made until the
 * first evolve/sample call, so load/partition work on a machine without a GPU).
 * Errors: EINVAL (bad precision / device < 0), ENOMEM (host). */
qsim_status qsim_create(qsim_ctx **out, qsim_precision prec, int device);
void qsim_destroy(qsim_ctx *ctx);
const char *qsim_last_error(const qsim_ctx *ctx);
const char *qsim_version(void);

/* Set a qsim_option.  EINVAL on an unknown key or value. */
qsim_status qsim_set_option(qsim_ctx *ctx, int key, int64_t value);

/* Launch all work on this cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL = the ctx's own non-blocking stream (default). */
qsim_status qsim_set_stream(qsim_ctx *ctx, void *cuda_stream);

/* qsim_load_circuit — the circuit and its bipartition (P:285-311 Supp. A).
 *  rows, cols: grid (n = rows*cols <= 72; halves above 32 qubits need QSIM_OPT_DISTRIBUTE);  depth: number of gate layers;
 *  gates[n_gates]: host array, any order; each qubit at most once per layer;
 *    CZ only between grid neighbours; single-qubit gates: SX, SY, T.
 *  cut_row: upper half = rows [0, cut_row); 0 = rows/2.  Both halves must have
 *    1 <= h <= 36 qubits; a half of more than 32 qubits is evolved only as a distributed half
 *    (QSIM_OPT_DISTRIBUTE over >= 2^(h-32) ranks: at most 32 qubits per shard), else the
 *    evolve calls return EINVAL.
 *  cut_layers[n_cut_layers]: optional cross-check of the layers holding cut CZs
 *    (e.g. {7, 8, 15, 16}); NULL = derive.  A mismatch is EINVAL.
 * Replaces any previous circuit (and drops blocks / accumulated amplitudes). */
qsim_status qsim_load_circuit(qsim_ctx *ctx, uint32_t rows, uint32_t cols, uint32_t depth,
                              const qsim_gate *gates, size_t n_gates, uint32_t cut_row,
                              const uint32_t *cut_layers, size_t n_cut_layers);

/* qsim_partition — branch enumeration (§2.1 P:38 "2^c copies").
 *  *n_cuts = c, *n_branches = 2^c; cuts (nullable, capacity >= c) receives the cut
 *  list in branch-bit order.  ESTATE without a circuit; EINVAL if c > 40. */
qsim_status qsim_partition(qsim_ctx *ctx, uint32_t *n_cuts, uint64_t *n_branches, qsim_cut *cuts);

/* qsim_set_blocks — the sampled index blocks S_u (upper, values < 2^h_u) and S_l
 * (lower, values < 2^h_l), host uint64 arrays, unique (any order; output follows it).
 * Zeroes the amplitude accumulator.  EINVAL on out-of-range / duplicate / empty. */
qsim_status qsim_set_blocks(qsim_ctx *ctx, const uint64_t *upper_block, size_t n_upper,
                            const uint64_t *lower_block, size_t n_lower);

/* qsim_evolve_range — evolve branches [branch_begin, branch_end) (both halves, prefix-
 * shared), gather their slices U[b, :] = U_b[S_u], L[b, :] = L_b[S_l] and accumulate
 * A += U^T L into the device block ("results are finally added to the resultant
 * vector").  ESTATE without blocks; EINVAL on a bad range; ENOMEM. */
qsim_status qsim_evolve_range(qsim_ctx *ctx, uint64_t branch_begin, uint64_t branch_end);

/* qsim_evolve_halves — qsim_set_blocks + qsim_evolve_range over this rank's share of
 * [0, 2^c) (all branches when not joined to a communicator; SURVEY §8(e) sharding). */
qsim_status qsim_evolve_halves(qsim_ctx *ctx, const uint64_t *upper_block, size_t n_upper,
                               const uint64_t *lower_block, size_t n_lower);

/* qsim_reset_block — zero the device amplitude accumulator (blocks kept). */
qsim_status qsim_reset_block(qsim_ctx *ctx);

/* qsim_amplitudes — the reconstructed block a(S_u[i], S_l[j]).
 *  The blocks passed must equal the ones set (ESTATE otherwise; NULL = the set ones).
 *  amps: host, n_upper*n_lower complex (float2 for QSIM_C64, double2 for QSIM_C128),
 *  row-major [i][j].  With a communicator, partial blocks are summed over ranks (NCCL)
 *  and only rank 0 writes amps (others may pass NULL).  amps == NULL: reduce only. */
qsim_status qsim_amplitudes(qsim_ctx *ctx, const uint64_t *upper_block, size_t n_upper,
                            const uint64_t *lower_block, size_t n_lower, void *amps);

/* qsim_sample — p = |a|^2 of the (reduced) block, then n_draws outcomes drawn with
 * Philox4x32-10 (key = seed) and the two-level inverse CDF of SURVEY §8(c):
 *  bitstrings: host uint64[n_draws], x = (S_u[i] << h_l) | S_l[j]; NULL = keep on device.
 *  block_mass: host double (nullable) = W = sum of p over the block.
 *  ENUMERIC if W == 0; EINVAL for circuits above 64 qubits (x does not fit; use qsim_amplitudes).
 *  With a communicator the row shards are sampled on their ranks and rank 0 writes the outputs. */
qsim_status qsim_sample(qsim_ctx *ctx, uint64_t seed, size_t n_draws, uint64_t *bitstrings,
                        double *block_mass);

/* qsim_sample_probs — the same sampler on caller-given probabilities (host double
 * p[n_upper*n_lower], row-major), for sampler parity tests.  h_lower = shift of the
 * upper index.  Outputs as qsim_sample.  No circuit needed. */
qsim_status qsim_sample_probs(qsim_ctx *ctx, const double *p, const uint64_t *upper_block,
                              size_t n_upper, const uint64_t *lower_block, size_t n_lower,
                              uint32_t h_lower, uint64_t seed, size_t n_draws,
                              uint64_t *bitstrings, double *block_mass);

/* ---------------------------------------------------------------- Porter-Thomas analyzer (f1) */

/* Statistics of x = N p, N = 2^n_qubits, over a probability block (Fig. 5).
 * Porter-Thomas: x ~ Exp(1), so mean ~ 1 and var ~ 1; z = ln x follows Eq. 7 (alpha = 1) with
 * CDF F(z) = 1 - exp(-e^z) = 1 - exp(-x).  The Kolmogorov-Smirnov distance
 * D = sup_t |F_emp(t) - t| of u = F(z) over the entries with p > 0 is bracketed from a
 * 2^20-bin histogram of u: ks_lo <= D <= ks_hi, ks_hi - ks_lo <= 2^-20 + (largest bin)/n_pos. */
typedef struct {
  double count;     /* entries analysed (zeros included)                             */
  double zeros;     /* entries with p == 0 (excluded from z and the KS distance)     */
  double mean_Np;   /* (1/count) sum N p                                             */
  double var_Np;    /* (1/count) sum (N p)^2 - mean_Np^2 (population variance)        */
  double ks_lo, ks_hi;
  double below, above; /* p > 0 entries with z < z_lo or z >= z_hi (not in hist)     */
  uint32_t n_qubits;
  uint32_t n_bins;
} qsim_pt_t;

/* qsim_porter_thomas — the analyzer on the (reduced) block of the last qsim_evolve_range calls
 * (p = |a|^2 as qsim_sample computes it) when p == NULL, else on caller-given host
 * probabilities p[n] (no circuit needed).
 *  n_qubits: N = 2^n_qubits; 0 = the loaded circuit's qubit count (EINVAL without one).
 *  z histogram: n_bins (1..8192) equal bins over [z_lo, z_hi); bin = floor((z - z_lo) n_bins /
 *  (z_hi - z_lo)) in fp64.  hist: host uint64[n_bins] counts (nullable); expected: host
 *  double[n_bins] (nullable) = (count - zeros) (F(e_{k+1}) - F(e_k)), the Eq. 7 prediction
 *  for the same bins (Fig. 5's theory curve).  ESTATE with p == NULL and no evolved block;
 *  EINVAL on n > 2^32 - 1, bad bins or p < 0.  With a communicator the block is reduced
 *  first (every rank calls) and only rank 0 writes outputs. */
qsim_status qsim_porter_thomas(qsim_ctx *ctx, const double *p, size_t n, uint32_t n_qubits, double z_lo,
                               double z_hi, uint32_t n_bins, uint64_t *hist, double *expected,
                               qsim_pt_t *out);

/* qsim_branch_sum — the reconstruction contraction alone (a6): A[i,j] = sum_b U[b,i] L[b,j]
 * for host slices U[n_branches, n_upper], L[n_branches, n_lower] (complex of the ctx
 * precision); A: host complex double [n_upper, n_lower].  No circuit needed. */
qsim_status qsim_branch_sum(qsim_ctx *ctx, const void *U, const void *L, size_t n_branches,
                            size_t n_upper, size_t n_lower, void *A);

/* qsim_branch_state — one half-state of one branch after the last layer (the leaf of
 * the branch tree, before gathering), evolved by the same kernels as qsim_evolve_range.
 *  half: 0 = upper, 1 = lower; out: host, 2^h complex of the ctx precision.
 *  For spot checks at full size.  ESTATE without circuit. */
qsim_status qsim_branch_state(qsim_ctx *ctx, int half, uint64_t branch, void *out);

/* qsim_branch_values — U_b[idx[j]] (half 0) or L_b[idx[j]] (half 1) for one branch b, computed by
 * the production path of qsim_evolve_range (deferred forks, lazy tail, gathers) with idx as the
 * sampled block: the a3-a5 half of one row of the reconstruction.
 *  idx: host, n canonical half indices (< 2^h, any order, repeats allowed); out: host, n complex
 *  of the ctx precision.  For full-size spot checks (h = 24-32) where the complete leaf of
 *  qsim_branch_state does not fit.  EINVAL on a bad half / branch / index, ESTATE without circuit. */
qsim_status qsim_branch_values(qsim_ctx *ctx, int half, uint64_t branch, const uint64_t *idx, size_t n, void *out);

/* qsim_info — what the context holds, so that callers can size and check their buffers. */
typedef struct {
  uint32_t precision;     /* qsim_precision: amplitudes are complex64 (0) or complex128 (1)     */
  uint32_t have_circuit;  /* 1 after a successful qsim_load_circuit                             */
  uint32_t h_upper, h_lower, n_cuts;
  uint64_t n_upper, n_lower; /* sizes of the current blocks (0: none set)                        */
  int32_t device;
} qsim_info_t;
qsim_status qsim_info(qsim_ctx *ctx, qsim_info_t *out);

/* Multi-GPU: SURVEY §8(b)'s "multi-process variant" (qsim_create_rank there), one process per GPU
 * as torchrun launches them, instead of one process driving every GPU through ncclCommInitAll:
 * each process creates its context on its own device (qsim_create), then qsim_nccl_unique_id writes
 * 128 bytes (ncclUniqueId) on rank 0; every rank passes the same bytes to qsim_comm_init, which
 * records rank / world (EINVAL if out of range) — the NCCL communicator is created at the first
 * collective (qsim_amplitudes / qsim_sample, called by every rank), ENCCL on failure.
 * qsim_amplitudes: the ranks' partial blocks are summed to rank 0 (ncclReduce).  qsim_sample: the
 * partial blocks are reduce-scattered by rows, each rank computes |a|^2 and the row prefixes of its
 * rows, the row masses are all-gathered, every rank draws the same Philox stream and resolves the
 * draws that fall in its rows, and the draws are summed to rank 0. */
qsim_status qsim_nccl_unique_id(void *out128);
qsim_status qsim_comm_init(qsim_ctx *ctx, int rank, int world, const void *unique_id128);
/* This rank's share [*begin, *end) of the 2^c branches: contiguous, and aligned to the prefix groups
 * of the first cut period (the cuts of the first two cut layers) whenever world <= their number
 * (every rank then shares its tree down to its groups); else B r / world. */
qsim_status qsim_rank_range(qsim_ctx *ctx, uint64_t *begin, uint64_t *end);

/* ---------------------------------------------------------------- planner / cost model (f2) */

/* Eq. 2: Time = sum_{i=1..depth} n_i * m * t / s, with n_i the effective
 * gates of layer i of each half circuit, m the number of half circuits, t the time per gate
 * and s the number of nodes.  n_i: host array of `depth` values.  EINVAL if s <= 0. */
qsim_status qsim_eq2_time(const double *n_i, size_t depth, double m, double t, double s, double *seconds);

/* The partition of the loaded circuit and this library's execution plan for it. */
typedef struct {
  uint32_t n_qubits;        /* N_r: real qubit count                                    */
  uint32_t h_upper, h_lower;
  uint32_t n_cuts;          /* c                                                                */
  double n_branches;        /* 2^c copies                                                       */
  double half_circuits;     /* m = 2^(c+1) (Table 2 "equivalent 28-qubit circuits")            */
  uint32_t N_e;             /* equivalent qubits = max(h_u, h_l) + c + 1 (Table 2)       */
  uint32_t N_m;             /* largest state the device stores: floor(log2(mem / amp bytes))   */
  int32_t regime;           /* 0: N_e <= N_m full vectors; 1: N_m < N_e < N_r lossy (sampled);
                               2: N_e >= N_r no compression                             */
  double flat_layer_evolutions; /* paper §2.3.1: every copy from scratch, both halves           */
  double tree_sweeps;       /* this plan: prefix-shared branch tree, both halves, whole job     */
  double lazy_gathers;      /* leaves whose tail is evaluated at the sampled indices            */
  double sweep_bytes;       /* algorithmic HBM bytes of tree_sweeps                             */
  double predicted_s;       /* sweep_bytes / hbm bandwidth (sweeps dominate the run time)       */
} qsim_cost_t;

/* Cost model of the loaded circuit for sampled blocks of n_upper x n_lower indices on a device
 * with `hbm_gbps` GB/s of sweep bandwidth.  ESTATE without a circuit; EINVAL if hbm_gbps <= 0. */
qsim_status qsim_cost_model(qsim_ctx *ctx, uint64_t n_upper, uint64_t n_lower, double hbm_gbps,
                            qsim_cost_t *out);

/* ---------------------------------------------------------------- multi-part partitions (f4) */

/* t-way partitions of the loaded circuit ("dividing the circuit into three or
 * four parts is more effective if the circuit depth is small"; Fig. 3).  Part k is
 * the band of rows [r_k, r_{k+1}) with r_0 = 0, r_t = rows and r_1 < ... < r_{t-1} given in
 * `row_cuts` (t - 1 host values; cut_row of qsim_load_circuit is ignored here); its qubits are
 * [r_k*cols, r_{k+1}*cols), its local index has qubit r_k*cols as the MSB, and the full index
 * is the concatenation x_0 x_1 ... x_{t-1} (part 0 in the top bits).  Every CZ crossing a
 * boundary is split by Eq. 1: P_b on its upper endpoint, I / Z on its lower endpoint;
 * boundary j's cuts are ordered by (layer, upper qubit), first cut = MSB of beta_j.
 *
 * qsim_multipart_plan (host only, no device needed): part_qubits[k] (t values, nullable),
 * boundary_cuts[j] = c_j (t - 1 values, nullable) and *log2_states = log2 of
 * sum_k 2^(n_k + c_{k-1} + c_k), the amplitudes of all part leaves this library evolves
 * (nullable).  ESTATE without a circuit; EINVAL if t is not in 2..8, the row cuts are not
 * strictly increasing inside (0, rows) or a part has more than 32 qubits. */
qsim_status qsim_multipart_plan(qsim_ctx *ctx, uint32_t n_parts, const uint32_t *row_cuts,
                                uint32_t *part_qubits, uint32_t *boundary_cuts, double *log2_states);

/* Amplitudes of the index blocks S_0 x ... x S_{t-1}:
 *   amps[i_0, ..., i_{t-1}] = sum_b prod_k psi^k_b[S_k[i_k]]   (row-major, i_{t-1} fastest)
 * blocks: the t blocks concatenated (host, part-local indices < 2^{n_k}, unique, any order);
 * n_block[k]: size of block k.  amps: host, prod_k n_block[k] complex values of the ctx
 * precision (float2 / double2).  Every part is evolved as a branch tree over the cuts of its
 * two boundaries (2^(c_{k-1} + c_k) leaves) and the blocks are contracted as a chain of fp64
 * GEMMs on the device.  The two-half state of qsim_evolve_range is not touched.
 * EINVAL as qsim_multipart_plan, for a bad block, a part with more than 30 cut bits, an
 * output above 64 GiB, or with distributed halves enabled; ENOMEM if the part states, slices
 * or contraction operands do not fit; ECUDA without a device. */
qsim_status qsim_multipart_amplitudes(qsim_ctx *ctx, uint32_t n_parts, const uint32_t *row_cuts,
                                      const uint64_t *blocks, const size_t *n_block, void *amps);

/* Counters (see qsim_stats_t).  Synchronises the ctx stream when sweeps are timed. */
qsim_status qsim_stats(qsim_ctx *ctx, qsim_stats_t *out);
qsim_status qsim_stats_reset(qsim_ctx *ctx);
/* Block until all work queued by this ctx has finished. */
qsim_status qsim_synchronize(qsim_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* QSIM_H */
