// C-ABI of include/qsim.h: argument checks, exception -> status translation.
#include <cstring>
#include <new>
#include <string>

#include <nccl.h>

#include "../../include/qsim.h"
#include "engine.h"

struct qsim_ctx {
  qsim::Engine *eng = nullptr;
  std::string err;
};

namespace {

template <typename F>
qsim_status guard(qsim_ctx *ctx, F &&f) {
  if (!ctx || !ctx->eng) return QSIM_EINVAL;
  ctx->err.clear();
  try {
    f(*ctx->eng);
    return QSIM_OK;
  } catch (const qsim::Error &e) {
    ctx->err = e.what();
    return e.code;
  } catch (const std::bad_alloc &) {
    ctx->err = "host allocation failed";
    return QSIM_ENOMEM;
  } catch (const std::exception &e) {
    ctx->err = e.what();
    return QSIM_EINVAL;
  } catch (...) {
    ctx->err = "unknown error";
    return QSIM_EINVAL;
  }
}

}  // namespace

extern "C" {

const char *qsim_version(void) { return "qsim-b200 0.1 (sm_100a)"; }

qsim_status qsim_create(qsim_ctx **out, qsim_precision prec, int device) {
  if (!out) return QSIM_EINVAL;
  *out = nullptr;
  qsim_ctx *c = new (std::nothrow) qsim_ctx();
  if (!c) return QSIM_ENOMEM;
  try {
    c->eng = new qsim::Engine(prec, device);
  } catch (const qsim::Error &e) {
    delete c;
    return e.code;
  } catch (...) {
    delete c;
    return QSIM_ENOMEM;
  }
  *out = c;
  return QSIM_OK;
}

void qsim_destroy(qsim_ctx *ctx) {
  if (!ctx) return;
  delete ctx->eng;
  delete ctx;
}

const char *qsim_last_error(const qsim_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

qsim_status qsim_set_option(qsim_ctx *ctx, int key, int64_t value) {
  return guard(ctx, [&](qsim::Engine &e) { e.set_option(key, value); });
}

qsim_status qsim_set_stream(qsim_ctx *ctx, void *s) {
  return guard(ctx, [&](qsim::Engine &e) { e.set_stream(s); });
}

qsim_status qsim_load_circuit(qsim_ctx *ctx, uint32_t rows, uint32_t cols, uint32_t depth,
                              const qsim_gate *gates, size_t n_gates, uint32_t cut_row,
                              const uint32_t *cut_layers, size_t n_cut_layers) {
  return guard(ctx, [&](qsim::Engine &e) {
    e.load_circuit(rows, cols, depth, gates, n_gates, cut_row, cut_layers, n_cut_layers);
  });
}

qsim_status qsim_partition(qsim_ctx *ctx, uint32_t *n_cuts, uint64_t *n_branches, qsim_cut *cuts) {
  return guard(ctx, [&](qsim::Engine &e) { e.partition(n_cuts, n_branches, cuts); });
}

qsim_status qsim_set_blocks(qsim_ctx *ctx, const uint64_t *up, size_t nu, const uint64_t *lo, size_t nl) {
  return guard(ctx, [&](qsim::Engine &e) { e.set_blocks(up, nu, lo, nl); });
}

qsim_status qsim_evolve_range(qsim_ctx *ctx, uint64_t b0, uint64_t b1) {
  return guard(ctx, [&](qsim::Engine &e) { e.evolve_range(b0, b1); });
}

qsim_status qsim_evolve_halves(qsim_ctx *ctx, const uint64_t *up, size_t nu, const uint64_t *lo, size_t nl) {
  return guard(ctx, [&](qsim::Engine &e) {
    e.set_blocks(up, nu, lo, nl);
    uint64_t b0 = 0, b1 = 0;
    e.rank_range(&b0, &b1);
    if (b1 > b0) e.evolve_range(b0, b1);
  });
}

qsim_status qsim_reset_block(qsim_ctx *ctx) {
  return guard(ctx, [&](qsim::Engine &e) { e.reset_block(); });
}

qsim_status qsim_amplitudes(qsim_ctx *ctx, const uint64_t *up, size_t nu, const uint64_t *lo, size_t nl,
                            void *amps) {
  return guard(ctx, [&](qsim::Engine &e) {
    e.check_blocks(up, nu, lo, nl);
    e.amplitudes(amps);
  });
}

qsim_status qsim_sample(qsim_ctx *ctx, uint64_t seed, size_t n, uint64_t *out, double *mass) {
  return guard(ctx, [&](qsim::Engine &e) { e.sample(seed, n, out, mass); });
}

qsim_status qsim_sample_probs(qsim_ctx *ctx, const double *p, const uint64_t *up, size_t nu, const uint64_t *lo,
                              size_t nl, uint32_t hl, uint64_t seed, size_t n, uint64_t *out, double *mass) {
  return guard(ctx, [&](qsim::Engine &e) { e.sample_probs(p, up, nu, lo, nl, hl, seed, n, out, mass); });
}

qsim_status qsim_porter_thomas(qsim_ctx *ctx, const double *p, size_t n, uint32_t n_qubits, double z_lo,
                               double z_hi, uint32_t n_bins, uint64_t *hist, double *expected,
                               qsim_pt_t *out) {
  return guard(ctx, [&](qsim::Engine &e) {
    e.porter_thomas(p, n, n_qubits, z_lo, z_hi, n_bins, hist, expected, out);
  });
}

qsim_status qsim_branch_sum(qsim_ctx *ctx, const void *U, const void *L, size_t nb, size_t nu, size_t nl,
                            void *A) {
  return guard(ctx, [&](qsim::Engine &e) { e.branch_sum(U, L, nb, nu, nl, A); });
}

qsim_status qsim_branch_state(qsim_ctx *ctx, int half, uint64_t b, void *out) {
  return guard(ctx, [&](qsim::Engine &e) { e.branch_state(half, b, out); });
}

qsim_status qsim_branch_values(qsim_ctx *ctx, int half, uint64_t b, const uint64_t *idx, size_t n, void *out) {
  return guard(ctx, [&](qsim::Engine &e) { e.branch_values(half, b, idx, n, out); });
}

qsim_status qsim_info(qsim_ctx *ctx, qsim_info_t *out) {
  return guard(ctx, [&](qsim::Engine &e) {
    if (!out) throw qsim::Error(QSIM_EINVAL, "null output");
    e.info(out);
  });
}

qsim_status qsim_nccl_unique_id(void *out128) {
  if (!out128) return QSIM_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return QSIM_ENCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return QSIM_OK;
}

qsim_status qsim_comm_init(qsim_ctx *ctx, int rank, int world, const void *id) {
  return guard(ctx, [&](qsim::Engine &e) { e.comm_init(rank, world, id); });
}

qsim_status qsim_rank_range(qsim_ctx *ctx, uint64_t *b0, uint64_t *b1) {
  return guard(ctx, [&](qsim::Engine &e) {
    if (!b0 || !b1) throw qsim::Error(QSIM_EINVAL, "null output");
    e.rank_range(b0, b1);
  });
}

qsim_status qsim_eq2_time(const double *n_i, size_t depth, double m, double t, double s, double *seconds) {
  if (!seconds || (depth && !n_i) || !(s > 0.0)) return QSIM_EINVAL;
  double sum = 0.0;
  for (size_t i = 0; i < depth; ++i) sum += n_i[i];
  *seconds = sum * m * t / s;
  return QSIM_OK;
}

qsim_status qsim_cost_model(qsim_ctx *ctx, uint64_t nu, uint64_t nl, double hbm_gbps, qsim_cost_t *out) {
  return guard(ctx, [&](qsim::Engine &e) { e.cost_model(nu, nl, hbm_gbps, out); });
}

qsim_status qsim_multipart_plan(qsim_ctx *ctx, uint32_t n_parts, const uint32_t *row_cuts, uint32_t *part_qubits,
                                uint32_t *boundary_cuts, double *log2_states) {
  return guard(ctx, [&](qsim::Engine &e) { e.multipart_plan(n_parts, row_cuts, part_qubits, boundary_cuts, log2_states); });
}

qsim_status qsim_multipart_amplitudes(qsim_ctx *ctx, uint32_t n_parts, const uint32_t *row_cuts,
                                      const uint64_t *blocks, const size_t *n_block, void *amps) {
  return guard(ctx, [&](qsim::Engine &e) { e.multipart_amplitudes(n_parts, row_cuts, blocks, n_block, amps); });
}

qsim_status qsim_stats(qsim_ctx *ctx, qsim_stats_t *out) {
  return guard(ctx, [&](qsim::Engine &e) {
    if (!out) throw qsim::Error(QSIM_EINVAL, "null output");
    e.stats(out);
  });
}

qsim_status qsim_stats_reset(qsim_ctx *ctx) {
  return guard(ctx, [&](qsim::Engine &e) { e.stats_reset(); });
}

qsim_status qsim_synchronize(qsim_ctx *ctx) {
  return guard(ctx, [&](qsim::Engine &e) { e.synchronize(); });
}

}  // extern "C"
