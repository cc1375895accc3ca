// Internal helpers shared by engine.cu and tree.cu (not part of the C-ABI).
#pragma once

#include <nvtx3/nvToolsExt.h>

#include "engine.h"

namespace qsim {

// NVTX range per host phase (visible in nsys / ncu --nvtx; no cost without a tool attached)
struct Nvtx {
  explicit Nvtx(const char *name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx &) = delete;
  Nvtx &operator=(const Nvtx &) = delete;
};

// device form of a fused diagonal (inactive when the identity unless force_active)
DiagDev to_dev(const Diag &d, bool force_active = false);
// a sweep as a lazily evaluated layer (gather_layer_kernel) with the given pre diagonal
LazyLayer lazy_layer(const Sweep &sw, const Diag &pre);

}  // namespace qsim
