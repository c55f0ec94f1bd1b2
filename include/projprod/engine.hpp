#pragma once
// Engine controls with no counterpart in the reference API (its arithmetic is
// Eigen FP64 throughout, proj/CMakeLists.txt:15). Not needed for normal use.

namespace projprod::engine {

// Arithmetic of the engine's large products. false (default): the Gram
// SYRKs, the compress chain's forward transform, the slice-SVD filter and the
// star-Q facewise product run on the INT8 tensor cores as exact FP64
// emulation (Ozaki digit splitting; ~1e-14 relative to the operands' scale,
// see DESIGN.md section 3b), everything else on FP64 DMMA. true: every
// product on FP64 DMMA (IEEE double FMAs, as the reference). Process-wide.
void set_fp64_only(bool on);
bool fp64_only();

}  // namespace projprod::engine
