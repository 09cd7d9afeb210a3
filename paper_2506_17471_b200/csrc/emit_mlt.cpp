// emit_mlt.cpp — placeholder until the MLT family lands.
#include "femgpu_internal.hpp"
namespace femgpu {
EmitResult emit_mlt(const Signature&, const KernelPlan&) {
    fail(FEMGPU_E_INFEASIBLE, "mlt: not implemented yet");
}
}  // namespace femgpu
