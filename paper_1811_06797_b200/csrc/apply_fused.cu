// apply_fused.cu — fused sm_100a apply kernel (placeholder until the fused kernel lands).
#include "internal.h"

namespace igalr {

bool fused_supported(const iga_lr_op*, const Plan&) { return false; }

iga_status apply_fused(const iga_lr_op*, const Plan&, const OutMap&, int, cudaStream_t) {
    return set_error(IGA_EUNSUPPORTED, "fused kernel not available");
}

}  // namespace igalr
