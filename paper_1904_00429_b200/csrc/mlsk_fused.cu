// mlsk_fused.cu -- placeholder until the fused engine lands.
#include "mlsk_internal.h"
namespace mlsk {
bool fused_supported(const Model&, int) { return false; }
void fused_run(const RunArgs&, const LevelSpec&, const std::vector<Segment>&, LevelState&) {
    throw Error(MLSK_ERUNTIME, "fused engine not built");
}
}  // namespace mlsk
