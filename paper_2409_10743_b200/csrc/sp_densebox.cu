// FDBSCAN-DenseBox (dbscan.hpp:298-449) — placeholder until the dense-grid
// kernels land.
#include "sp_internal.hpp"
#include "sp_query.hpp"

namespace spb {

void densebox(Ctx &, const float *, int64_t, int, float, int32_t, int, int32_t *, uint8_t *, DbscanResult *) {
  throw InvalidArgument("densebox: not implemented yet");
}

}  // namespace spb
