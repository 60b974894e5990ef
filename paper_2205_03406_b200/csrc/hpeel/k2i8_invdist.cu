// K2 int8 tensor-core apply, invdist kernel instantiations (k2_i8.cuh).
#include "k2_i8.cuh"

#include <stdexcept>

namespace hpeel {
namespace k2i8 {
void launch_invdist(HP_K2I8_ARGS) {
  launch_kind<kOpInvDist4Pi>(op, tasks, rowtab, ntasks, pay_off, step_off, xstep, pb_off, pb_box, box_bbox, bdig, half_stride, r, out, s);
}
}  // namespace k2i8
}  // namespace hpeel
