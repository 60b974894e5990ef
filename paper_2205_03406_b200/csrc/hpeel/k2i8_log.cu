// K2 int8 tensor-core apply, log kernel instantiations (k2_i8.cuh).
#include "k2_i8.cuh"

#include <stdexcept>

namespace hpeel {
namespace k2i8 {
void launch_log(HP_K2I8_ARGS) {
  launch_kind<kOpLog>(op, tasks, rowtab, ntasks, pay_off, step_off, xstep, pb_off, pb_box, box_bbox, bdig, half_stride, r, out, s);
}
}  // namespace k2i8
}  // namespace hpeel
