// K2 warp-specialized apply: instantiations for dense operators (k2_ws.cuh).
#include "k2_ws.cuh"

namespace hpeel {
namespace k2 {

void launch_dense(HP_K2_LAUNCH_ARGS) {
#define HP_ARGS op, trans, tasks, rowtab, ntasks, pay_off, pc, gc, gld, gcol0, ncols, xc, nnz, out, ocol0, flags, s
#define HP_CASE(NT) \
  case NT: return launch_nt_kind_dim<NT, kOpDense, 0>(HP_ARGS);
  switch ((ncols + 7) / 8) {
    HP_CASE(1) HP_CASE(2) HP_CASE(3) HP_CASE(4) HP_CASE(5) HP_CASE(6) HP_CASE(7) HP_CASE(8)
    HP_CASE(9) HP_CASE(10) HP_CASE(11) HP_CASE(12) HP_CASE(13) HP_CASE(14) HP_CASE(15)
    HP_CASE(16) HP_CASE(17) HP_CASE(18) HP_CASE(19) HP_CASE(20)
    default: throw std::invalid_argument("sample width 2r > 160 is not supported by the apply kernel");
  }
#undef HP_CASE
#undef HP_ARGS
}

}  // namespace k2
}  // namespace hpeel
