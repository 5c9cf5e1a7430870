// scan_mat2.cu — vjp_scan instantiations for the MAT2 operator (f32, f64).
#include "scan_impl.cuh"
namespace vjph {
vjp_status scan_dispatch_mat2(int phase, const ScanCall &c, size_t *out) { return scan_dispatch<vjpk::OpMat2>(phase, c, out); }
}  // namespace vjph
