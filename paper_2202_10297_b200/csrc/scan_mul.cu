// scan_mul.cu — vjp_scan instantiations for the MUL operator (f32, f64).
#include "scan_impl.cuh"
namespace vjph {
vjp_status scan_dispatch_mul(int phase, const ScanCall &c, size_t *out) { return scan_dispatch<vjpk::OpMul>(phase, c, out); }
}  // namespace vjph
