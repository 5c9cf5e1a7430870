// scan_max.cu — vjp_scan instantiations for the MAX operator (f32, f64).
#include "scan_impl.cuh"
namespace vjph {
vjp_status scan_dispatch_max(int phase, const ScanCall &c, size_t *out) { return scan_dispatch<vjpk::OpMax>(phase, c, out); }
}  // namespace vjph
