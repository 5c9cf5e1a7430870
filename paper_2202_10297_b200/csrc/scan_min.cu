// scan_min.cu — vjp_scan instantiations for the MIN operator (f32, f64).
#include "scan_impl.cuh"
namespace vjph {
vjp_status scan_dispatch_min(int phase, const ScanCall &c, size_t *out) { return scan_dispatch<vjpk::OpMin>(phase, c, out); }
}  // namespace vjph
