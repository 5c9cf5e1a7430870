// scan_add.cu — vjp_scan instantiations for the ADD operator (f32, f64).
#include "scan_impl.cuh"
namespace vjph {
vjp_status scan_dispatch_add(int phase, const ScanCall &c, size_t *out) { return scan_dispatch<vjpk::OpAdd>(phase, c, out); }
}  // namespace vjph
