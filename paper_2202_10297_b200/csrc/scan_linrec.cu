// scan_linrec.cu — vjp_scan instantiations for the LINREC operator (f32, f64).
#include "scan_impl.cuh"
namespace vjph {
vjp_status scan_dispatch_linrec(int phase, const ScanCall &c, size_t *out) { return scan_dispatch<vjpk::OpLinrec>(phase, c, out); }
}  // namespace vjph
