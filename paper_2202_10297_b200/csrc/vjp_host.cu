// vjp_host.cu — host-side plumbing of libvjp_b200.so: status strings, the
// launch counter, TMA tensor-map construction through the driver entry point.
#include <atomic>
#include <cstring>
#include <mutex>

#include <cudaTypedefs.h>

#include "common.cuh"

namespace {
std::atomic<uint64_t> g_launches{0};

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}
}  // namespace

namespace vjph {
void count_launch(int k) { g_launches.fetch_add((uint64_t)k, std::memory_order_relaxed); }

bool make_row_tmap(CUtensorMap *map, const void *base, int64_t rows, bool f64, int box_rows) {
    std::memset(map, 0, sizeof(*map));
    if (rows <= 0) return true;  // never dereferenced by the kernels
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t inner = f64 ? 16 : 32;
    cuuint64_t dims[2] = {inner, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)vjpk::kRowBytes};
    cuuint32_t box[2] = {(cuuint32_t)inner, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
int sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
    return n;
}
}  // namespace vjph

extern "C" {

const char *vjp_status_string(vjp_status s) {
    switch (s) {
    case VJP_OK: return "VJP_OK";
    case VJP_EINVAL: return "VJP_EINVAL: invalid argument";
    case VJP_EUNSUPPORTED: return "VJP_EUNSUPPORTED: no rule for this operator/call";
    case VJP_EWORKSPACE: return "VJP_EWORKSPACE: workspace too small";
    case VJP_ECUDA: return "VJP_ECUDA: CUDA launch/runtime error";
    case VJP_EDUPINDEX: return "VJP_EDUPINDEX: duplicate scatter target";
    case VJP_EOOB: return "VJP_EOOB: index out of range";
    case VJP_EALIGN: return "VJP_EALIGN: array base not 16-byte aligned";
    }
    return "VJP_?: unknown status";
}

uint64_t vjp_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
