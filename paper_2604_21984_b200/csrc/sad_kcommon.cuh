// sad_kcommon.cuh — helpers shared by the kernel translation units (sad_kernels.cu, sad_fwdbwd.cu):
// programmatic dependent launch, the FieldDims row range / cell index, finiteness tests.
#pragma once
#include <cstdlib>

#include "sad_device.cuh"
#include "sad_kernels.h"

namespace sadk {

// Checked build (-DSAD_CHECKED=1, __graft_entry__.build_checked -> libsad_b200_checked.so): index bounds
// of shared-memory tables, record pools and site ids are tested in the kernels and violations counted in
// a device counter (sad_debug_checks).  The stand-in for compute-sanitizer memcheck, which is unavailable
// on the GPU pool used here.  Compiles to nothing in the product build.
#ifndef SAD_CHECKED
#define SAD_CHECKED 0
#endif
#if SAD_CHECKED
static __device__ unsigned long long g_check_fail = 0;  // (kernels and reader live in sad_kernels.cu)
#define SAD_CHECK(cond) do { if (!(cond)) atomicAdd(&::sadk::g_check_fail, 1ull); } while (0)
#else
#define SAD_CHECK(cond) do { } while (0)
#endif

// ---------------------------------------------------------------------- programmatic dependent launch
// The per-iteration kernels (warm pass, fwd+bwd, Adam, bookkeeping) are launched with programmatic
// stream serialisation, so the launch of each is prepared while its predecessor runs; every one waits
// in griddepcontrol.wait before ANY global access (every RAW and WAR dependency on the predecessor is
// respected).  Early triggers (launch_dependents at block start) let dependents occupy SMs during the
// predecessor's last wave; measured on the config-2 fit that is neutral to +9 ms (the fwd+bwd -> Adam
// edge), so by default no kernel triggers early and the gain is the launch latency (about 3 ms per
// fit).  Without the attribute (or a programmatic predecessor) both instructions are no-ops.
// SAD_NO_PDL=1 turns the attribute off (A/B).
#ifndef SAD_PDL_TRIGGER
#define SAD_PDL_TRIGGER 0  // bitmask of kernels that trigger early (1 prop, 2 bwd, 4 adam, 8 advance): measured no gain
#endif
template <int BIT>
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (SAD_PDL_TRIGGER & BIT) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
inline bool pdl_enabled() {
    static const bool on = getenv("SAD_NO_PDL") == nullptr;
    return on;
}
template <typename... KP, typename... A>
inline void launch_pdl(void (*kern)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, A... args) {
    if (!pdl_enabled()) {
        kern<<<grid, block, smem, stream>>>(args...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KP>(args)...);
}

// Rows a kernel covers under the optional FieldDims row range (host and device).
__host__ __device__ inline int rows_of(const FieldDims& f, int n) {
    const int hi = f.row1 < n ? f.row1 : n;
    return hi > f.row0 ? hi - f.row0 : 0;
}

// Candidate cell of pixel (px, py) (CandidateField::cell_x/cell_y, types.hpp:95-101); the fit's cell
// size is 1, so the two integer divisions are skipped on that (launch-uniform) path.
__device__ __forceinline__ size_t cell_index(const FieldDims& f, int px, int py) {
    if (f.cell == 1) return static_cast<size_t>(py) * f.gw + px;
    return static_cast<size_t>(py / f.cell) * f.gw + px / f.cell;
}

template <typename CT>
__device__ __forceinline__ bool c_finite(CT x);
template <>
__device__ __forceinline__ bool c_finite<float>(float x) {
    return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}
template <>
__device__ __forceinline__ bool c_finite<double>(double x) {
    return isfinite(x);
}

}  // namespace sadk
