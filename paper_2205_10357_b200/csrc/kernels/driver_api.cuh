// driver_api.cuh -- CUDA driver entry points resolved through the runtime
// (cudaGetDriverEntryPoint), so libnncb.so does not link libcuda.so and the
// host library loads on machines without a driver (plan compilation, tests).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

namespace nncb::drv {

struct Table {
    PFN_cuGetErrorString_v6000 getErrorString = nullptr;
    PFN_cuModuleLoadData_v2000 moduleLoadData = nullptr;
    PFN_cuModuleUnload_v2000 moduleUnload = nullptr;
    PFN_cuModuleGetFunction_v2000 moduleGetFunction = nullptr;
    PFN_cuLaunchKernel_v4000 launchKernel = nullptr;
    PFN_cuTensorMapEncodeTiled_v12000 tensorMapEncodeTiled = nullptr;
    PFN_cuFuncSetAttribute_v9000 funcSetAttribute = nullptr;
    bool ok = false;
};

inline const Table& table() {
    static Table t = [] {
        Table r;
        cudaDriverEntryPointQueryResult q;
        auto get = [&](const char* name, void** fn) {
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess;
        };
        r.ok = get("cuGetErrorString", reinterpret_cast<void**>(&r.getErrorString)) &&
               get("cuModuleLoadData", reinterpret_cast<void**>(&r.moduleLoadData)) &&
               get("cuModuleUnload", reinterpret_cast<void**>(&r.moduleUnload)) &&
               get("cuModuleGetFunction", reinterpret_cast<void**>(&r.moduleGetFunction)) &&
               get("cuLaunchKernel", reinterpret_cast<void**>(&r.launchKernel)) &&
               get("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&r.tensorMapEncodeTiled)) &&
               get("cuFuncSetAttribute", reinterpret_cast<void**>(&r.funcSetAttribute));
        return r;
    }();
    return t;
}

inline const char* error_string(CUresult r) {
    const char* s = nullptr;
    if (table().getErrorString) table().getErrorString(r, &s);
    return s ? s : "unknown driver error";
}

}  // namespace nncb::drv
