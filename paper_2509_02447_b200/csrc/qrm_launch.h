// Host-side launch helpers shared by the kernel launchers.
#pragma once

#include <cuda_runtime.h>

#include <mutex>

namespace qrm {

constexpr int kMaxDevices = 64;

// One-time setup per device: function attributes (dynamic shared memory size,
// non-portable cluster sizes) belong to each device's context, so a process
// that launches on several devices configures every one of them, once, and
// concurrent first launches from per-device host threads are safe.
struct PerDeviceOnce {
    std::once_flag flag[kMaxDevices];
    cudaError_t err[kMaxDevices] = {};
    template <typename F>
    cudaError_t run(F f) {
        int d = 0;
        const cudaError_t e = cudaGetDevice(&d);
        if (e != cudaSuccess) return e;
        if (d < 0 || d >= kMaxDevices) return cudaErrorInvalidDevice;
        std::call_once(flag[d], [&] { err[d] = f(); });
        return err[d];
    }
};

}  // namespace qrm
