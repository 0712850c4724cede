// fbf_cuda_util.h -- small CUDA host helpers shared by the library's .cu files.
#pragma once

#include <cuda_runtime.h>

namespace fbf_b200 {

// Restores the calling thread's current device on scope exit: entry points
// switch to the device they were asked to use, and the caller's own device
// selection (e.g. torch's) must survive the call.
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

}  // namespace fbf_b200
