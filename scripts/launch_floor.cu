// Launch-cost floor on this GPU: event-timed duration of EMPTY kernels with the
// decode kernel's launch shape (132 CTAs of 160 threads, clusters of 4,
// 101 KB dynamic shared memory, programmatic stream serialization) next to a
// plain launch. Each timed launch is pre-queued behind a spin kernel, so the
// span is device time, not host submission.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 scripts/launch_floor.cu -o /tmp/launch_floor
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void spin(long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < static_cast<unsigned long long>(ns));
}
__global__ void empty_kernel(int* sink) {
    extern __shared__ int sm[];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (sink) sink[blockIdx.x] = sm[(threadIdx.x + 1) % blockDim.x];
}

static float timed(bool cluster, size_t smem, bool pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(132);
    cfg.blockDim = dim3(160);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (cluster) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 4; attr[na].val.clusterDim.y = 1; attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> v;
    for (int i = 0; i < 25; ++i) {
        spin<<<1, 32>>>(50000);
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
        if (e != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(e)); return -1.f; }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        v.push_back(ms * 1000.f);
    }
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}

int main() {
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 101 * 1024 + 256);
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const size_t big = 101 * 1024 + 256;
    printf("{\"plain_us\": %.2f, \"smem101k_us\": %.2f, \"cluster4_us\": %.2f, \"cluster4_smem101k_us\": %.2f, "
           "\"cluster4_smem101k_pdl_us\": %.2f}\n",
           timed(false, 1024, false), timed(false, big, false), timed(true, 1024, false), timed(true, big, false),
           timed(true, big, true));
    return 0;
}
