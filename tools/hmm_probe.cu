// Pageable host memory from the GPU (B200 box): does the device support HMM / pageable memory
// access, and at what rate can a kernel stream a malloc'd buffer (read) and write one back,
// against cudaMemcpy from the same pageable buffer and from pinned memory?
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/hmm_probe.cu -o tools/hmm_probe.bin
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__global__ void rd(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    int v1 = 0, v2 = 0, v3 = 0, v4 = 0;
    cudaDeviceGetAttribute(&v1, cudaDevAttrPageableMemoryAccess, 0);
    cudaDeviceGetAttribute(&v2, cudaDevAttrPageableMemoryAccessUsesHostPageTables, 0);
    cudaDeviceGetAttribute(&v3, cudaDevAttrConcurrentManagedAccess, 0);
    cudaDeviceGetAttribute(&v4, cudaDevAttrHostRegisterSupported, 0);
    printf("pageableMemoryAccess %d usesHostPageTables %d concurrentManaged %d hostRegister %d\n", v1, v2, v3, v4);
    const size_t bytes = 403ull << 20, n = bytes / 16;
    double2* h = (double2*)malloc(bytes);
    memset(h, 1, bytes);
    double2* d;
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("memcpy H2D pageable: %.2f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
    }
    if (v1) {
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            rd<<<148 * 8, 256>>>(h, d, n);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("kernel read pageable: %.2f ms %.1f GB/s %s\n", ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            rd<<<148 * 8, 256>>>(d, h, n);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("kernel write pageable: %.2f ms %.1f GB/s %s\n", ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
        // fresh (never touched by the GPU) buffer: first-touch cost
        double2* h2 = (double2*)malloc(bytes);
        memset(h2, 2, bytes);
        cudaEventRecord(a);
        rd<<<148 * 8, 256>>>(h2, d, n);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("kernel read fresh pageable: %.2f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
        const auto t0 = std::chrono::steady_clock::now();
        volatile double s = 0;
        for (size_t i = 0; i < n; i += 512) s = s + h2[i].x;  // CPU touch after GPU access
        const double cpu_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        printf("cpu re-touch after gpu read: %.2f ms\n", cpu_ms);
    }
    double2* hp;
    cudaMallocHost(&hp, bytes);
    memset(hp, 1, bytes);
    cudaEventRecord(a);
    cudaMemcpyAsync(d, hp, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("memcpy H2D pinned: %.2f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
    const auto t0 = std::chrono::steady_clock::now();
    cudaHostRegister(h, bytes, cudaHostRegisterDefault);
    const double reg_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    printf("cudaHostRegister 403 MB: %.2f ms (%s)\n", reg_ms, cudaGetErrorString(cudaGetLastError()));
    const auto t1 = std::chrono::steady_clock::now();
    cudaHostUnregister(h);
    printf("cudaHostUnregister: %.2f ms\n", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
    return 0;
}
