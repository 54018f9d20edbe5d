// Probe: can the runtime launch our kernels into a green-context stream (an SM partition of
// the primary context), and do events order work across partition / full-device streams?
//   nvcc -gencode arch=compute_100a,code=sm_100a tools/green_probe.cu -o green_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

__global__ void smid_kernel(int* out, long long spin) {
    unsigned s;
    asm("mov.u32 %0, %%smid;" : "=r"(s));
    if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
    long long t0 = clock64();
    while (clock64() - t0 < spin) {}
}

#define DR(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* m; cuGetErrorString(r, &m); printf("%s failed: %s\n", #x, m); return 1; } } while (0)
#define RT(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

int main() {
    RT(cudaSetDevice(0));
    RT(cudaFree(0));  // primary context
    CUdevice dev;
    DR(cuDeviceGet(&dev, 0));
    CUdevResource all;
    DR(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("SMs: %u\n", all.sm.smCount);
    CUdevResource parts[2], rest;
    unsigned n = 1;
    DR(cuDevSmResourceSplitByCount(parts, &n, &all, &rest, 0, 16));
    printf("split: group %u SMs, rest %u SMs\n", parts[0].sm.smCount, rest.sm.smCount);
    CUdevResourceDesc d_small, d_rest;
    DR(cuDevResourceGenerateDesc(&d_small, &parts[0], 1));
    DR(cuDevResourceGenerateDesc(&d_rest, &rest, 1));
    CUgreenCtx g_small, g_rest;
    DR(cuGreenCtxCreate(&g_small, d_small, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    DR(cuGreenCtxCreate(&g_rest, d_rest, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s_small, s_rest;
    DR(cuGreenCtxStreamCreate(&s_small, g_small, CU_STREAM_NON_BLOCKING, 0));
    DR(cuGreenCtxStreamCreate(&s_rest, g_rest, CU_STREAM_NON_BLOCKING, 0));
    int* buf;
    RT(cudaMalloc(&buf, 4096 * sizeof(int)));
    cudaStream_t full;
    RT(cudaStreamCreateWithFlags(&full, cudaStreamNonBlocking));
    for (auto [name, st] : {std::pair<const char*, cudaStream_t>{"small", (cudaStream_t)s_small},
                            {"rest", (cudaStream_t)s_rest}, {"full", full}}) {
        RT(cudaMemset(buf, 0xff, 4096 * sizeof(int)));
        smid_kernel<<<1024, 128, 0, st>>>(buf, 200000);
        RT(cudaGetLastError());
        RT(cudaStreamSynchronize(st));
        std::vector<int> h(1024);
        RT(cudaMemcpy(h.data(), buf, 1024 * sizeof(int), cudaMemcpyDeviceToHost));
        std::set<int> sms(h.begin(), h.end());
        printf("%s stream: %zu distinct SMs (min %d max %d)\n", name, sms.size(), *sms.begin(), *sms.rbegin());
    }
    // ordering across partition streams with runtime events
    cudaEvent_t e;
    RT(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    smid_kernel<<<64, 128, 0, (cudaStream_t)s_small>>>(buf, 20000000);
    RT(cudaEventRecord(e, (cudaStream_t)s_small));
    RT(cudaStreamWaitEvent((cudaStream_t)s_rest, e, 0));
    RT(cudaMemsetAsync(buf + 2048, 7, 4, (cudaStream_t)s_rest));
    RT(cudaStreamWaitEvent(full, e, 0));
    smid_kernel<<<64, 128, 0, full>>>(buf + 1024, 1000);
    RT(cudaDeviceSynchronize());
    printf("cross-partition event ordering ok\n");
    return 0;
}
