// FP64 pipe probe (B200): DFMA dependent latency and throughput vs warps per SM sub-partition
// and independent chains per thread -- the numbers the Legendre kernels' schedule is built on.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_probe.cu -o tools/fp64_probe.bin
//   ./tools/fp64_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chains(double* out, int iters, double a, long long* cyc) {
    double v[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = threadIdx.x * 1e-3 + k;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < ILP; ++k) v[k] = __fma_rn(v[k], a, 0.25);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += v[k];
    if (s == 12345.678) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

// DMUL feeding a DFMA (the recurrence's shape): q2 = (A x) q1 - q0
template <int ILP>
__global__ void recur(double* out, int iters, double A, long long* cyc) {
    double q0[ILP], q1[ILP], x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) { q0[k] = 0.1 * k; q1[k] = 0.2; x[k] = 0.3 + threadIdx.x * 1e-4 + k * 1e-3; }
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < ILP; ++k) {
                const double q2 = __fma_rn(__dmul_rn(A, x[k]), q1[k], -q0[k]);
                q0[k] = q1[k];
                q1[k] = q2;
            }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += q1[k];
    if (s == 12345.678) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, int ilp, int instr_per_inner, int threads, int blocks, double* out, long long* cyc) {
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(out, iters, 0.999999, cyc);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters, 0.999999, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double ops = (double)iters * 8 * ilp * instr_per_inner;  // per thread
    const double tf = ops * threads * blocks * 2.0 / (ms * 1e-3) / 1e12;  // DMUL counted as 2 too
    printf("%-6s ilp=%d threads=%4d blocks=%4d  cyc/op/thread=%.2f  %.2f TF-equiv (%.3f ms)\n", name, ilp,
           threads, blocks, (double)c / ops, tf, ms);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // latency: one warp, one chain
    run("dfma", chains<1>, 1, 1, 32, 1, out, cyc);
    run("recur", recur<1>, 1, 2, 32, 1, out, cyc);
    for (int w : {1, 2, 3, 4, 6, 8}) {
        run("dfma", chains<1>, 1, 1, 128 * w, sms, out, cyc);
        run("dfma", chains<2>, 2, 1, 128 * w, sms, out, cyc);
        run("dfma", chains<4>, 4, 1, 128 * w, sms, out, cyc);
        run("dfma", chains<8>, 8, 1, 128 * w, sms, out, cyc);
        run("recur", recur<2>, 2, 2, 128 * w, sms, out, cyc);
        run("recur", recur<4>, 4, 2, 128 * w, sms, out, cyc);
        run("recur", recur<8>, 8, 2, 128 * w, sms, out, cyc);
    }
    return 0;
}
