// Microbenchmark: ceiling of the FP64 pipe for the Legendre FAST-step instruction mix
// (register-only, coefficients from shared memory), against a pure-DFMA loop.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/rec_probe.cu -o /tmp/rec_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_only(double* out, int iters) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
    const double b = 0.999999999, c = 1e-12;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    double r = 0;
    for (int i = 0; i < 8; ++i) r += a[i];
    if (r == 1234.5) out[0] = r;
}

// alm2map FAST step: q2 = fma(A*x, q1, -q0); ae += ar*q2 (complex), per stream accumulators
template <int R>
__global__ void a2m_mix(double* out, int iters) {
    __shared__ double sA[64], sR[64], sI[64];
    for (int i = threadIdx.x; i < 64; i += blockDim.x) {
        sA[i] = 1.0 + 1e-3 * i;
        sR[i] = 1e-3 * i;
        sI[i] = 2e-3 * i;
    }
    __syncthreads();
    double x[R], q0[R], q1[R], er[R], ei[R];
    for (int r = 0; r < R; ++r) {
        x[r] = 0.1 + 0.01 * r + threadIdx.x * 1e-6;
        q0[r] = 0.5;
        q1[r] = 0.25;
        er[r] = ei[r] = 0;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
            const double2 a = *reinterpret_cast<const double2*>(&sA[u]);
            const double2 ar = *reinterpret_cast<const double2*>(&sR[u]);
            const double2 ai = *reinterpret_cast<const double2*>(&sI[u]);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double q2 = __fma_rn(__dmul_rn(a.x, x[r]), q1[r], -q0[r]);
                er[r] = __fma_rn(ar.x, q2, er[r]);
                ei[r] = __fma_rn(ai.x, q2, ei[r]);
                q0[r] = q1[r];
                q1[r] = q2;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double q2 = __fma_rn(__dmul_rn(a.y, x[r]), q1[r], -q0[r]);
                er[r] = __fma_rn(ar.y, q2, er[r]);
                ei[r] = __fma_rn(ai.y, q2, ei[r]);
                q0[r] = q1[r];
                q1[r] = q2;
            }
        }
    }
    double s = 0;
    for (int r = 0; r < R; ++r) s += er[r] + ei[r] + q1[r];
    if (s == 1234.5) out[0] = s;
}

// map2alm FAST step: q2 as above; part += d*q2 summed over the lane's R streams, stored
template <int R>
__global__ void m2a_mix(double* out, int iters) {
    __shared__ double sA[64];
    __shared__ double2 row[4][32][8];
    for (int i = threadIdx.x; i < 64; i += blockDim.x) sA[i] = 1.0 + 1e-3 * i;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double x[R], q0[R], q1[R], dr[R], di[R];
    for (int r = 0; r < R; ++r) {
        x[r] = 0.1 + 0.01 * r + threadIdx.x * 1e-6;
        q0[r] = 0.5;
        q1[r] = 0.25;
        dr[r] = 0.3 * r;
        di[r] = 0.2 * r;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const double a = sA[u];
            double2 p = make_double2(0, 0);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double q2 = __fma_rn(__dmul_rn(a, x[r]), q1[r], -q0[r]);
                p.x = __fma_rn(dr[r], q2, p.x);
                p.y = __fma_rn(di[r], q2, p.y);
                q0[r] = q1[r];
                q1[r] = q2;
            }
            row[w][lane][u & 7] = p;
        }
    }
    double s = 0;
    for (int r = 0; r < R; ++r) s += q1[r];
    if (s == 1234.5) out[0] = s + row[w][lane][0].x;
}

template <typename K>
float run(K k, int blocks, int threads, int iters) {
    double* d;
    cudaMalloc(&d, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<blocks, threads>>>(d, iters);
    cudaEventRecord(a);
    k<<<blocks, threads>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(d);
    return ms;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int it = 4000;
    for (int per : {2, 4, 8, 16}) {
        const int blocks = sms * per, thr = 128;
        const double lanes = (double)blocks * thr;
        float t = run(dfma_only, blocks, thr, it);
        printf("warps/SM %2d  dfma_only: %.2f TF/s\n", per * 4, lanes * it * 16 * 8 * 2 / t / 1e9);
        t = run(a2m_mix<4>, blocks, thr, it);
        printf("warps/SM %2d  a2m R=4   : %.2f Tinstr/s (x2 = %.2f 'DFMA TF/s')\n", per * 4,
               lanes * it * 16 * 4 * 4 / t / 1e9, 2 * lanes * it * 16 * 4 * 4 / t / 1e9);
        t = run(m2a_mix<4>, blocks, thr, it);
        printf("warps/SM %2d  m2a R=4   : %.2f Tinstr/s (x2 = %.2f)\n", per * 4,
               lanes * it * 16 * 4 * 4 / t / 1e9, 2 * lanes * it * 16 * 4 * 4 / t / 1e9);
    }
    return 0;
}
