// Recurrence-form probe (B200): does the Legendre step's DMUL -> DFMA shape cost FP64 issue
// rate, and which bit-identical instruction forms avoid it?  Runs the alm2map / map2alm
// steady-state step patterns of tools/leg_pattern_probe.cu with the recurrence written as
//   REC 0: t = A*x (DMUL), q2 = t*q1 - q0 (DFMA)            -- the kernels today
//   REC 1: t = fma(A, x, z) with a runtime z = -0.0 (DFMA)  -- bit-identical to A*x
//   REC 2: pure DFMA stand-in q2 = A*q1 - q0 (not the recurrence: the no-DMUL ceiling)
//   REC 3: REC 1 through inline PTX fma.rn.f64 (no compiler rewrite back to DMUL)
//   REC 4: t = A*x, q2 = t*q1 + q0 (no negated addend: the sign-folded recurrence)
//   REC 5: pure DFMA q2 = A*q1 + q0
// plus VAR 1: coefficients from registers (no LDS in the loop).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/rec_form_probe.cu -o tools/rec_form_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

template <int REC>
__device__ __forceinline__ double rec(double A, double x, double q1, double q0, double z) {
    if constexpr (REC == 0) return __fma_rn(__dmul_rn(A, x), q1, -q0);
    if constexpr (REC == 1) return __fma_rn(__fma_rn(A, x, z), q1, -q0);
    if constexpr (REC == 2) return __fma_rn(A, q1, -q0);
    if constexpr (REC == 3) {
        double t;
        asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(t) : "d"(A), "d"(x), "d"(z));
        return __fma_rn(t, q1, -q0);
    }
    if constexpr (REC == 4) return __fma_rn(__dmul_rn(A, x), q1, q0);
    if constexpr (REC == 5) return __fma_rn(A, q1, q0);
    return 0.0;
}

template <int R, int G, int MINB, int REC, int VAR>
__global__ void __launch_bounds__(128, MINB) a2m(double* out, int reps, double z) {
    __shared__ double sA[4][128], sR[4][128], sI[4][128];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = lane; j < 128; j += 32) {
        sA[w][j] = 1.0 + j * 1e-6;
        sR[w][j] = 0.5 - j * 1e-6;
        sI[w][j] = 0.25 + j * 1e-7;
    }
    __syncwarp();
    double x[R], q0[R], q1[R], aex[R], aey[R], aox[R], aoy[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        x[r] = 0.3 + 1e-3 * (lane + 32 * r);
        q0[r] = 0.1;
        q1[r] = 0.2;
        aex[r] = aey[r] = aox[r] = aoy[r] = 0.0;
    }
    for (int rep = 0; rep < reps; ++rep) {
        for (int j = 0; j < 128; j += G) {
            double A[G], ar[G], ai[G];
#pragma unroll
            for (int u = 0; u < G; u += 2) {
                if (VAR == 1) {
                    A[u] = 1.0 + (u + rep) * 1e-9; A[u + 1] = 1.0 - (u + rep) * 1e-9;
                    ar[u] = 0.5 + u * 1e-9; ar[u + 1] = 0.5 - u * 1e-9;
                    ai[u] = 0.25 - u * 1e-9; ai[u + 1] = 0.25 + u * 1e-9;
                } else {
                    const double2 a = *reinterpret_cast<const double2*>(&sA[w][j + u]);
                    const double2 b = *reinterpret_cast<const double2*>(&sR[w][j + u]);
                    const double2 c = *reinterpret_cast<const double2*>(&sI[w][j + u]);
                    A[u] = a.x; A[u + 1] = a.y; ar[u] = b.x; ar[u + 1] = b.y; ai[u] = c.x; ai[u + 1] = c.y;
                }
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double q2 = rec<REC>(A[u], x[r], q1[r], q0[r], z);
                    if (u & 1) {
                        aox[r] = __fma_rn(ar[u], q2, aox[r]);
                        aoy[r] = __fma_rn(ai[u], q2, aoy[r]);
                    } else {
                        aex[r] = __fma_rn(ar[u], q2, aex[r]);
                        aey[r] = __fma_rn(ai[u], q2, aey[r]);
                    }
                    q0[r] = q1[r];
                    q1[r] = q2;
                }
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += aex[r] + aey[r] + aox[r] + aoy[r] + q1[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// alm2map pattern with the next group's coefficients loaded while this group runs (register
// double buffer): no step waits on an LDS issued in its own group
template <int R, int G, int MINB, int REC>
__global__ void __launch_bounds__(128, MINB) a2m_pipe(double* out, int reps, double z) {
    __shared__ double sA[4][136], sR[4][136], sI[4][136];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = lane; j < 136; j += 32) {
        sA[w][j] = 1.0 + j * 1e-6;
        sR[w][j] = 0.5 - j * 1e-6;
        sI[w][j] = 0.25 + j * 1e-7;
    }
    __syncwarp();
    double x[R], q0[R], q1[R], aex[R], aey[R], aox[R], aoy[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        x[r] = 0.3 + 1e-3 * (lane + 32 * r);
        q0[r] = 0.1;
        q1[r] = 0.2;
        aex[r] = aey[r] = aox[r] = aoy[r] = 0.0;
    }
    double2 nA[G / 2], nR[G / 2], nI[G / 2];
    auto load = [&](int j) {
#pragma unroll
        for (int u = 0; u < G; u += 2) {
            nA[u / 2] = *reinterpret_cast<const double2*>(&sA[w][j + u]);
            nR[u / 2] = *reinterpret_cast<const double2*>(&sR[w][j + u]);
            nI[u / 2] = *reinterpret_cast<const double2*>(&sI[w][j + u]);
        }
    };
    load(0);
    for (int rep = 0; rep < reps; ++rep) {
        for (int j = 0; j < 128; j += G) {
            double A[G], ar[G], ai[G];
#pragma unroll
            for (int u = 0; u < G; u += 2) {
                A[u] = nA[u / 2].x; A[u + 1] = nA[u / 2].y;
                ar[u] = nR[u / 2].x; ar[u + 1] = nR[u / 2].y;
                ai[u] = nI[u / 2].x; ai[u + 1] = nI[u / 2].y;
            }
            load(j + G);
#pragma unroll
            for (int u = 0; u < G; ++u) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double q2 = rec<REC>(A[u], x[r], q1[r], q0[r], z);
                    if (u & 1) {
                        aox[r] = __fma_rn(ar[u], q2, aox[r]);
                        aoy[r] = __fma_rn(ai[u], q2, aoy[r]);
                    } else {
                        aex[r] = __fma_rn(ar[u], q2, aex[r]);
                        aey[r] = __fma_rn(ai[u], q2, aey[r]);
                    }
                    q0[r] = q1[r];
                    q1[r] = q2;
                }
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += aex[r] + aey[r] + aox[r] + aoy[r] + q1[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int S, int MINB, int REC>
__global__ void __launch_bounds__(128, MINB) m2a(double* out, int reps, double z) {
    extern __shared__ double sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* sA = sm + w * (128 + 32 * 34);
    double(*red)[34] = reinterpret_cast<double(*)[34]>(sA + 128);
    for (int j = lane; j < 128; j += 32) sA[j] = 1.0 + j * 1e-6;
    __syncwarp();
    double x[S], q0[S], q1[S], dsx[S], dsy[S], ddx[S], ddy[S];
#pragma unroll
    for (int r = 0; r < S; ++r) {
        x[r] = 0.3 + 1e-3 * (lane + 32 * r);
        q0[r] = 0.1;
        q1[r] = 0.2;
        dsx[r] = 0.1 * r; dsy[r] = 0.2 * r; ddx[r] = 0.3 - r; ddy[r] = 0.4 + r;
    }
    double tot = 0;
    for (int rep = 0; rep < reps; ++rep) {
        for (int g = 0; g < 128; g += 16) {
            double2* row = reinterpret_cast<double2*>(&red[lane][0]);
            double2 a = *reinterpret_cast<const double2*>(&sA[g]);
#pragma unroll
            for (int u = 0; u < 16; u += 2) {
                const double2 an = *reinterpret_cast<const double2*>(&sA[g + (u + 2 < 16 ? u + 2 : u)]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double A = h ? a.y : a.x;
                    double px = 0, py = 0;
#pragma unroll
                    for (int r = 0; r < S; ++r) {
                        const double q2 = rec<REC>(A, x[r], q1[r], q0[r], z);
                        px = __fma_rn(h ? ddx[r] : dsx[r], q2, px);
                        py = __fma_rn(h ? ddy[r] : dsy[r], q2, py);
                        q0[r] = q1[r];
                        q1[r] = q2;
                    }
                    row[u + h] = make_double2(px, py);
                }
                a = an;
            }
            __syncwarp();
            double s[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) s[k] = red[k][lane];
#pragma unroll
            for (int rr = 8; rr < 32; rr += 8)
#pragma unroll
                for (int k = 0; k < 8; ++k) s[k] += red[rr + k][lane];
            double v = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) v += s[k];
            tot += v;
            __syncwarp();
        }
    }
    double q = 0;
#pragma unroll
    for (int r = 0; r < S; ++r) q += q1[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = tot + q;
}

template <typename K>
void run(const char* name, K kern, size_t smem, double fp64_per_warp_rep, double* out, double z) {
    int sms = 0, clk = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 128, smem);
    const int blocks = sms * per, reps = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, 128, smem>>>(out, 2, z);
    cudaEventRecord(e0);
    kern<<<blocks, 128, smem>>>(out, reps, z);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = fp64_per_warp_rep * reps * blocks * 4;
    const double cap = (double)sms * 4 * 0.5 * clk * 1e3 * ms * 1e-3;
    printf("%-30s blocks/SM=%d %.3f ms  FP64 issue %.1f%%  %s\n", name, per, ms, 100.0 * warp_instr / cap,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 24);
    const double z = -0.0;
    const double a2 = 128.0 * 4 * 4, a8 = 128.0 * 8 * 4;
    run("a2m R4 G8 dmul", a2m<4, 8, 3, 0, 0>, 0, a2, out, z);
    run("a2m R4 G8 fma-z", a2m<4, 8, 3, 1, 0>, 0, a2, out, z);
    run("a2m R4 G8 fma-z ptx", a2m<4, 8, 3, 3, 0>, 0, a2, out, z);
    run("a2m R4 G8 pure-dfma", a2m<4, 8, 3, 2, 0>, 0, a2 * 3 / 4, out, z);
    run("a2m R4 G8 dmul +q0", a2m<4, 8, 3, 4, 0>, 0, a2, out, z);
    run("a2m R4 G8 pure-dfma +q0", a2m<4, 8, 3, 5, 0>, 0, a2 * 3 / 4, out, z);
    run("a2m R4 G8 fma-z ptx noLDS", a2m<4, 8, 3, 3, 1>, 0, a2, out, z);
    run("a2m R4 G8 pipelined", a2m_pipe<4, 8, 3, 0>, 0, a2, out, z);
    run("a2m R4 G4 pipelined", a2m_pipe<4, 4, 3, 0>, 0, a2, out, z);
    run("a2m R4 G8 pipelined minb4", a2m_pipe<4, 8, 4, 0>, 0, a2, out, z);
    run("a2m R8 G4 pipelined", a2m_pipe<8, 4, 2, 0>, 0, a8, out, z);
    run("a2m R8 G4 dmul", a2m<8, 4, 2, 0, 0>, 0, a8, out, z);
    run("a2m R8 G4 fma-z ptx", a2m<8, 4, 2, 3, 0>, 0, a8, out, z);
    run("a2m R8 G4 pure-dfma", a2m<8, 4, 2, 2, 0>, 0, a8 * 3 / 4, out, z);
    const size_t sm = 4 * (128 + 32 * 34) * sizeof(double);
    run("m2a S8 dmul", m2a<8, 3, 0>, sm, a8 + 8 * 31, out, z);
    run("m2a S8 fma-z ptx", m2a<8, 3, 3>, sm, a8 + 8 * 31, out, z);
    run("m2a S8 pure-dfma", m2a<8, 3, 2>, sm, a8 * 3 / 4 + 8 * 31, out, z);
    run("m2a S8 dmul +q0", m2a<8, 3, 4>, sm, a8 + 8 * 31, out, z);
    run("m2a S4 dmul", m2a<4, 4, 0>, sm, a2 + 8 * 31, out, z);
    run("m2a S4 fma-z ptx", m2a<4, 4, 3>, sm, a2 + 8 * 31, out, z);
    return 0;
}
