// Steady-state probe of the Legendre FAST loops (B200): the alm2map / map2alm inner step
// patterns run on synthetic in-register data, no items, no tails, no activation windows --
// the ceiling of the instruction schedule itself, to compare against the kernels' measured
// FP64-pipe utilisation.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xptxas -v tools/leg_pattern_probe.cu -o tools/leg_pattern_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

#ifndef NSTEP
#define NSTEP 4096
#endif

__device__ __forceinline__ double rec_step(double A, double x, double q1, double q0) {
    return __fma_rn(__dmul_rn(A, x), q1, -q0);
}

// alm2map: per stream 1 DMUL + 3 DFMA per step; coefficients (A, ar, ai) staged in smem
// VAR 0: as the kernel; 1: recurrence only (no accumulation); 2: coefficients from registers
// (no LDS in the loop); 3: accumulation only (Q from a cheap DADD chain instead of the recurrence);
// 4: only A from shared memory (ar, ai from a per-rep register set: 1/3 of the LDS bytes);
// 5: as 0 plus 6 extra LDS.128 per group consumed by integer ops (doubles the LDS bytes)
template <int R, int G, int MINB, int VAR = 0>
__global__ void __launch_bounds__(128, MINB) a2m_pattern(double* out, int reps) {
    __shared__ double sA[4][128], sR[4][128], sI[4][128];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = lane; j < 128; j += 32) {
        sA[w][j] = 1.0 + j * 1e-6;
        sR[w][j] = 0.5 - j * 1e-6;
        sI[w][j] = 0.25 + j * 1e-7;
    }
    __syncwarp();
    __shared__ double sX[4][256];
    for (int j = lane; j < 256; j += 32) sX[w][j] = j;
    unsigned junk = 0;
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
            if (VAR == 2) {
#pragma unroll
                for (int u = 0; u < G; ++u) { A[u] = 1.0 + (u + rep) * 1e-9; ar[u] = 0.5 + u * 1e-9; ai[u] = 0.25 - u * 1e-9; }
            } else if (VAR == 4) {
#pragma unroll
                for (int u = 0; u < G; u += 2) {
                    const double2 a = *reinterpret_cast<const double2*>(&sA[w][j + u]);
                    A[u] = a.x; A[u + 1] = a.y;
                    ar[u] = 0.5 + (u + rep) * 1e-9; ar[u + 1] = 0.5 - (u + rep) * 1e-9;
                    ai[u] = 0.25 + u * 1e-9; ai[u + 1] = 0.25 - u * 1e-9;
                }
            } else
#pragma unroll
            for (int u = 0; u < G; u += 2) {
                if (VAR == 5) {
                    const int4 e = *reinterpret_cast<const int4*>(&sX[w][(j + 2 * u) & 255]);
                    const int4 f = *reinterpret_cast<const int4*>(&sX[w][(j + 2 * u + 128) & 255]);
                    junk ^= e.x ^ e.y ^ e.z ^ e.w ^ f.x ^ f.y ^ f.z ^ f.w;
                }
                const double2 a = *reinterpret_cast<const double2*>(&sA[w][j + u]);
                const double2 b = *reinterpret_cast<const double2*>(&sR[w][j + u]);
                const double2 c = *reinterpret_cast<const double2*>(&sI[w][j + u]);
                A[u] = a.x; A[u + 1] = a.y; ar[u] = b.x; ar[u + 1] = b.y; ai[u] = c.x; ai[u + 1] = c.y;
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double q2 = VAR == 3 ? __dadd_rn(q1[r], A[u]) : rec_step(A[u], x[r], q1[r], q0[r]);
                    if (VAR == 1) {
                    } else if (u & 1) {
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
    for (int r = 0; r < R; ++r) s += aex[r] + aey[r] + aox[r] + aoy[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (junk == 12345u ? 1.0 : 0.0);
}

// map2alm: per stream 1 DMUL + 3 DFMA per step, lane partial summed over S streams and
// written to a transpose row; every 16 steps lane j sums column j over 32 rows (CH chains)
template <int S, int MINB, int CH>
__global__ void __launch_bounds__(128, MINB) m2a_pattern(double* out, int reps) {
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
                        const double q2 = rec_step(A, x[r], q1[r], q0[r]);
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
            double s[CH];
#pragma unroll
            for (int k = 0; k < CH; ++k) s[k] = red[k][lane];
#pragma unroll
            for (int rr = CH; rr < 32; rr += CH)
#pragma unroll
                for (int k = 0; k < CH; ++k) s[k] += red[rr + k][lane];
            double v = 0;
#pragma unroll
            for (int k = 0; k < CH; ++k) v += s[k];
            tot += v;
            __syncwarp();
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
}

template <typename K>
void run(const char* name, K kern, int minb, size_t smem, double fp64_per_warp_rep, double* out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 128, smem);
    const int blocks = sms * per;
    const int reps = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, 128, smem>>>(out, 2);
    cudaEventRecord(e0);
    kern<<<blocks, 128, smem>>>(out, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    // FP64 warp-instruction issue slots: 1 per 2 cycles per SMSP
    const double warp_instr = fp64_per_warp_rep * reps * blocks * 4;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cap = (double)sms * 4 * 0.5 * clk * 1e3 * ms * 1e-3;
    printf("%-28s blocks/SM=%d  %.3f ms  FP64 issue = %.1f%% of the 1-per-2-cycles peak (at %d MHz) %s\n", name, per, ms,
           100.0 * warp_instr / cap, clk / 1000, err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 24);
    // per warp per rep: 128 steps x R streams x 4 FP64
    run("a2m R=4 G=8 minb=3", a2m_pattern<4, 8, 3>, 3, 0, 128.0 * 4 * 4, out);
    run("a2m R=4 G=4 minb=4", a2m_pattern<4, 4, 4>, 4, 0, 128.0 * 4 * 4, out);
    run("a2m R=4 G=8 A-only LDS", a2m_pattern<4, 8, 3, 4>, 3, 0, 128.0 * 4 * 4, out);
    run("a2m R=4 G=8 2x LDS", a2m_pattern<4, 8, 3, 5>, 3, 0, 128.0 * 4 * 4, out);
    run("a2m R=8 G=8 A-only LDS", a2m_pattern<8, 8, 2, 4>, 2, 0, 128.0 * 8 * 4, out);
    run("a2m R=2 G=8 minb=6", a2m_pattern<2, 8, 6>, 6, 0, 128.0 * 2 * 4, out);
    run("a2m R=6 G=4 minb=3", a2m_pattern<6, 4, 3>, 3, 0, 128.0 * 6 * 4, out);
    run("a2m R=8 G=4 minb=2", a2m_pattern<8, 4, 2>, 2, 0, 128.0 * 8 * 4, out);
    const size_t sm = 4 * (128 + 32 * 34) * sizeof(double);
    // per warp per rep: 128 steps x S x 4 + 8 groups x 31 DADD
    run("m2a S=4 minb=4 ch=4", m2a_pattern<4, 4, 4>, 4, sm, 128.0 * 4 * 4 + 8 * 31, out);
    run("m2a S=4 minb=4 ch=8", m2a_pattern<4, 4, 8>, 4, sm, 128.0 * 4 * 4 + 8 * 31, out);
    run("m2a S=8 minb=3 ch=8", m2a_pattern<8, 3, 8>, 3, sm, 128.0 * 8 * 4 + 8 * 31, out);
    run("m2a S=8 minb=2 ch=8", m2a_pattern<8, 2, 8>, 2, sm, 128.0 * 8 * 4 + 8 * 31, out);
    run("m2a S=6 minb=3 ch=8", m2a_pattern<6, 3, 8>, 3, sm, 128.0 * 6 * 4 + 8 * 31, out);
    return 0;
}
