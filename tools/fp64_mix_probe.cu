// FP64 instruction-mix probe (B200): throughput of DFMA / DMUL / DADD with register operands,
// independent chains, 4 warps per SM sub-partition -- what issue rate the Legendre step's
// operand mix (DMUL A*x, DFMA m*q1-q0, DFMA d*q+acc) can reach at best.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_mix_probe.cu -o tools/fp64_mix_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

// MODE 0: DFMA r = r*b + c (3 register operands, b/c per chain)
// MODE 1: DFMA r = r*u + 0.25 (uniform operand, like fp64_probe)
// MODE 2: DMUL r = r*b
// MODE 3: DADD r = r + b
// MODE 4: DMUL t = b*c (independent) ; DFMA r = t*r - d   (the recurrence pair)
// MODE 5: DFMA r = b*c + r (accumulate: 2 fresh operands, chain through r)
template <int MODE>
__global__ void __launch_bounds__(128) mix(double* out, int iters, double u) {
    constexpr int C = 8;
    double r[C], b[C], c[C], d[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        r[k] = 1.0 + threadIdx.x * 1e-6 + k * 1e-3;
        b[k] = 0.999999 - k * 1e-9 + out[k] * 0;  // runtime-ish values
        c[k] = 1e-7 * k + out[8 + k] * 0;
        d[k] = 1e-8 * k + out[16 + k] * 0;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int s = 0; s < 8; ++s)
#pragma unroll
            for (int k = 0; k < C; ++k) {
                if (MODE == 0) r[k] = __fma_rn(r[k], b[k], c[k]);
                if (MODE == 1) r[k] = __fma_rn(r[k], u, 0.25);
                if (MODE == 2) r[k] = __dmul_rn(r[k], b[k]);
                if (MODE == 3) r[k] = __dadd_rn(r[k], b[k]);
                if (MODE == 4) {
                    const double t = __dmul_rn(b[k], c[k] + s);  // s varies: not hoistable after unroll? keep dep on s
                    r[k] = __fma_rn(t, r[k], -d[k]);
                }
                if (MODE == 5) r[k] = __fma_rn(b[k], c[k], r[k]);
            }
        if (MODE == 4 || MODE == 5) {
#pragma unroll
            for (int k = 0; k < C; ++k) { b[k] = __dmul_rn(b[k], r[k]) ; }
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) s += r[k] + b[k];
    out[32 + blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, double instr_per_inner, double* out) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 4, iters = 4000;  // 16 warps per SM: 4 per SMSP
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, 128>>>(out, 10, 0.999999);
    cudaEventRecord(e0);
    kern<<<blocks, 128>>>(out, iters, 0.999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = (double)iters * instr_per_inner * blocks * 4;
    const double cycles = (double)clk * 1e3 * ms * 1e-3;
    printf("%-34s %.3f ms  %.3f cycles per FP64 warp-instruction per SMSP\n", name, ms,
           cycles * sms * 4 / warp_instr);
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 24);
    cudaMemset(out, 0, 1 << 24);
    run("DFMA 3 reg operands", mix<0>, 64, out);
    run("DFMA reg*uniform+imm", mix<1>, 64, out);
    run("DMUL reg*reg", mix<2>, 64, out);
    run("DADD reg+reg", mix<3>, 64, out);
    run("DMUL + DFMA (recurrence pair)", mix<4>, 128 + 8, out);
    run("DFMA accumulate b*c + r", mix<5>, 64 + 8, out);
    return 0;
}
