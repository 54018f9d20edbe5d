// Per-ring Fourier stage for sm_100a: one CTA per ring, the whole ring transform in shared
// memory, all rings of a size class in ONE launch (no per-length plans, no per-ring launches).
//
// Reference semantics (/root/reference/proj):
//   synthesis  ring_synthesis_into   src/fourier.cpp:10-28
//     bins[m mod n] += Delta_m e^{i m phi0}; bins[(n - m mod n) mod n] += conj (m >= 1);
//     inverse unnormalised DFT; real part (so Im Delta_0 is dropped)
//   analysis   ring_analysis_into    src/fourier.cpp:36-56
//     forward unnormalised DFT of the real samples; Delta_m = w bins[m mod n] e^{-i m phi0}
//   DFT        fft::transform        src/fft.cpp:116-132 (mixed radix for 13-smooth lengths,
//              Bluestein otherwise; sign -1 forward, +1 inverse, unnormalised)
//
// B200 design: the real ring of n samples is transformed as ONE complex FFT of length n/2
// (even n; odd n use a length-n complex FFT).  The fold of the a_lm-side Delta row into the
// Hermitian half spectrum is fused into the FFT prologue and the ring samples are written
// straight to the map (synthesis); analysis fuses the R2C split and the aliasing unfold into
// the epilogue and writes Delta^S straight into the (exchange) panel layout.
// 7-smooth lengths run a register-staged in-place Stockham FFT (radix 8/4/2/3/5/7);
// other lengths run Bluestein with a power-of-two convolution in the same buffer.

#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace shtk {

namespace {

// cos/sin(2 pi j / R) for the odd radices
__constant__ double kC3[3] = {1.0, -0.5, -0.5};
__constant__ double kS3[3] = {0.0, 0.86602540378443864676, -0.86602540378443864676};
__constant__ double kC5[5] = {1.0, 0.30901699437494742410, -0.80901699437494742410,
                              -0.80901699437494742410, 0.30901699437494742410};
__constant__ double kS5[5] = {0.0, 0.95105651629515357212, 0.58778525229247312917,
                              -0.58778525229247312917, -0.95105651629515357212};
__constant__ double kC7[7] = {1.0, 0.62348980185873353053, -0.22252093395631440429,
                              -0.90096886790241912624, -0.90096886790241912624,
                              -0.22252093395631440429, 0.62348980185873353053};
__constant__ double kS7[7] = {0.0, 0.78183148246802980871, 0.97492791218182360702,
                              0.43388373911755812048, -0.43388373911755812048,
                              -0.97492791218182360702, -0.78183148246802980871};

template <int R>
__device__ __forceinline__ void dft_generic(double2 (&v)[R], int sign, const double* cs,
                                            const double* sn) {
    double2 out[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        double2 acc = v[0];
#pragma unroll
        for (int r = 1; r < R; ++r) {
            const int e = (r * k) % R;
            const double c = cs[e], s = sign * sn[e];
            acc.x += v[r].x * c - v[r].y * s;
            acc.y += v[r].x * s + v[r].y * c;
        }
        out[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = out[k];
}

__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3, int sign) {
    const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2);
    const double2 t2 = cadd(a1, a3), t3 = cmul_si(csub(a1, a3), sign);
    a0 = cadd(t0, t2);
    a2 = csub(t0, t2);
    a1 = cadd(t1, t3);
    a3 = csub(t1, t3);
}

template <int R>
__device__ __forceinline__ void dft(double2 (&v)[R], int sign) {
    if constexpr (R == 2) {
        const double2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else if constexpr (R == 4) {
        dft4(v[0], v[1], v[2], v[3], sign);
    } else if constexpr (R == 8) {
        double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
        double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
        dft4(e0, e1, e2, e3, sign);
        dft4(o0, o1, o2, o3, sign);
        constexpr double h = 0.70710678118654752440;
        // w^k = e^{sign 2 pi i k / 8}
        const double2 w1 = make_double2(h, sign * h);
        const double2 w3 = make_double2(-h, sign * h);
        o1 = cmul(o1, w1);
        o2 = cmul_si(o2, sign);
        o3 = cmul(o3, w3);
        v[0] = cadd(e0, o0);
        v[4] = csub(e0, o0);
        v[1] = cadd(e1, o1);
        v[5] = csub(e1, o1);
        v[2] = cadd(e2, o2);
        v[6] = csub(e2, o2);
        v[3] = cadd(e3, o3);
        v[7] = csub(e3, o3);
    } else if constexpr (R == 3) {
        dft_generic<3>(v, sign, kC3, kS3);
    } else if constexpr (R == 5) {
        dft_generic<5>(v, sign, kC5, kS5);
    } else if constexpr (R == 7) {
        dft_generic<7>(v, sign, kC7, kS7);
    }
}

// b / Ns and b % Ns for b < 2^24 through a float reciprocal (exact after one correction).
__device__ __forceinline__ void divmod_small(int b, int Ns, float inv, int& q, int& r) {
    q = __float2int_rz(__int2float_rn(b) * inv);
    r = b - q * Ns;
    if (r >= Ns) { ++q; r -= Ns; }
    if (r < 0) { --q; r += Ns; }
}

// One in-place Stockham pass (register staged): all inputs of the pass are read into
// registers, then the CTA synchronises and writes the outputs.
// e^{-2 pi i k / B} = lo[k & 63] * hi[k >> 6] from exact table entries (shared memory)
struct TwTab {
    const double2* lo;
    const double2* hi;
    __device__ __forceinline__ double2 at(int k) const { return cmul(lo[k & 63], hi[k >> 6]); }
};

template <int R, int T, int BMAX>
__device__ __forceinline__ void stockham_pass(double2* buf, int B, int Ns, int sign,
                                              const TwTab& tw) {
    constexpr int Q = (BMAX + R * T - 1) / (R * T);
    const int nb = B / R;
    const int tstride = B / (Ns * R);
    const float inv = 1.0f / (float)Ns;
    double2 v[Q][R];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int b = threadIdx.x + q * T;
        if (b < nb) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[q][r] = buf[b + r * nb];
            if (Ns > 1) {
                int bq, k;
                divmod_small(b, Ns, inv, bq, k);
                // w^r for r = 1..R-1 from one table lookup, as a running product (2 live
                // complex temporaries; error grows by ~1 ulp per power, <= 7 ulp)
                double2 w = tw.at(k * tstride);
                if (sign > 0) w.y = -w.y;
                double2 wr = w;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    v[q][r] = cmul(v[q][r], wr);
                    if (r + 1 < R) wr = cmul(wr, w);
                }
            }
            dft<R>(v[q], sign);
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int b = threadIdx.x + q * T;
        if (b < nb) {
            int bq, k;
            divmod_small(b, Ns, inv, bq, k);
            const int base = bq * Ns * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) buf[base + r * Ns] = v[q][r];
        }
    }
    __syncthreads();
}

template <int T, int BMAX>
__device__ __forceinline__ void fft_run(double2* buf, int npass, unsigned long long radices, int B,
                                     int sign, const TwTab& tw) {
    int Ns = 1;
    for (int pidx = 0; pidx < npass; ++pidx) {
        const int R = (int)((radices >> (4 * pidx)) & 0xF);
        switch (R) {
            case 8: stockham_pass<8, T, BMAX>(buf, B, Ns, sign, tw); break;
            case 4: stockham_pass<4, T, BMAX>(buf, B, Ns, sign, tw); break;
            case 2: stockham_pass<2, T, BMAX>(buf, B, Ns, sign, tw); break;
            default:
                // odd radices only in the small classes (register budget of the in-place
                // staging); the planner sends larger non-power-of-two lengths to Bluestein
                if constexpr (BMAX <= 1024) {
                    if (R == 3) stockham_pass<3, T, BMAX>(buf, B, Ns, sign, tw);
                    else if (R == 5) stockham_pass<5, T, BMAX>(buf, B, Ns, sign, tw);
                    else if (R == 7) stockham_pass<7, T, BMAX>(buf, B, Ns, sign, tw);
                }
                break;
        }
        Ns *= R;
    }
}

// Length-N DFT (sign) of buf[0..N) in place; Bluestein rings use the whole B-length buffer
// (chirp, forward FFT_B, multiply by FFT_B(conj chirp), inverse FFT_B, chirp / B).
// Stage the two-level twiddle table of length B (64 + B/64 entries) into twsm.
template <int T>
__device__ __forceinline__ TwTab stage_twiddles(double2* twsm, const double2* __restrict__ tw, int B) {
    const int nhi = (B + 63) >> 6;
    for (int j = threadIdx.x; j < 64 + nhi; j += T) {
        if (j < 64) twsm[j] = (j < B) ? __ldg(&tw[j]) : make_double2(1.0, 0.0);
        else twsm[j] = __ldg(&tw[(j - 64) << 6]);
    }
    return TwTab{twsm, twsm + 64};
}

template <int T, int BMAX>
__device__ void ring_dft(double2* buf, const RingDesc& d, int sign,
                         const double2* __restrict__ tabs, double2* twsm) {
    const TwTab tw = stage_twiddles<T>(twsm, tabs + d.tw_off, d.B);  // published by a barrier below
    const bool blue = d.flags & 2;
    const int N = d.N, M = d.B;
    const double2* __restrict__ chirp = tabs + d.chirp_off;
    const double2* __restrict__ H = tabs + d.h_off;
    if (blue) {
        for (int j = threadIdx.x; j < M; j += T) {
            if (j < N) {
                double2 c = __ldg(&chirp[j]);
                if (sign > 0) c.y = -c.y;
                buf[j] = cmul(buf[j], c);
            } else {
                buf[j] = make_double2(0.0, 0.0);
            }
        }
        __syncthreads();
    }
    if (!blue) __syncthreads();
    const int nrun = blue ? 2 : 1;
    for (int run = 0; run < nrun; ++run) {
        const int sg = blue ? (run == 0 ? -1 : +1) : sign;
        fft_run<T, BMAX>(buf, d.npass, d.radices, M, sg, tw);
        if (blue && run == 0) {
            for (int j = threadIdx.x; j < M; j += T) {
                double2 h = __ldg(&H[j]);
                if (sign > 0) h.y = -h.y;
                buf[j] = cmul(buf[j], h);
            }
            __syncthreads();
        }
    }
    if (blue) {
        const double inv = 1.0 / (double)M;
        for (int j = threadIdx.x; j < N; j += T) {
            double2 c = __ldg(&chirp[j]);
            if (sign > 0) c.y = -c.y;
            buf[j] = cscale(cmul(buf[j], c), inv);
        }
        __syncthreads();
    }
}

// e^{i m phi0} = lo[m & 63] * hi[m >> 6]: 64 + (mmax+1)/64 sincos per ring instead of one per
// order (ring_synthesis_into evaluates polar(1, m*phi0) per order, fourier.cpp:13).
struct PhaseTab {
    const double2* lo;
    const double2* hi;
    __device__ __forceinline__ double2 at(int m) const { return cmul(lo[m & 63], hi[m >> 6]); }
};

__device__ __forceinline__ void build_phase(double2* lo, double2* hi, int nhi, double phi0, int T) {
    for (int j = threadIdx.x; j < 64 + nhi; j += T) {
        double s, c;
        if (j < 64) {
            sincos((double)j * phi0, &s, &c);
            lo[j] = make_double2(c, s);
        } else {
            sincos((double)((j - 64) * 64) * phi0, &s, &c);
            hi[j - 64] = make_double2(c, s);
        }
    }
}

__device__ __forceinline__ int64_t delta_index(const RingStageArgs& a, int pos, int m) {
    return a.m_base ? a.m_base[m] + (int64_t)pos * a.m_stride[m] : (int64_t)m + (int64_t)pos * a.ld;
}
__device__ __forceinline__ double2 delta_at(const RingStageArgs& a, int pos, int m) {
    return a.delta_in[delta_index(a, pos, m)];
}

// v_m = Delta_m e^{i m phi0} as in ring_synthesis_into (fourier.cpp:11-14); m==0 keeps Re only.
__device__ __forceinline__ double2 folded_value(const RingStageArgs& a, int pos, int m,
                                                bool rot, const PhaseTab& ph) {
    double2 v = delta_at(a, pos, m);
    if (m == 0) return make_double2(v.x, 0.0);
    if (rot) v = cmul(v, ph.at(m));
    return v;
}

// Fold sums of bin pair p over the wraps w = g, g+G, ... (ring_synthesis_into's bins,
// fourier.cpp:17-25): H_p = sum_{m = p mod n} v_m + sum_{m = -p mod n, m >= 1} conj v_m.
__device__ __forceinline__ void fold_pair(const RingStageArgs& a, int pos, int p, int g, int G,
                                          int n, int N, bool half, int mmax, bool rot,
                                          const PhaseTab& ph, double2& hp, double2& hq) {
    hp = make_double2(0.0, 0.0);
    hq = make_double2(0.0, 0.0);
    const int q = half ? N - p : -1;
    for (int w = g;; w += G) {
        const int base = w * n;
        if (base > mmax) break;
        if (p == 0) {
            // bin 0 (and bin N in half mode): the conjugate lands on the same bin -> 2 Re
            const double2 v = folded_value(a, pos, base, rot, ph);
            hp.x += (base == 0) ? v.x : 2.0 * v.x;
            if (half && base + N <= mmax) hq.x += 2.0 * folded_value(a, pos, base + N, rot, ph).x;
        } else {
            int m = base + p;
            if (m <= mmax) hp = cadd(hp, folded_value(a, pos, m, rot, ph));
            m = base + n - p;
            if (m <= mmax) hp = cadd(hp, cconj(folded_value(a, pos, m, rot, ph)));
            if (half && q != p) {
                m = base + q;  // H_q: bin q (v) and bin n - q = N + p (conj v)
                if (m <= mmax) hq = cadd(hq, folded_value(a, pos, m, rot, ph));
                m = base + N + p;
                if (m <= mmax) hq = cadd(hq, cconj(folded_value(a, pos, m, rot, ph)));
            }
        }
    }
}

// Half mode: Z_k = (H_k + conj H_{N-k}) + i (H_k - conj H_{N-k}) e^{+2 pi i k/n} for k = p and
// k = N-p (C2R of length n as a complex length-N inverse FFT).  Full mode: Hermitian bins.
__device__ __forceinline__ void store_z(double2* buf, const double2* __restrict__ hw, int p,
                                       double2 Hp, double2 Hq, int n, int N, bool half) {
    if (half) {
        const int q = N - p;
        if (q == p) Hq = Hp;  // N even, k = N/2 pairs with itself
        {
            const double2 e = cadd(Hp, cconj(Hq));
            const double2 o = cmul(csub(Hp, cconj(Hq)), cconj(__ldg(&hw[p])));
            buf[p] = cadd(e, cmul_si(o, +1));
        }
        if (q != p && q < N) {
            const double2 e = cadd(Hq, cconj(Hp));
            const double2 o = cmul(csub(Hq, cconj(Hp)), cconj(__ldg(&hw[q])));
            buf[q] = cadd(e, cmul_si(o, +1));
        }
    } else {
        buf[p] = Hp;
        if (p > 0) buf[n - p] = cconj(Hp);
    }
}

}  // namespace

// ---------------------------------------------------------------------------------------
// synthesis: Delta rows -> ring samples
// ---------------------------------------------------------------------------------------
template <int T, int BMAX>
__global__ void __launch_bounds__(T, (T >= 1024 ? 1 : 1024 / T)) ring_synth_kernel(RingStageArgs a) {
    extern __shared__ __align__(16) double2 smem[];
    double2* buf = smem;               // BMAX
    double2* red = smem + BMAX;        // 2T fold partials
    double2* twsm = red + 2 * T;       // 64 + BMAX/64 twiddles
    double2* phlo = twsm + 64 + (BMAX >> 6);  // 64 + (mmax >> 6) + 1 phase factors
    const RingDesc d = a.rings[blockIdx.x];
    const int n = d.n, N = d.N, pos = d.ring_pos, mmax = a.mmax;
    const bool half = d.flags & 1;
    const double phi0 = d.phi0;
    const bool rot = phi0 != 0.0;
    const PhaseTab ph{phlo, phlo + 64};
    if (rot) {
        build_phase(phlo, phlo + 64, (mmax >> 6) + 1, phi0, T);
        __syncthreads();
    }

    // ---- fold Delta into the Hermitian half spectrum H_k (k = 0..n/2) ----
    // half mode: bin pair p handles H_p and H_{N-p}; full mode: H_p only.  When the pairs fit
    // the CTA several thread groups split the wraps of m (aliasing for small rings) and are
    // reduced in a fixed order; otherwise each thread walks pairs with a CTA stride.
    const int np = half ? (N / 2 + 1) : ((n - 1) / 2 + 1);
    const int t = threadIdx.x;
    const double2* __restrict__ hw = a.tabs + d.hw_off;
    if (np <= T) {
        const int G = T / np;
        if (t < G * np) {
            const int g = t / np, p = t - g * np;
            double2 hp, hq;
            fold_pair(a, pos, p, g, G, n, N, half, mmax, rot, ph, hp, hq);
            red[2 * t] = hp;
            red[2 * t + 1] = hq;
        }
        __syncthreads();
        if (t < np) {
            double2 Hp = make_double2(0.0, 0.0), Hq = make_double2(0.0, 0.0);
            for (int g = 0; g < G; ++g) {
                Hp = cadd(Hp, red[2 * (g * np + t)]);
                Hq = cadd(Hq, red[2 * (g * np + t) + 1]);
            }
            store_z(buf, hw, t, Hp, Hq, n, N, half);
        }
    } else {
        for (int p = t; p < np; p += T) {
            double2 Hp, Hq;
            fold_pair(a, pos, p, 0, 1, n, N, half, mmax, rot, ph, Hp, Hq);
            store_z(buf, hw, p, Hp, Hq, n, N, half);
        }
    }
    __syncthreads();

    ring_dft<T, BMAX>(buf, d, +1, a.tabs, twsm);

    double* __restrict__ out = a.map_out + d.pix_off;
    if (half) {
        for (int j = t; j < N; j += T) {
            const double2 z = buf[j];
            out[2 * j] = z.x;
            out[2 * j + 1] = z.y;
        }
    } else {
        for (int j = t; j < n; j += T) out[j] = buf[j].x;
    }
}

// ---------------------------------------------------------------------------------------
// analysis: ring samples -> Delta^S rows
// ---------------------------------------------------------------------------------------
template <int T, int BMAX>
__global__ void __launch_bounds__(T, (T >= 1024 ? 1 : 1024 / T)) ring_anal_kernel(RingStageArgs a) {
    extern __shared__ __align__(16) double2 smem[];
    double2* buf = smem;
    double2* red = smem + BMAX;
    double2* twsm = red + 2 * T;
    double2* phlo = twsm + 64 + (BMAX >> 6);
    const RingDesc d = a.rings[blockIdx.x];
    const int n = d.n, N = d.N, pos = d.ring_pos, mmax = a.mmax;
    const bool half = d.flags & 1;
    const double phi0 = d.phi0, wgt = d.weight;
    const bool rot = phi0 != 0.0;
    const PhaseTab ph{phlo, phlo + 64};
    const double* __restrict__ in = a.map_in + d.pix_off;
    const int t = threadIdx.x;
    if (rot) build_phase(phlo, phlo + 64, (mmax >> 6) + 1, phi0, T);  // ordered by later barriers

    if (half) {
        for (int j = t; j < N; j += T) buf[j] = make_double2(in[2 * j], in[2 * j + 1]);
    } else {
        for (int j = t; j < n; j += T) buf[j] = make_double2(in[j], 0.0);
    }
    __syncthreads();

    ring_dft<T, BMAX>(buf, d, -1, a.tabs, twsm);

    if (half) {
        // B_k = E_k + e^{-2 pi i k/n} O_k, E = (Z_k + conj Z_{N-k})/2, O = -i (Z_k - conj Z_{N-k})/2
        const double2* __restrict__ hw = a.tabs + d.hw_off;
        const int np = N / 2 + 1;
        // each bin pair (p, N-p) reads and writes only its own two slots: no cross-thread hazard
        for (int p = t; p < np; p += T) {
            const int q = N - p;
            const double2 Zp = buf[p];
            const double2 Zq = buf[q % N];
            double2 Bp, Bq;
            {
                const double2 e = cscale(cadd(Zp, cconj(Zq)), 0.5);
                const double2 o = cmul_si(cscale(csub(Zp, cconj(Zq)), 0.5), -1);
                Bp = cadd(e, cmul(__ldg(&hw[p]), o));
            }
            {
                const double2 e = cscale(cadd(Zq, cconj(Zp)), 0.5);
                const double2 o = cmul_si(cscale(csub(Zq, cconj(Zp)), 0.5), -1);
                Bq = cadd(e, cmul(__ldg(&hw[q]), o));
            }
            buf[p] = Bp;
            if (q == N) red[0] = Bq;  // B_N (Nyquist) beside the buffer
            else if (q != p) buf[q] = Bq;
        }
        __syncthreads();
    }

    // ---- unfold: Delta^S_m = w * bins[m mod n] * e^{-i m phi0} (fourier.cpp:42-47) ----
    for (int m = t; m <= mmax; m += T) {
        const int b = m % n;
        double2 val;
        if (half) {
            if (b < N) val = buf[b];
            else if (b == N) val = red[0];
            else val = cconj(buf[n - b]);
        } else {
            val = buf[b];
        }
        double2 v = cscale(val, wgt);
        if (rot && m > 0) v = cmul(v, cconj(ph.at(m)));
        a.delta_out[delta_index(a, pos, m)] = v;
    }
}

// ---------------------------------------------------------------------------------------
// plan-time tables
// ---------------------------------------------------------------------------------------
__global__ void fill_tables_kernel(const TableJob* __restrict__ jobs, double2* __restrict__ tabs) {
    const TableJob jb = jobs[blockIdx.y];
    const int count = jb.kind == 1 ? jb.L / 2 + 1 : jb.L;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) {
        double s, c;
        if (jb.kind == 2) {
            const long long e = ((long long)k * k) % (2LL * jb.L);
            sincospi((double)e / (double)jb.L, &s, &c);  // e^{-i pi e / L}
        } else {
            sincospi(2.0 * (double)k / (double)jb.L, &s, &c);  // e^{-2 pi i k / L}
        }
        tabs[jb.off + k] = make_double2(c, -s);
    }
}

void launch_fill_tables(const TableJob* jobs_dev, int n_jobs, double2* tabs, cudaStream_t s) {
    for (int j0 = 0; j0 < n_jobs; j0 += 65535) {
        const int nj = n_jobs - j0 < 65535 ? n_jobs - j0 : 65535;
        fill_tables_kernel<<<dim3(16, nj), 256, 0, s>>>(jobs_dev + j0, tabs);
    }
}

template <int T, int BMAX>
__global__ void __launch_bounds__(T, 1) bluestein_h_kernel(const RingDesc* __restrict__ descs,
                                                        double2* __restrict__ tabs) {
    extern __shared__ __align__(16) double2 smem[];
    double2* buf = smem;
    const RingDesc d = descs[blockIdx.x];
    const int N = d.N, M = d.B;
    const double2* chirp = tabs + d.chirp_off;
    // h_d = conj(chirp_d) for |d| < N, cyclic in M
    for (int j = threadIdx.x; j < M; j += T) {
        double2 v = make_double2(0.0, 0.0);
        if (j < N) v = cconj(chirp[j]);
        else if (j > M - N) v = cconj(chirp[M - j]);
        buf[j] = v;
    }
    __syncthreads();
    const TwTab tw = stage_twiddles<T>(buf + BMAX, tabs + d.tw_off, M);
    __syncthreads();
    fft_run<T, BMAX>(buf, d.npass, d.radices, M, -1, tw);
    for (int j = threadIdx.x; j < M; j += T) tabs[d.h_off + j] = buf[j];
}

// ---------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------
namespace {
constexpr int kBmax[FFT_N_CLASSES] = {256, 1024, 4096, 8192};
constexpr int kThr[FFT_N_CLASSES] = {64, 256, 512, 1024};

// buffer + fold partials + phase table (orders up to kMaxPhaseM)
constexpr int kMaxPhaseM = 65535;
template <int C>
size_t class_smem(int mmax) {
    return (size_t)kBmax[C] * sizeof(double2) + 2 * (size_t)kThr[C] * sizeof(double2) +
           (size_t)(64 + (kBmax[C] >> 6)) * sizeof(double2) +
           (size_t)(64 + (mmax >> 6) + 1) * sizeof(double2);
}

template <int C, class K>
void set_smem_attr(K kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)class_smem<C>(kMaxPhaseM));
}

template <int C>
void synth_c(const RingStageArgs& a, cudaStream_t s) {
    static bool once = (set_smem_attr<C>(ring_synth_kernel<kThr[C], kBmax[C]>), true);
    (void)once;
    for (int r0 = 0; r0 < a.n_rings; r0 += 65535) {
        RingStageArgs b = a;
        b.rings = a.rings + r0;
        const int nr = a.n_rings - r0 < 65535 ? a.n_rings - r0 : 65535;
        ring_synth_kernel<kThr[C], kBmax[C]><<<nr, kThr[C], class_smem<C>(a.mmax), s>>>(b);
    }
}
template <int C>
void anal_c(const RingStageArgs& a, cudaStream_t s) {
    static bool once = (set_smem_attr<C>(ring_anal_kernel<kThr[C], kBmax[C]>), true);
    (void)once;
    for (int r0 = 0; r0 < a.n_rings; r0 += 65535) {
        RingStageArgs b = a;
        b.rings = a.rings + r0;
        const int nr = a.n_rings - r0 < 65535 ? a.n_rings - r0 : 65535;
        ring_anal_kernel<kThr[C], kBmax[C]><<<nr, kThr[C], class_smem<C>(a.mmax), s>>>(b);
    }
}
template <int C>
void blue_c(const RingDesc* descs, int n, double2* tabs, cudaStream_t s) {
    static bool once = (set_smem_attr<C>(bluestein_h_kernel<kThr[C], kBmax[C]>), true);
    (void)once;
    for (int r0 = 0; r0 < n; r0 += 65535) {
        const int nr = n - r0 < 65535 ? n - r0 : 65535;
        bluestein_h_kernel<kThr[C], kBmax[C]><<<nr, kThr[C], class_smem<C>(0), s>>>(descs + r0, tabs);
    }
}
}  // namespace

int fft_class_bmax(int c) { return kBmax[c]; }
int fft_class_for(int B) {
    for (int c = 0; c < FFT_N_CLASSES; ++c)
        if (B <= kBmax[c]) return c;
    return -1;
}

void launch_ring_synthesis(int cls, const RingStageArgs& a, cudaStream_t s) {
    if (a.n_rings == 0) return;
    switch (cls) {
        case 0: synth_c<0>(a, s); break;
        case 1: synth_c<1>(a, s); break;
        case 2: synth_c<2>(a, s); break;
        case 3: synth_c<3>(a, s); break;
    }
}
void launch_ring_analysis(int cls, const RingStageArgs& a, cudaStream_t s) {
    if (a.n_rings == 0) return;
    switch (cls) {
        case 0: anal_c<0>(a, s); break;
        case 1: anal_c<1>(a, s); break;
        case 2: anal_c<2>(a, s); break;
        case 3: anal_c<3>(a, s); break;
    }
}
void launch_bluestein_h(int cls, const RingDesc* descs_dev, int n, double2* tabs,
                        cudaStream_t s) {
    if (n == 0) return;
    switch (cls) {
        case 0: blue_c<0>(descs_dev, n, tabs, s); break;
        case 1: blue_c<1>(descs_dev, n, tabs, s); break;
        case 2: blue_c<2>(descs_dev, n, tabs, s); break;
        case 3: blue_c<3>(descs_dev, n, tabs, s); break;
    }
}

// ---------------------------------------------------------------------------------------
// FP64 peak probe: independent DFMA chains, resident on every SM
// ---------------------------------------------------------------------------------------
__global__ void dfma_peak_kernel(double* out, int iters) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
    double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
    const double b = 0.999999999, c = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (r == 1234.5) out[0] = r;  // keep the chains alive
}

void launch_dfma_peak(double* out, int blocks, int threads, int iters, cudaStream_t s) {
    dfma_peak_kernel<<<blocks, threads, 0, s>>>(out, iters);
}

}  // namespace shtk
