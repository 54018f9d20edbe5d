// Host-side launch interface of the sm_100a kernels (internal to libshtc).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace shtk {

// Every kernel launch of the library is counted (process-wide), so a caller can state how many
// of the library's kernels ran inside a timed region (shtc_kernel_launches).
void count_launch();
unsigned long long launch_count();

// ---------------------------------------------------------------------------------------
// Legendre stage
// ---------------------------------------------------------------------------------------

// Streams of the recurrence: one per mirror pair (north, south) or per unpaired ring.
struct LegStreams {
    const double* x;       // cos(theta) of the north member
    const double* log2s2;  // log2((1-x)(1+x)) computed on the host with glibc (parity)
    const int* s2pos;      // (1-x)(1+x) > 0
    const int* north;      // ring index of the north member
    const int* south;      // ring index of the south member, -1 if unpaired
    int n;
};

// Per-order recurrence tables for the renormalised recurrence
//   Q_l = (A_l x) Q_{l-1} - Q_{l-2},   P_l = c_l Q_l,   activation threshold T_l = 2^512 / c_l
// stored per order m contiguously for i = l - m = 0..lmax-m at tab_off[mi].
struct LegTables {
    double* A;
    double* C;
    double* T;
    const int64_t* tab_off;
};

// Tile = LEG_TILE consecutive streams handled by one warp (32 lanes x LEG_R streams).
#ifndef LEG_R_DEF
#define LEG_R_DEF 4
#endif
constexpr int LEG_R = LEG_R_DEF;
constexpr int LEG_TILE = 32 * LEG_R;
constexpr int LEG_WARPS = 4;      // warps per block of the persistent Legendre kernels
// Degree steps staged per chunk (LEG_CL / 32 entries per lane; the next chunk's raw entries
// are held in registers across the current chunk).  Measured at C4 with the round-2 kernels:
// alm2map 6.88 / 6.83 / 6.83 / 6.90 ms at 128 / 96 / 64 / 32; map2alm 8.30 / 8.25 / 8.25 /
// 8.13 ms (its 8-stream lanes sit at the 168-register cap: every prefetched entry costs a
// register, and at 32 nothing spills).
#ifndef LEG_CL_DEF
#define LEG_CL_DEF 64
#endif
#ifndef LEG_M2A_CL_DEF
#define LEG_M2A_CL_DEF 32
#endif
constexpr int LEG_CL = LEG_CL_DEF;          // alm2map
constexpr int LEG_M2A_CL = LEG_M2A_CL_DEF;  // map2alm
static_assert(LEG_CL % 32 == 0 && LEG_M2A_CL % 32 == 0, "whole entries per lane");
#ifndef LEG_A2M_P
#define LEG_A2M_P 1  // tiles an alm2map warp runs at once; 2 (8 streams per lane) measured slower at C4:
                     // 7.0 ms at 2 CTAs/SM, 7.4 ms at 3 (spills) against 6.89 ms
#endif
#ifndef LEG_A2M_MINB
#define LEG_A2M_MINB 4  // resident CTAs per SM the alm2map kernel is compiled for (122 registers)
#endif
#ifndef LEG_M2A_P
#define LEG_M2A_P 2  // tiles a map2alm warp runs at once (LEG_R x LEG_M2A_P streams per lane)
#endif
#ifndef LEG_M2A_MINB
#define LEG_M2A_MINB (LEG_M2A_P > 1 ? 3 : 4)
#endif
#ifndef LEG_M2A_GROUP_DEF
#define LEG_M2A_GROUP_DEF 4
#endif
constexpr int LEG_M2A_GROUP = LEG_M2A_GROUP_DEF;  // tiles per map2alm work item (partials reduce G-fold)
#ifndef LEG_M2A_ITEMS_PER_WARP
#define LEG_M2A_ITEMS_PER_WARP 8  // fewer tiles per item when a plan has fewer items per resident warp
#endif

// One warp-sized unit of work of the persistent kernels.
//   alm2map: (mi, tile id, second tile id or -1, -); map2alm: (mi, first index into tile_list, tile count, item
//   index g within the order), items of an order write partial sums into scratch slots.
struct LegItem {
    int mi, a, b, g;
};

struct LegPlanView {
    int lmax;
    int n_m;
    const int* ms;             // [n_m] ascending orders
    const double* log_mu;      // [mmax+1] indexed by m (host glibc lgamma)
    double exp_lmu0;           // exp(log_mu(0)) from the host (pmm_from_log m==0 path)
    LegTables tab;
    LegStreams st;
    int n_tiles;               // ceil(st.n / LEG_TILE)
    const int2* tile_info;     // [n_m * n_tiles]: (i_s, i_e) activation window, i_s < 0: dead
    const int* tile_list;      // alive tiles, grouped per order
    const int* tile_list_off;  // [n_m]
    const int* tile_list_cnt;  // [n_m]
    const LegItem* a2m_items;  // cost-descending
    int n_a2m_items;
    const LegItem* m2a_items;  // cost-descending
    int n_m2a_items;
    const double2* ck_q;       // [n_m * st.n] (Q_{act-1}, Q_act) at activation, k == 0 scale
    const int* ck_act;         // [n_m * st.n] activation step (0: seed; INT_MAX: dead)
    const int* m2a_items_per_m;     // [n_m]
    const int64_t* m2a_slot_base;   // [n_m] double2 offset of the order's first partial slot
    int64_t m2a_scratch_elems;
    // map2alm: 0 = the last item of an order to finish sums the order's partial slots;
    // 1 = the slots are left for leg_m2a_finalize (launched once the order's items are done)
    int defer_final;
    // fused exchange (alm2map): ring r's output row is row_ptr[r] (an address in the ring
    // owner's receive buffer, peer memory) instead of delta + row_off[r]; nullptr: local
    double2* const* row_ptr;
    // element (ring r, order index mi) of the alm2map output at row + mi * row_stride[r]
    // (nullptr: stride 1, rows of contiguous orders).  m-major exchange blocks (order-major
    // [|M_i| x |R_j|], stride |R_j|) make a warp's stores -- consecutive rings -- contiguous.
    const int64_t* row_stride;
    // ScaleLadder::unscaled() (legendre.hpp:26-47, the reference's transparency check): no
    // rescaling, so a stream counts from its seed if the seed is at scale k == 0 and never
    // otherwise (plan-time only: it changes the activation scan)
    int unscaled;
};

void launch_leg_tables(const int* ms_dev, int n_m, int lmax, LegTables tab, cudaStream_t s);
// activation degree offset per (order, stream) (INT_MAX = dead stream) and the recurrence
// state right after it (same arithmetic as the reference's prefix, so bit-identical).
void launch_leg_scan(const LegPlanView& p, int* act_dev, double2* ck_dev, cudaStream_t s);
// per (order, tile) activation window and useful-step totals.
void launch_leg_tile_summary(const LegPlanView& p, const int* act_dev, int2* tile_info_dev,
                             unsigned long long* useful_dev, cudaStream_t s);

// A tile's run starts at the even step ic = i_s & ~1 (i_s: its first activation).
__host__ __device__ inline int leg_tile_start(int is) { return is >= 2 ? (is & ~1) : 0; }

// Delta rows: element (ring r, order index mi) at delta[row_off[r] + mi].
// counters: >= 1 + n_m ints of device scratch (zeroed by the launcher).
// phases: bit0 = zero pass (dead tiles / orders without alive tiles), bit1 = the persistent
// kernel over p's item list (callers may pass a view restricted to one chunk of items).
// bit3 = the
// caller has zeroed the queue counter: concurrent launches on different streams each get
// their own queue word.
constexpr int LEG_PHASE_ZERO = 1, LEG_PHASE_MAIN = 2, LEG_PHASE_ALL = 3, LEG_PHASE_NO_RESET = 8;
void launch_leg_alm2map(const LegPlanView& p, const double2* alm, double2* delta,
                        const int64_t* row_off, int* counters, cudaStream_t s,
                        int phases = LEG_PHASE_ALL);
// a_lm (= or +=) sum over streams; accumulate != 0 adds into alm.  scratch: m2a_scratch_elems.
// counters[0] is the work queue.  Unless p.defer_final, a finalize kernel sums every order's
// slots after the main kernel (pipelined band launches call launch_leg_m2a_finalize
// themselves once an order's last launch is done).
void launch_leg_map2alm(const LegPlanView& p, const double2* delta, const int64_t* row_off,
                        double2* alm, int accumulate, int* counters, double2* scratch,
                        cudaStream_t s, int phases = LEG_PHASE_ALL);
int leg_persistent_blocks(int device);
int leg_m2a_warps(int device);  // resident warps of the persistent map2alm kernel
// a_lm of the listed order indices from their partial slots (p's item set): slots summed in
// slot order, scaled by c_l, stored (or added when accumulate) -- one thread per coefficient
void launch_leg_m2a_finalize(const LegPlanView& p, const int* mis, int n_mis, const double2* scratch,
                             double2* alm, int accumulate, cudaStream_t s);

// ---------------------------------------------------------------------------------------
// Ring Fourier stage
// ---------------------------------------------------------------------------------------
constexpr int FFT_MAX_PASSES = 16;

struct RingDesc {
    int64_t pix_off;    // first pixel of the ring in the map
    int64_t tw_off;     // e^{-2 pi i k / B}, k < B
    int64_t hw_off;     // e^{-2 pi i k / n}, k <= N (half mode)
    int64_t chirp_off;  // Bluestein chirp e^{-i pi (j^2 mod 2N)/N}, j < N
    int64_t h_off;      // Bluestein FFT_B of conj(chirp) (cyclic), B entries
    int64_t ph_off;     // e^{i m phi0}: m < 64, then m = 64 j (j <= mmax / 64); phi0 != 0 only
    double phi0;
    double weight;
    int n;              // samples on the ring
    int N;              // complex transform length (n/2 if n even, else n)
    int B;              // buffer length (N if 7-smooth, else Bluestein power of two >= 2N-1)
    int flags;          // bit0: half-length real trick, bit1: Bluestein
    int ring_pos;       // row position of the ring in the Delta panel addressing
    int npass;
    unsigned long long radices;  // radix of pass p in bits [4p, 4p+4)
    int K;              // odd rings of the 2-CTA cluster class: one-sided spectrum length
                        // min(n, mmax + 1) (pruned Bluestein: n + K - 1 <= 16384)
    int pad_[3];        // 16-byte multiple (descriptors are staged with 16-byte async copies)
};

struct RingStageArgs {
    const RingDesc* rings;
    int n_rings;
    const double2* tabs;
    int mmax;
    const int64_t* m_base;    // Delta(ring_pos, m) at m_base[m] + ring_pos * m_stride[m],
    const int64_t* m_stride;  // or (m_base == nullptr) at m + ring_pos * ld
    int64_t ld;
    const double2* delta_in;  // synthesis
    double2* delta_out;       // analysis
    const double* map_in;     // analysis
    double* map_out;          // synthesis
    int* counter;             // power-of-two engine: ring queue of this launch (zeroed)
    const double2* p2_tw;     // power-of-two engine: e^{-2 pi i k/B}, k < B, of the class
    // fused exchange (analysis): Delta^S(ring_pos, m) goes to col_ptr[m] + ring_pos *
    // m_stride[m] (an address in the order owner's send buffer, peer memory); nullptr: local
    double2* const* col_ptr;
    // analysis: the order in which the unfold visits m (thread t takes m_order[t + T j]); the
    // exchange layouts list orders grouped by owner so consecutive threads store into one
    // owner's block contiguously.  nullptr: ascending m.
    const int* m_order;
    // 1: the class runs its alternative kernel (8192-point Bluestein: two 4096-point halves per
    // CTA, p2_tw = the 4096-point table); chosen at plan time (every ring n > mmax)
    int alt;
};

// size classes.  Generic (any 7-smooth length, in-place mixed radix, odd-length rings):
//   0: B<=256 (64 thr), 1: B<=1024 (256), 2: B<=4096 (512), 3: B<=8192 (1024).
// Power-of-two engine (half-mode rings with a power-of-two buffer B = 256, 512, ..., 8192):
//   4..9 direct FFTs of length B, 10..15 Bluestein convolutions of length B.
// Cluster class: Bluestein buffers of 16384 points, one ring per 2-CTA cluster (class 16).
constexpr int FFT_N_GENERIC = 4;
constexpr int FFT_P2_MIN = 256, FFT_P2_MAX = 8192, FFT_N_P2 = 6;
constexpr int FFT_P2C_CLASS = FFT_N_GENERIC + 2 * FFT_N_P2, FFT_P2C_B = 16384;
constexpr int FFT_N_CLASSES = FFT_P2C_CLASS + 1;
int fft_class_bmax(int c);
int fft_class_for(int B);     // generic class, -1 if unsupported
int fft_p2_class_for(int B, bool bluestein);  // power-of-two engine class, -1: not one of its lengths

void launch_ring_synthesis(int cls, const RingStageArgs& a, cudaStream_t s);
void launch_ring_analysis(int cls, const RingStageArgs& a, cudaStream_t s);

// Plan-time tables.
struct TableJob {
    int64_t off;
    int L;     // length parameter
    int kind;  // 0: e^{-2 pi i k/L}, k<L ; 1: e^{-2 pi i k/L}, k<=L/2 ; 2: chirp, k<L ;
               // 3: phase factors of phi0, k < L = 64 + mmax/64 + 1
    double phi0;
};
void launch_fill_tables(const TableJob* jobs_dev, int n_jobs, double2* tabs, cudaStream_t s);
// For each Bluestein ring descriptor (deduplicated by N): tabs[h_off..] = FFT_B(h).
void launch_bluestein_h(int cls, const RingDesc* descs_dev, int n, double2* tabs,
                        cudaStream_t s);
// Cluster class: tabs[h_off..] = FFT_16384(h) (tw_off: e^{-2 pi i k/16384}; tw_half: the
// 8192-point table of the half transforms).
void launch_p2c_h(const RingDesc* descs_dev, int n, double2* tabs, const double2* tw_half, cudaStream_t s);

// Device-side barrier of the fused exchange: worker `rank` publishes `epoch` into every
// worker's flag array (system-scope release) and waits until all workers published it into
// its own (acquire).  flags[w]: address of worker w's n-word flag array, valid on this device.
constexpr int PEER_MAX = 64;
struct PeerFlags {
    unsigned int* f[PEER_MAX];
};
void launch_peer_barrier(const PeerFlags& flags, int rank, int n, unsigned int epoch, cudaStream_t s);

// FP64 peak probe.
void launch_dfma_peak(double* out, int blocks, int threads, int iters, cudaStream_t s);

}  // namespace shtk
