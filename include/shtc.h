/*
 * shtc.h — C ABI of the B200-native spherical harmonic transform (sm_100a, FP64).
 *
 * This is the drop-in boundary for the reference's accelerated path.
 * Plain C types only: pointers, sizes, status codes.  Complex values are interleaved
 * (re, im) float64 pairs.  a_lm use the reference AlmSet m-major triangle
 * (offset(m) = m(lmax+1) - m(m-1)/2, alm.hpp:27-31); maps are ring-ordered pixels
 * (alm.hpp:39-42); Delta panels are ring-major [ring][m] (alm.hpp:49-64).
 *
 * Reference interfaces each entry point replaces (file:line in /root/reference/proj):
 *   shtc_alm2map / shtc_alm2map_dev   sht::synthesis              include/sht/transforms.hpp:73-74
 *   shtc_map2alm / shtc_map2alm_dev   sht::analysis               include/sht/transforms.hpp:78-79
 *   shtc_delta_a                      sht::compute_delta_a         include/sht/transforms.hpp:32-35
 *                                     (and compute_delta_a_ring_major :40-43, same numbers)
 *   shtc_accumulate_alm               sht::accumulate_alm /        include/sht/transforms.hpp:48-51
 *                                     accumulate_alm_partial        include/sht/transforms.hpp:61-64
 *   shtc_legendre_alm2map_dev         detail::delta_a_columns_paired  transforms.hpp:116-119
 *   shtc_legendre_map2alm_dev         detail::accumulate_columns_paired transforms.hpp:121-124
 *   shtc_ring_synthesis_dev           ring_synthesis_into (per ring)  include/sht/fourier.hpp:22-23
 *   shtc_ring_analysis_dev            ring_analysis_into  (per ring)  include/sht/fourier.hpp:28-29
 *   shtc_set_exchange_layout + the two stage calls above
 *                                     distributed_synthesis / distributed_analysis stages
 *                                     (distribution.cpp:300-490); the panel transpose
 *                                     exchange_m_to_rings/rings_to_m (distribution.hpp:52-57)
 *                                     becomes either the caller's NCCL all-to-all on the
 *                                     packed buffers these calls read and write, or the
 *                                     fused peer-memory path (shtc_*_peer + shtc_peer_barrier).
 *
 * Error behaviour mirrors the reference: argument/layout violations -> SHTC_EINVAL
 * (std::invalid_argument), beta_lm(l==m) style domain errors -> SHTC_EDOMAIN
 * (std::domain_error); CUDA failures -> SHTC_ECUDA.  shtc_last_error() returns the message.
 * There is no CPU fallback: without a usable sm_100 device every compute call fails.
 */
#ifndef SHTC_H
#define SHTC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct shtc_ctx shtc_ctx;

typedef enum {
    SHTC_OK = 0,
    SHTC_EINVAL = 1,       /* std::invalid_argument in the reference */
    SHTC_EDOMAIN = 2,      /* std::domain_error in the reference */
    SHTC_ECUDA = 3,        /* CUDA runtime / driver failure, no device */
    SHTC_ENOMEM = 4,       /* device allocation failed */
    SHTC_EUNSUPPORTED = 5  /* configuration outside what the kernels implement */
} shtc_status;

/* Per-call timing, CUDA events on the context stream (ms), plus side channels that the
 * reference keeps in TransformOptions::step_counter / Profiler (perfmodel.hpp:63-84). */
typedef struct {
    double legendre_ms;     /* Legendre stage kernel time (host-buffer paths: sum over the
                               pipelined launches, which overlap each other and the copies) */
    double fft_ms;          /* fold + ring FFT + unfold kernel time (same convention) */
    double h2d_ms;          /* host->device copy span (host-buffer entry points only) */
    double d2h_ms;          /* device->host copies from the first copy's start to the end of
                               the call (host-buffer entry points only) */
    double total_ms;        /* whole call on the stream */
    uint64_t nominal_steps; /* reference step count: sum over streams of lmax-m+1 */
    uint64_t executed_steps;/* (l, m, stream) steps the kernels actually ran */
} shtc_timing;

/* ---- context ------------------------------------------------------------------------- */
shtc_status shtc_create(int device, shtc_ctx** out);
void shtc_destroy(shtc_ctx* ctx);
const char* shtc_last_error(const shtc_ctx* ctx); /* ctx may be NULL (last global error) */
/* Kernel launches issued by the library so far (process-wide counter; a caller brackets a
 * region with two reads to state how many of the library's kernels ran in it). */
uint64_t shtc_kernel_launches(void);
int shtc_device_count(void);
/* Use an external CUDA stream (cudaStream_t passed as void*; NULL = the context's own). */
shtc_status shtc_set_stream(shtc_ctx* ctx, void* cuda_stream);

/* ---- geometry and band (reference PixelGrid / AlmSet, grid.hpp:13-37, alm.hpp:16-35) --- */
/* Copies the ring arrays.  mirror != 0 requests north/south stream pairing
 * (PairPolicy::mirror, transforms.hpp:19-20); it is honoured only for grids that are
 * mirror symmetric (symmetric_ring_pairs, grid.cpp:133-151), else rings run unpaired. */
shtc_status shtc_set_grid(shtc_ctx* ctx, int n_rings, const double* cos_theta,
                          const int32_t* n_phi, const double* phi_0, const double* weight,
                          const int64_t* pixel_offset, int mirror);
/* Band limits and the orders this context owns (NULL / n_m<=0 = all of 0..mmax).  The
 * owned set is the worker's M_i of assign_m (distribution.cpp:82-99) for multi-GPU runs. */
shtc_status shtc_set_band(shtc_ctx* ctx, int lmax, int mmax, int n_m, const int32_t* ms);
/* Rescaling ladder of the recurrence (ScaleLadder, legendre.hpp:26-47): enabled != 0 is
 * ScaleLadder::standard() (the default, the 2^+-512 window), 0 is ScaleLadder::unscaled()
 * (thresholds never trip: a stream whose seed lies below the window never counts).  Applies to
 * the plans built afterwards (whole transforms and the Legendre-stage operators). */
shtc_status shtc_set_ladder(shtc_ctx* ctx, int enabled);
/* Builds (and caches) the Legendre plan (recurrence tables, underflow activation scan)
 * and the ring-FFT plan; otherwise built lazily by the first transform. */
shtc_status shtc_plan(shtc_ctx* ctx, double* plan_ms);
/* Exact pair-step accounting of the plan: nominal, executed (map2alm, after dead-tile
 * skipping; its passes run tile pairs from the earlier start), useful (steps whose term the
 * reference keeps, i.e. ladder scale k == 0). */
shtc_status shtc_plan_stats(shtc_ctx* ctx, uint64_t* nominal, uint64_t* executed,
                            uint64_t* useful);
/* Executed pair-steps split by kernel phase: before the tile's first activation (recurrence +
 * ladder check only), inside the activation window (checked), after it (unchecked). */
shtc_status shtc_plan_phase_stats(shtc_ctx* ctx, uint64_t* prefix, uint64_t* checked,
                                  uint64_t* fast);
/* Executed pair-steps per transform: alm2map (single-tile items) and map2alm (tile pairs). */
shtc_status shtc_plan_executed(shtc_ctx* ctx, uint64_t* alm2map, uint64_t* map2alm);

/* ---- whole transforms ---------------------------------------------------------------- */
/* alm: 2*AlmSet::count(lmax,mmax) doubles; map: n_pix doubles.  Host buffers: the copies are
 * pipelined against the kernels over latitude bands.  Page-locked buffers (cudaHostAlloc,
 * cudaHostRegister, pinned tensors) are copied directly; pageable ones (std::vector, numpy) go
 * through page-locked staging buffers the context keeps, copied on all host cores.  Returns when
 * the output is in place. */
shtc_status shtc_alm2map(shtc_ctx* ctx, const double* alm, double* map, shtc_timing* t);
shtc_status shtc_map2alm(shtc_ctx* ctx, const double* map, double* alm, shtc_timing* t);
/* Same, device-resident buffers (no host copies). */
shtc_status shtc_alm2map_dev(shtc_ctx* ctx, const double* alm_dev, double* map_dev,
                             shtc_timing* t);
shtc_status shtc_map2alm_dev(shtc_ctx* ctx, const double* map_dev, double* alm_dev,
                             shtc_timing* t);

/* ---- stages (multi-GPU building blocks; device buffers) ------------------------------ */
/* Exchange layout of one worker (distributed_synthesis, distribution.cpp:300-380).
 *   delta rows: the owned orders' panel is written ring-row by ring-row; row_off[r] is the
 *     complex-element offset of ring r's row (n_cols = owned orders per row).  Grouping the
 *     rows of each destination worker contiguously makes the Legendre output the NCCL send
 *     buffer of exchange_m_to_rings without a pack kernel.
 *   ring side: the rings this worker transforms (ring_list, ascending) and, per order m of
 *     0..mmax, where Delta(ring_list[p], m) lives: m_base[m] + p * m_stride[m]
 *     (complex elements) — the receive buffer of the all-to-all, unpacked in the fold.
 * Passing NULL restores the single-GPU identity layout. */
shtc_status shtc_set_exchange_layout(shtc_ctx* ctx, const int64_t* row_off, int n_ring_list,
                                     const int32_t* ring_list, const int64_t* m_base,
                                     const int64_t* m_stride);
/* Synthesis-direction layout on top of shtc_set_exchange_layout (same blocks, same ring list):
 * Delta(r, order index mi) of the Legendre output at row_off[r] + mi * row_stride[r] and the
 * ring synthesis input (ring_list[p], m) at m_base[m] + p * m_stride[m].  Order-major blocks
 * ([|M_i| orders x |R_j| rings], row_stride = |R_j|) turn the Legendre kernel's stores --
 * one order, consecutive rings per warp -- into contiguous runs (the NVLink stores of the
 * fused exchange).  The analysis direction keeps the ring-major layout, whose unfold visits
 * the orders grouped by m_base so each owner's block is stored contiguously.  NULL row_off:
 * both directions use the shtc_set_exchange_layout layout.  Clears the peer targets. */
shtc_status shtc_set_exchange_layout_synthesis(shtc_ctx* ctx, const int64_t* row_off,
                                               const int64_t* row_stride, const int64_t* m_base,
                                               const int64_t* m_stride);
shtc_status shtc_legendre_alm2map_dev(shtc_ctx* ctx, const double* alm_dev, double* delta_dev,
                                      shtc_timing* t);
shtc_status shtc_legendre_map2alm_dev(shtc_ctx* ctx, const double* delta_dev, double* alm_dev,
                                      shtc_timing* t);
shtc_status shtc_ring_synthesis_dev(shtc_ctx* ctx, const double* delta_dev, double* map_dev,
                                    shtc_timing* t);
shtc_status shtc_ring_analysis_dev(shtc_ctx* ctx, const double* map_dev, double* delta_dev,
                                   shtc_timing* t);

/* ---- fused exchange over peer memory (multi-GPU, one process per GPU) ----------------- */
/* exchange_m_to_rings / exchange_rings_to_m (distribution.cpp:233-298) without a collective:
 * the producing stage kernel stores each Delta entry straight into the consumer's buffer
 * (NVLink peer memory, mapped through CUDA IPC), then every worker passes one device-side
 * barrier.  Buffers that other processes map must be allocated with shtc_dev_alloc (an IPC
 * handle covers an allocation from its base).  Zero-filled. */
shtc_status shtc_dev_alloc(int device, uint64_t bytes, void** ptr);
shtc_status shtc_dev_free(void* ptr);
shtc_status shtc_ipc_handle(const void* ptr, unsigned char* handle64);      /* 64 bytes */
shtc_status shtc_ipc_open(int device, const unsigned char* handle64, void** ptr);
shtc_status shtc_ipc_close(void* ptr);
/* Targets of this worker's stores (device addresses valid on this context's device), on top
 * of shtc_set_exchange_layout:
 *   row_ptr[r] (n_rings): ring r's element of this worker's first order in the ring owner's
 *     receive buffer, further orders row_stride[r] apart (1 without a synthesis layout)
 *     (alm2map); col_ptr[m] (mmax+1): order m's column for this worker's first ring in the
 *     order owner's send buffer, rows m_stride[m] apart (map2alm).
 * NULL clears them. */
shtc_status shtc_set_exchange_peers(shtc_ctx* ctx, const uint64_t* row_ptr, const uint64_t* col_ptr);
/* Legendre stage writing Delta through row_ptr; ring analysis writing Delta^S through col_ptr. */
shtc_status shtc_legendre_alm2map_peer(shtc_ctx* ctx, const double* alm_dev, shtc_timing* t);
shtc_status shtc_ring_analysis_peer(shtc_ctx* ctx, const double* map_dev, shtc_timing* t);
/* Device-side barrier on the context stream: flags[w] = address of worker w's n_workers-word
 * uint32 flag array (zeroed at allocation); epoch must increase by one per barrier.
 * Ordering contract: a peer-store stage writes into buffers another worker's consumer stage of
 * the PREVIOUS call of the same direction may still read.  alm2map and map2alm calls that
 * alternate are ordered by the other direction's barrier; when a direction repeats, every
 * worker passes one extra barrier before its peer stores (sht.PeerExchange does this). */
shtc_status shtc_peer_barrier(shtc_ctx* ctx, int rank, int n_workers, const uint64_t* flags,
                              uint32_t epoch);
/* Host <-> device copy of this context's orders (the set_band order set) between two full
 * m-major a_lm triangles (2*AlmSet::count(lmax,mmax) doubles each): the a_lm share a worker
 * of an m-distributed run reads (to_device != 0) or returns.  One async copy per order on the
 * context stream; page-locked host memory for overlap. */
shtc_status shtc_copy_orders(shtc_ctx* ctx, const double* src, double* dst, int to_device);

/* Page-locked host memory (cudaHostAlloc, portable): buffers the copy engines read and write
 * directly, e.g. the C++ drop-in's result buffers.  shtc_host_free(NULL) is a no-op. */
shtc_status shtc_host_alloc(size_t bytes, void** out);
void shtc_host_free(void* p);

/* ---- single-process multi-GPU group -------------------------------------------------- */
/* distributed_synthesis / distributed_analysis (distribution.cpp:300-490; distribution.hpp:
 * 70-77) as one process driving W device contexts, worker i on device_ids[i] (NULL: device
 * i mod device count; workers may share a device).  Orders and rings are owned per worker
 * (m_owner[m], ring_owner[r]: a partition, e.g. from assign_m / assign_rings,
 * distribution.cpp:82-124); every worker must own at least one order and one ring.
 * Exchange of the Delta panel between the stages (exchange_m_to_rings / rings_to_m,
 * distribution.cpp:233-298):
 *   SHTC_EXCHANGE_PEER  fused: the producing stage kernel stores each entry straight into the
 *                       consumer's buffer (NVLink peer memory; plain stores on a shared device),
 *                       consumers wait on the producers' completion events;
 *   SHTC_EXCHANGE_NCCL  ncclCommInitAll + grouped ncclSend/ncclRecv on the packed buffers
 *                       (libnccl dlopen'ed on first use; needs one distinct device per worker).
 * Results equal the single-context transforms.  Calls are synchronous (return with the output
 * in place). */
typedef struct shtc_group shtc_group;
enum { SHTC_EXCHANGE_PEER = 0, SHTC_EXCHANGE_NCCL = 1 };
typedef struct {
    double legendre_ms;      /* stage maxima over the workers (CUDA events per worker) */
    double fft_ms;
    double exchange_ms;      /* end of the producer stage -> start of the consumer stage */
    double h2d_ms;
    double d2h_ms;
    double total_ms;         /* wall clock of the whole call */
    uint64_t exchange_bytes; /* Delta bytes moved between distinct workers */
    uint64_t nominal_steps;  /* reference step count summed over the workers */
} shtc_group_timing;
shtc_status shtc_group_create(int n_workers, const int32_t* device_ids, int exchange_mode,
                              shtc_group** out);
void shtc_group_destroy(shtc_group* g);
const char* shtc_group_last_error(const shtc_group* g); /* g may be NULL */
shtc_status shtc_group_device(const shtc_group* g, int worker, int* device);
shtc_status shtc_group_set_grid(shtc_group* g, int n_rings, const double* cos_theta,
                                const int32_t* n_phi, const double* phi_0, const double* weight,
                                const int64_t* pixel_offset, int mirror);
/* Band limits + ownership; builds every worker's plans and exchange buffers. */
shtc_status shtc_group_set_layout(shtc_group* g, int lmax, int mmax, const int32_t* m_owner,
                                  const int32_t* ring_owner);
shtc_status shtc_group_plan_ms(const shtc_group* g, double* plan_ms);
/* Host buffers (pageable or page-locked), the whole a_lm triangle / map. */
shtc_status shtc_group_alm2map(shtc_group* g, const double* alm, double* map, shtc_group_timing* t);
shtc_status shtc_group_map2alm(shtc_group* g, const double* map, double* alm, shtc_group_timing* t);
/* Device buffers, one per worker on its device: a full a_lm triangle / full map each (a worker
 * reads and writes only its own orders / rings). */
shtc_status shtc_group_alm2map_dev(shtc_group* g, const uint64_t* alm_dev, const uint64_t* map_dev,
                                   shtc_group_timing* t);
shtc_status shtc_group_map2alm_dev(shtc_group* g, const uint64_t* map_dev, const uint64_t* alm_dev,
                                   shtc_group_timing* t);

/* ---- Legendre-stage operators (transforms.cpp:269-365), host buffers ------------------ */
/* Delta^A_m(r) for the given latitudes and orders; delta: n_lat x n_m complex, ring-major.
 * ms must be ascending and unique (the reference sorts, checked_m_set transforms.cpp:224). */
shtc_status shtc_delta_a(shtc_ctx* ctx, const double* alm, int lmax, int mmax, int n_lat,
                         const double* x, int n_m, const int32_t* ms, double* delta,
                         uint64_t* steps);
/* a_lm += sum_r Delta^S_m(r) P_lm(x_r) for the orders in ms (others untouched). */
shtc_status shtc_accumulate_alm(shtc_ctx* ctx, const double* delta, int n_lat,
                                const double* x, int n_m, const int32_t* ms, int lmax,
                                int mmax, double* alm_inout, uint64_t* steps);

/* ---- device helpers ------------------------------------------------------------------ */
shtc_status shtc_device_info(int device, char* name, int name_len, int* sm_count,
                             int* cc_major, int* cc_minor);
/* Measured FP64 DFMA peak of the device (TFLOP/s), from a resident-loop kernel. */
shtc_status shtc_measure_fp64_peak(int device, double* tflops, double* sm_clock_mhz);

#ifdef __cplusplus
}
#endif
#endif /* SHTC_H */
