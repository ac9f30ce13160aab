/*
 * vx.h -- C ABI of the B200-native dynamic-M GEMM library (Vortex, arXiv 2409.01075, rebuilt
 * for sm_100a).  Plain C types only: no CUDA, torch or C++ types cross this boundary.
 *
 * The operation (Sec. 4.1; shapes PAPER.md:866-867, Sec. 2.2):
 *     C = A x B,   A: M x K (M = batch x sequence, known only at launch),  B: K x N,  C: M x N
 * and its batched form C_b = A_b x B_b (BASELINE.json config 4).
 *
 * The method (two stages, PAPER.md:1320-1341 overview; DESIGN.md sections 2-3):
 *   vx_plan        offline, sample-free: builds the hierarchical strategy table from
 *                  (N, K, dtypes) and the hardware alone -- Alg. 2 "Candidates Generation"
 *                   over the sm_100a levels
 *                  (tcgen05 instruction -> TMEM accumulator -> SMEM/CTA tile -> grid).
 *   vx_plan_select runtime: integer analytical cost of every (rung, split) for the runtime
 *                  shape, Eqs. 2-4, argmin Eq. 1,
 *                  plus grid configuration.  Host-only, pure.
 *   vx_gemm        runtime: selection + launch of the chosen hand-written sm_100a kernel
 *                  (tcgen05/TMEM/TMA) on the caller's stream.
 *
 * Conventions for every entry point
 *   - Memory: A, B, C are DEVICE pointers owned by the caller (e.g. torch tensors); the
 *     library never copies to the host and allocates device memory only for the stream-K
 *     workspace of a stream, once, on that stream's first stream-K launch (see Thread
 *     safety); vx_plan pre-allocates the legacy stream's.
 *   - Layout: row-major with a contiguous inner dimension.  A is [M,K] (K contiguous).
 *     B is [K,N] (VX_B_KN, the paper's B) or [N,K] (VX_B_NK, an nn.Linear weight / K^T of
 *     attention).  C is [M,N] (N contiguous).  Batched: element (b,i,j) of X lives at
 *     X + b*sX + (row-major offset), strides sX in ELEMENTS.
 *   - Alignment (TMA): 16-bit inputs need K % 8 == 0, 16-byte aligned A and B base
 *     pointers and A/B batch strides that are multiples of 8 elements; B stored K x N
 *     (VX_B_KN) additionally needs N % 8 == 0 (its row stride is N elements).  C needs only
 *     element alignment (rows that are not 16-B aligned are written with scalar stores).
 *     Violations return VX_ERR_ALIGN.  There is no silent fallback and no CPU fallback.
 *   - Streams are passed as `void*` holding a cudaStream_t (NULL = legacy default stream).
 *   - Asynchrony: vx_gemm* enqueue work and return; device faults surface at the caller's
 *     next synchronisation.  Launch errors are returned as VX_ERR_CUDA.
 *   - Errors: every function returns a vx_status; vx_last_error() gives a thread-local
 *     one-line detail for the most recent failure on the calling thread.
 *   - Thread safety: a plan's strategy table is immutable after creation (selections are
 *     memoised in a write-once table) and concurrent vx_gemm calls with the same plan on
 *     different streams are safe: the only mutable device state, the stream-K partial
 *     workspace, is kept per (device, stream) -- allocated on the first stream-K launch on
 *     a stream (inside a capture that allocation runs in relaxed capture mode), reused by
 *     later launches on that stream, which the stream serialises.  Two CUDA graphs
 *     captured on the same stream share that stream's workspace, so they must not be
 *     replayed concurrently.
 *   - Device: a plan from vx_plan(device=d) launches only while d is the calling thread's
 *     current device (VX_ERR_INVALID otherwise).
 */
#ifndef VX_H
#define VX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VX_ABI_VERSION 1

typedef struct vx_plan_s* vx_plan_t; /* opaque, immutable after vx_plan */
typedef struct vx_calib_s* vx_calib_t; /* opaque calibration (empirical tier), immutable once
                                          handed to a plan */

typedef enum { VX_BF16 = 0, VX_FP16 = 1, VX_FP32 = 2 } vx_dtype;

typedef enum {
    VX_B_KN = 0, /* B stored row-major K x N                          */
    VX_B_NK = 1, /* B stored row-major N x K (its transpose: linear weight, K^T of QK^T) */
    VX_B_PACKED = 2 /* B pre-packed by vx_pack_b into contiguous 64 x 64 K-major tiles,
                       [batch][ceil(N/64)][ceil(K/64)][64][64] (zero padded): every TMA box
                       is one 8-KB contiguous block (weights streamed at full DRAM rate) */
} vx_blayout;

typedef enum {
    VX_OK = 0,
    VX_ERR_INVALID = 1,     /* bad argument (NULL, negative size, N/K mismatch with plan) */
    VX_ERR_UNSUPPORTED = 2, /* dtype / layout combination without a kernel               */
    VX_ERR_ALIGN = 3,       /* TMA alignment rule violated (see conventions)             */
    VX_ERR_CUDA = 4,        /* CUDA runtime / driver error (detail in vx_last_error)     */
    VX_ERR_NODEV = 5,       /* no usable sm_100 device                                    */
    VX_ERR_OOM = 6,         /* host allocation failed                                     */
    VX_ERR_BUFFER = 7       /* output buffer too small (vx_plan_dump)                     */
} vx_status;

/* GetHardwareInfo (Table tab:hardware PAPER.md:2343-2351): the level
 * capacities and unit counts that bound the candidate space.  Filled by vx_device_probe
 * from cudaDeviceProp + cudaOccupancyMaxActiveClusters, or supplied by the caller to
 * vx_plan_ex (e.g. a descriptor captured once on a B200, for host-only planning). */
typedef struct {
    int32_t sm_count;              /* |HardwareUnit| at grid level (148 on B200)         */
    int32_t smem_optin;            /* max dynamic shared memory per CTA, bytes           */
    int32_t smem_per_sm;           /* shared memory per SM, bytes                         */
    int32_t max_threads_per_block; /* 1024                                */
    int32_t max_threads_per_sm;
    int32_t tmem_cols;             /* tensor-memory columns per SM (512)                  */
    int32_t cc_major, cc_minor;
    int32_t clock_khz;
    int32_t max_active_clusters[4];/* resident clusters of size 1, 2, 4, 8 (full-SMEM CTAs) */
    int64_t l2_bytes;
} vx_device_desc;

/* One runtime decision ("SchedulePlan"): the rung (a full chain of the
 * strategy table), the split of the reduction loop, and the launch geometry. */
typedef struct {
    int32_t rung_id;  /* index into the plan's strategy table (vx_plan_dump order)          */
    int32_t split;    /* K-loop schedule: 1 = persistent CTAs over whole-K tiles; s > 1 =
                         split-K over a cluster of s CTAs reducing through DSMEM; 0 =
                         stream-K over (tile, k-block) units (R19)                          */
    int32_t family;   /* 0 tcgen05, 1 tcgen05 with A/B swapped, 2 fp32 SIMT, 3 CUDA-core
                         GEMV (adaptive backend, R20)                                       */
    int32_t swap;
    int32_t bm, bn;   /* CTA tile on the (UMMA-M, UMMA-N) axes                              */
    int32_t stages;   /* shared-memory pipeline depth                                      */
    int32_t tiles_m;  /* tiles along the UMMA-M axis (M, or N when swapped)                */
    int32_t tiles_n;  /* tiles along the UMMA-N axis                                        */
    int32_t grid;     /* CTAs launched                                                      */
    int32_t cluster;  /* CTAs per cluster: split s (DSMEM split-K), 2 (cta_group::2 pair),
                         mc (TMA-multicast cluster) or 1                                    */
    int32_t mc;       /* TMA-multicast cluster size sharing the A tile (1 = no multicast)   */
    int64_t cost;     /* predicted cycles, Eq. 4 (integer)                   */
} vx_choice;

/* Library version (VX_ABI_VERSION) -- lets the binding reject a stale .so. */
int32_t vx_abi_version(void);

/* Human-readable name of a status code; never NULL. */
const char* vx_status_str(vx_status s);

/* Thread-local detail of the last failure on this thread ("" if none); never NULL. */
const char* vx_last_error(void);

/* Fill *out for CUDA device `device` (must be sm_100).  VX_ERR_NODEV if absent. */
vx_status vx_device_probe(int device, vx_device_desc* out);

/* Offline stage: build the strategy table for C[M,N] = A[M,K] x B for every M.
 *   N   > 0: static N (linear layer); N == 0: N dynamic too (batched attention scores),
 *            given per call.
 *   K   > 0 (16-bit inputs: K % 8 == 0).
 *   in  : VX_BF16 / VX_FP16 (tensor cores, fp32 accumulation) or VX_FP32 (CUDA cores).
 *   out : output element type (VX_BF16 / VX_FP16 / VX_FP32; fp32 inputs need fp32 out).
 *   bl  : layout of B.
 *   device: CUDA device whose descriptor is probed (vx_device_probe).
 * On success *plan owns host memory only; free with vx_plan_destroy. */
vx_status vx_plan(int64_t N, int64_t K, vx_dtype in, vx_dtype out, vx_blayout bl, int device,
                  vx_plan_t* plan);

/* Same, with an explicit descriptor (copied); no CUDA call is made, so this works on a
 * host without a GPU (used by the selector-parity tests).  Such a plan can still launch
 * if the process later runs on a matching device. */
vx_status vx_plan_ex(int64_t N, int64_t K, vx_dtype in, vx_dtype out, vx_blayout bl,
                     const vx_device_desc* desc, vx_plan_t* plan);

vx_status vx_plan_destroy(vx_plan_t plan);

/* ---- the empirical tier of the hybrid analyzer (Sec. 5.2) ----------
 * Every plan prices its rungs with per-rung constants (mac / l2s / epi rates in bytes or
 * MACs per SM cycle x1000, fixed cycles) plus chip constants.  By default
 * they are the compiled-in table, measured offline on a B200 (vx_calib.cpp).  These entry
 * points let a caller measure them LIVE on its device and freeze them into plans. */

/* Profile every 16-bit tcgen05 / CUDA-core rung and schedule on `device` over a fixed
 * generic grid of shapes (never a workload shape), fit the per-rung constants of the same
 * integer Eqs. 2-4 vx_plan_select evaluates, and return them with the compiled-in chip
 * constants.  bl: layout of B the timings use (VX_B_KN or VX_B_NK).
 * effort 0: 4 (N,K) x 7 M (seconds); 1: 7 (N,K) x 14 M.  Allocates ~768 MB of device
 * memory for the duration of the call; synchronises the device.  Free with
 * vx_calib_destroy. */
vx_status vx_calibrate(int device, vx_blayout bl, int32_t effort, vx_calib_t* out);

/* A calibration from explicit values (e.g. a JSON table): chip constants, then one
 * vx_calib_set_rung per rung key ("umma_128x128", "umma_swap_mc2_128x64", "gemv_4x8", ...;
 * the keys vx_plan_dump reports through its rung fields). */
vx_status vx_calib_new(int64_t hbm_milli, int64_t dsm_milli, int64_t fixed_cluster,
                       int64_t skfix_milli, int64_t stagger, vx_calib_t* out);
vx_status vx_calib_set_rung(vx_calib_t calib, const char* key, int64_t mac_milli,
                            int64_t l2s_milli, int64_t epi_milli, int64_t fixed);
vx_status vx_calib_destroy(vx_calib_t calib);

/* Canonical JSON of a calibration ({"source", chip constants, "rungs": {key: {...}}});
 * calib NULL = the compiled-in table.  Same buffer protocol as vx_plan_dump. */
vx_status vx_calib_dump(vx_calib_t calib, char* buf, size_t cap, size_t* need);

/* vx_plan / vx_plan_ex with the given calibration (copied: the plan owns its copy, the
 * calibration may be destroyed afterwards).  A rung whose key the calibration lacks makes
 * the call fail with VX_ERR_UNSUPPORTED. */
vx_status vx_plan_calibrated(int64_t N, int64_t K, vx_dtype in, vx_dtype out, vx_blayout bl,
                             int device, vx_calib_t calib, vx_plan_t* plan);
vx_status vx_plan_ex_calibrated(int64_t N, int64_t K, vx_dtype in, vx_dtype out, vx_blayout bl,
                                const vx_device_desc* desc, vx_calib_t calib, vx_plan_t* plan);

/* Runtime selection only (host, pure, deterministic): argmin of Eq. 4 cost over the
 * plan's (rung, split) pairs for (batch, M, N).  N must equal the plan's N when static
 * (pass it anyway).  batch >= 1, M >= 1, N >= 1. */
vx_status vx_plan_select(vx_plan_t plan, int64_t batch, int64_t M, int64_t N, vx_choice* out);

/* Runtime selection for a ragged batch (host, pure): the decision vx_gemm_varlen makes for
 * sequence offsets cu[0..ngroups] (cu[0] = 0, non-decreasing). */
vx_status vx_plan_select_varlen(vx_plan_t plan, int32_t ngroups, const int32_t* cu,
                                vx_choice* out);

/* Cost of one forced (rung, split) for the shape (same model vx_plan_select minimises);
 * VX_ERR_INVALID if the pair is not in the table. */
vx_status vx_plan_cost(vx_plan_t plan, int32_t rung_id, int32_t split, int64_t batch,
                       int64_t M, int64_t N, vx_choice* out);

/* Canonical JSON of the strategy table (levels' candidate counts, rungs, calibration
 * constants).  Writes at most cap bytes including the NUL; *need = required size.
 * VX_ERR_BUFFER if cap is too small (buf may be NULL with cap 0 to query). */
vx_status vx_plan_dump(vx_plan_t plan, char* buf, size_t cap, size_t* need);

/* Runtime stage: C = A x B for M rows (M == 0 is a no-op returning VX_OK).
 * N and K must equal the plan's (N only checked when static). */
vx_status vx_gemm(vx_plan_t plan, int64_t M, int64_t N, int64_t K, const void* A,
                  const void* B, void* C, void* stream);

/* Batched: C_b = A_b x B_b for b < batch with element strides sA, sB, sC. */
vx_status vx_gemm_batched(vx_plan_t plan, int64_t batch, int64_t M, int64_t N, int64_t K,
                          const void* A, int64_t sA, const void* B, int64_t sB, void* C,
                          int64_t sC, void* stream);

/* Full-control form used by tests and the regret sweep: force_rung < 0 selects with the
 * cost model; otherwise (force_rung, force_split) must be a pair of the table.  If `used`
 * is non-NULL it receives the launched decision.  Otherwise identical to vx_gemm_batched. */
vx_status vx_gemm_ex(vx_plan_t plan, int64_t batch, int64_t M, int64_t N, int64_t K,
                     const void* A, int64_t sA, const void* B, int64_t sB, void* C, int64_t sC,
                     int32_t force_rung, int32_t force_split, void* stream, vx_choice* used);

/* Fused GEMM + row all-gather (BASELINE.json configs[4] "optional NCCL
 * all-gather of C", PAPER.md:866-867 row independence): computes this rank's C_local =
 * A x B (M rows, batch 1) and writes it -- tile by tile, straight from the GEMM epilogue, so
 * the transfer of finished tiles overlaps the mainloop of later ones -- into rows
 * [row_offset, row_offset + M) of EVERY destination dst[0..ndst), 1 <= ndst <= 8.  Each
 * destination is a row-major [*, N] matrix of the plan's output dtype with at least
 * row_offset + M rows: typically every rank's gathered C, mapped into this process (NVLink
 * peer or symmetric-memory pointers, paper_2409_01075_b200/dist.py), this rank's own
 * included.  No C is written besides the destinations.  Candidates are the non-swapped
 * tcgen05 rungs with split 1 or stream-K (force_rung < 0 selects among them with the cost
 * model; a forced pair outside that set is VX_ERR_INVALID).  Synchronisation with the
 * readers (e.g. a barrier after the stream completes) is the caller's.  `used` (optional)
 * receives the launched decision. */
vx_status vx_gemm_gather(vx_plan_t plan, int64_t M, int64_t N, int64_t K, const void* A,
                         const void* B, int32_t ndst, void* const* dst, int64_t row_offset,
                         int32_t force_rung, int32_t force_split, void* stream, vx_choice* used);

/* Ragged attention batch (the varlen reading of BASELINE config 4):
 * S_g = Q_g x K_g^T for g < ngroups sequences of lengths s_g = cu[g+1] - cu[g], in ONE
 * launch.  Q and Kt are packed row-major [cu[ngroups], K] (sequence g in rows [cu[g],
 * cu[g+1])), Kt being K stored N x K; S is packed: S_g is s_g x s_g row-major at element
 * offset sum_{j<g} s_j^2.  The plan must have N = 0 (dynamic), 16-bit inputs and
 * VX_B_NK.  cu_host is read on the host (selection: Eqs. 2-4 over the ragged tile set,
 * grid); cu_dev (same ngroups + 1 int32 values, device) is read by the kernel.
 * force_rung < 0 selects; used (optional) receives the decision (tiles_m = tiles_n = 0). */
vx_status vx_gemm_varlen(vx_plan_t plan, int32_t ngroups, const int32_t* cu_host,
                         const int32_t* cu_dev, int64_t K, const void* Q, const void* Kt, void* S,
                         int32_t force_rung, void* stream, vx_choice* used);

/* Host-staged form (the e2e measurement): A, B, C are HOST pointers (pinned for full
 * speed); dA, dB, dC are caller-owned device buffers of the same sizes.  Enqueues
 * H2D(A,B) -> vx_gemm_batched -> D2H(C) on `stream` and returns without synchronising. */
vx_status vx_gemm_host(vx_plan_t plan, int64_t batch, int64_t M, int64_t N, int64_t K,
                       const void* A, const void* B, void* C, void* dA, void* dB, void* dC,
                       void* stream);

/* Elements (of the plan's input dtype) of a packed B for (batch, N, K): batch x
 * ceil(N/64)*64 x ceil(K/64)*64.  0 on bad arguments. */
int64_t vx_packed_b_elems(vx_plan_t plan, int64_t batch, int64_t N, int64_t K);

/* Pack B (device, stored in layout `src_layout` = VX_B_KN or VX_B_NK, batch stride sB
 * elements) into the VX_B_PACKED layout at Bp (device, vx_packed_b_elems elements, 16-B
 * aligned).  One kernel launch on `stream`; the plan must have b_layout VX_B_PACKED and a
 * 16-bit input dtype.  Packing is a one-time cost per weight (inference weights are
 * constant); vx_gemm on a VX_B_PACKED plan then takes Bp as its B. */
vx_status vx_pack_b(vx_plan_t plan, int64_t batch, int64_t N, int64_t K, vx_blayout src_layout,
                    const void* B, int64_t sB, void* Bp, void* stream);

/* Number of kernel launches this process has issued through the library (evidence for
 * bench.py's gpu_launches). */
int64_t vx_launch_count(void);

/* Tensor-map memo statistics (process-wide): encodes served from the memo / encoded anew.
 * vx_gemm* encodes a CUtensorMap per operand; one with the same address, shape and box as a
 * recent one (typically B, the weights) is reused instead of re-encoded.
 * Either pointer may be NULL. */
void vx_map_cache_stats(int64_t* hits, int64_t* misses);

#ifdef __cplusplus
}
#endif
#endif /* VX_H */
