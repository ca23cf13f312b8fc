/* ===========================================================================
 * hps_leaf_gpu.h — C-ABI of the B200 HPS leaf stage (libhps_leaf_b200.so).
 *
 * The reference (arXiv 2211.14969, /root/reference) specifies the leaf stage as
 * C++ operations in namespace hps with exceptions
 * from proj/include/hps/errors.hpp and batching from proj/include/hps/parallel.hpp.
 * It has no compiled implementation, so this C-ABI is the boundary its own FFI
 * would bind for the path; each entry point names the reference operation it
 * replaces.  include/hps/leaf_gpu.hpp is the SPEC-shaped C++ layer over it.
 *
 * Conventions
 *   - No exceptions cross this boundary.  Return codes:
 *       HPS_OK 0, HPS_ERR_RESONANCE 1 (see status[]), HPS_ERR_PARAM 2,
 *       HPS_ERR_CUDA 3.  hps_gpu_last_error(ctx) returns the message.
 *   - Ownership: the library owns device memory and streams; the caller owns
 *     every host buffer (pinned memory from hps_host_alloc gives full overlap;
 *     pageable T/w outputs of hps_gpu_condense are staged through library-owned
 *     pinned double buffers, status[] always is).
 *   - Threading: one ctx per GPU, driven by one host thread; calls on distinct
 *     ctxs are concurrent-safe; one ctx is not reentrant (parallel.hpp's
 *     per-worker scratch rule).
 *   - Layouts (leaf-major, element e = ey*nx + ex; local node l = iy*p + ix;
 *     boundary order S,E,N,W with corners owned by the first listing edge,
 *     SPEC.md:314):  b, f, u : p*p per leaf ; T : n_b*n_b row-major per leaf ;
 *     w, v : n_b per leaf ; S_solve : n_i*n_b row-major per leaf.
 *     n_i = (p-2)^2, n_b = 4(p-1).
 *   - Results are bitwise-independent of chunking, leaf range and GPU count
 *     (parallel.hpp:21-22).
 * =========================================================================== */
#ifndef HPS_LEAF_GPU_H
#define HPS_LEAF_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_OK 0
#define HPS_ERR_RESONANCE 1
#define HPS_ERR_PARAM 2
#define HPS_ERR_CUDA 3

/* SPEC.md:313 storage policy for leaf factors (recompute vs store):
 *   RECOMPUTE  leaf_solve rebuilds and refactors A_ii (default; nothing kept);
 *   STORE      the LU factors of the condensed range stay in HBM (25.7 MB/leaf at p=42, so the
 *              whole range must fit one device chunk); leaf_solve re-solves with its f;
 *   S_SOLVE    condense also back-substitutes [S_solve | A_ii^{-1} f_i] (K3, +~12% condense
 *              time) and keeps it for every leaf (n_i (n_b+1) doubles: 2.1 MB/leaf at p=42,
 *              20 GB at C4); leaf_solve is then one HBM-bound GEMV per leaf (K5s), using the
 *              load f_i of the condense call (its b, f arguments are not read). */
#define HPS_STORAGE_RECOMPUTE 0
#define HPS_STORAGE_STORE 1
#define HPS_STORAGE_S_SOLVE 2

typedef struct hps_gpu_ctx hps_gpu_ctx;

/* Leaf-stage descriptor: the (p, a, kappa) of build_leaf_operator
 * (SPEC.md:270-273, 62-70), the element grid of MeshParams,
 * the storage policy and the device budget for in-flight leaves. */
typedef struct {
  int32_t p;               /* nodes per leaf side, 4 <= p <= 45 */
  int32_t nx, ny;          /* leaf grid (elements) */
  int32_t storage;         /* HPS_STORAGE_RECOMPUTE (default), _STORE or _S_SOLVE */
  double a;                /* leaf side length, > 0 */
  double kappa;            /* wavenumber, >= 0 */
  int64_t workspace_bytes; /* 0: 70% of free device memory */
} hps_leaf_desc;

typedef struct {
  int32_t p, n_i, n_b, n_leaves;
  int32_t chunk_leaves;    /* leaves per device chunk */
  int32_t resident_ctas;   /* leaves in flight per wave (2 per SM) */
  int64_t workspace_bytes_per_leaf;
  int64_t n_active;        /* reduced-system unknowns */
  int64_t N;               /* global DOF */
} hps_gpu_info_t;

/* Device-side timing (CUDA events on the launching stream). */
typedef struct {
  float ms_total;          /* first kernel start -> last kernel end */
  float ms_assemble;       /* K1, summed over chunks */
  float ms_lu_schur;       /* K2+K3, summed over chunks */
  float ms_scatter;        /* K4 */
  int32_t kernels;         /* kernels launched by the call */
  int32_t chunks;
} hps_gpu_timing_t;

/* Create a context on `device` (hps_gpu_ctx holds streams, tables, workspace). */
int hps_gpu_create(int device, const hps_leaf_desc* desc, hps_gpu_ctx** out);
void hps_gpu_destroy(hps_gpu_ctx* ctx);
const char* hps_gpu_last_error(const hps_gpu_ctx* ctx);
int hps_gpu_get_info(const hps_gpu_ctx* ctx, hps_gpu_info_t* out);
/* Device time of the kernels enqueued since the last reset (host-buffer calls
 * reset on entry; device-resident calls accumulate).  Synchronizes on the last
 * recorded event. */
int hps_gpu_get_timing(hps_gpu_ctx* ctx, hps_gpu_timing_t* out);
int hps_gpu_reset_timing(hps_gpu_ctx* ctx);

/* batched_condense (per leaf condense_leaf :279-287) for
 * elements [e0, e1).  Inputs b, f are the (e1-e0) leaves' samples (host).
 * Outputs (host, caller-owned): T (T_flux), w (w_equiv), S (S_solve, nullable: when
 * given, K3 back-substitutes -A_ii^{-1} A_ib from the factors, n_i x n_b per leaf),
 * status (0 ok / 1 resonance).  Returns HPS_ERR_RESONANCE if any leaf failed;
 * the message names the smallest failing element id and all failing ids. */
int hps_gpu_condense(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* b, const double* f,
                     double* T, double* w, double* S, int32_t* status);

/* batched_condense + assemble_reduced of the whole mesh with the
 * leaves' T/w kept resident in HBM: b, f are all n_leaves leaves' samples (host), g_bnd the
 * Dirichlet samples (layout of hps_gpu_assemble_reduced); the host receives the CSR values
 * (pattern: hps_gpu_reduced_pattern) and rhs, bit-identical to condense + assemble_reduced,
 * plus T/w when both are non-null.  T never round-trips through the host for K4. */
int hps_gpu_condense_assemble(hps_gpu_ctx* ctx, const double* b, const double* f, const double* g_bnd,
                              double* values, double* rhs, double* T, double* w, int32_t* status);

/* Same operation on device-resident buffers (inputs already in HBM, outputs
 * stay in HBM), enqueued on `stream` (cudaStream_t, NULL = ctx stream). */
int hps_gpu_condense_device(hps_gpu_ctx* ctx, int32_t e0, int32_t n, const double* d_b,
                            const double* d_f, double* d_T, double* d_w, int32_t* d_status,
                            void* stream);

/* Device-side sampling of the crystal coefficient field (SPEC.md:209-217,
 * problems.crystal_field) at the p*p local nodes of elements
 * [e0, e0+n) into d_b (leaf-major, the layout hps_gpu_condense_device reads):
 *   b = clamp(1 - sum_i depth exp(-|x - c_i|^2 / sigma^2), 0, 1)
 * with the ncent centres c_i given as (x, y) pairs in host memory.  Enqueued on
 * `stream` (NULL = ctx stream).  Replaces the host sampling + H2D of b. */
int hps_gpu_sample_crystal(hps_gpu_ctx* ctx, int32_t e0, int32_t n, const double* centres, int32_t ncent,
                           double sigma, double depth, double* d_b, void* stream);

/* Matrix-free residual of the global collocation system (SPEC.md:337-342,354-362,
 * Eq. 7) for the whole mesh, from leaf-major b, f and local
 * solutions u (p*p per leaf, e.g. hps_gpu_leaf_solve's output):
 *   out[0] = sum over interior rows of (A_loc u - f)^2,
 *   out[1] = sum over active interface rows of (sum of the two outward fluxes)^2,
 *   out[2] = sum over interior rows of f^2.
 * Dirichlet / interior-corner rows are identity rows, satisfied by construction;
 * relerr_res = sqrt((out[0] + out[1]) / (out[2] + sum g^2)).  Partials are summed in a
 * fixed order: bitwise reproducible.  Host-buffer and device-buffer variants. */
int hps_gpu_residual(hps_gpu_ctx* ctx, const double* b, const double* f, const double* u, double* out);
int hps_gpu_residual_device(hps_gpu_ctx* ctx, const double* d_b, const double* d_f, const double* d_u,
                            double* out, void* stream);

/* Batched leaf_solve for elements [e0, e1): u = p*p local
 * values, interior = A_ii^{-1}(f_i - A_ib v), boundary = v.  Recompute policy
 * rebuilds and refactors A_ii; store policy reuses the
 * factors kept by the last hps_gpu_condense over the same elements
 * (bitwise-identical results). */
int hps_gpu_leaf_solve(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* b, const double* f,
                       const double* v, double* u, int32_t* status);

/* reconstruct_full_solution on the device: boundary vectors of every
 * leaf from the reduced solution u_active (n_active, active_index order) and the Dirichlet
 * samples g_bnd (hps_gpu_assemble_reduced layout), interiors by batched leaf_solve (b, f:
 * all leaves' samples), placement into the full grid u_full (N values, g = gy*Nx + gx),
 * element corners on Gamma from g and interior corners by the corner policy (SPEC.md:152:
 * mean of the four adjacent edge interpolants).  status: per leaf (resonance).  The
 * device variant also returns the local solutions (d_u_leaf, nullable; p*p per leaf). */
int hps_gpu_reconstruct(hps_gpu_ctx* ctx, const double* u_active, const double* g_bnd, const double* b,
                        const double* f, double* u_full, int32_t* status);
int hps_gpu_reconstruct_device(hps_gpu_ctx* ctx, const double* d_u_active, const double* d_g_bnd,
                               const double* d_b, const double* d_f, double* d_u_full, double* d_u_leaf,
                               int32_t* d_status, void* stream);

/* assemble_reduced — K4.  Pattern: CSR of the reduced system
 * over active nodes, int64 row_ptr (n_active+1), int32 col_idx
 * (nnz).  Call with row_ptr == NULL to get nnz only. */
int hps_gpu_reduced_pattern(hps_gpu_ctx* ctx, int64_t* nnz, int64_t* row_ptr, int32_t* col_idx);
/* Per-leaf scatter map of assemble_reduced (SURVEY.md §8b hps_gpu_scatter_indices; the
 * COO/CSR indexing of SPEC.md:345-353,382), leaves [e0, e1), caller-owned host buffers:
 *   row[(e-e0)*nb + r]            active row of local boundary node r, -1 if corner/Dirichlet;
 *   slot[((e-e0)*nb + r)*nb + c]  index into the CSR values of hps_gpu_reduced_pattern that
 *                                 T_e[r, c] is summed into, -1 if row or column is inactive.
 * nb = 4(p-1); local boundary order S, E, N, W.  Bit-exact with
 * the CPU oracle's pattern; values[slot] accumulated in ascending e reproduce
 * hps_gpu_assemble_reduced's values bit for bit. */
int hps_gpu_scatter_indices(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, int64_t* slot, int64_t* row);
/* Values/rhs from all leaves' T and w (host, leaf-major, all nx*ny leaves) and
 * Dirichlet samples g_bnd = [south(Nx) | north(Nx) | west(Ny) | east(Ny)],
 * Nx = nx(p-1)+1, Ny = ny(p-1)+1. */
int hps_gpu_assemble_reduced(hps_gpu_ctx* ctx, const double* T, const double* w,
                             const double* g_bnd, double* values, double* rhs);
/* Device-resident variant (T, w, g_bnd, values, rhs in HBM). */
int hps_gpu_assemble_reduced_device(hps_gpu_ctx* ctx, const double* d_T, const double* d_w,
                                    const double* d_g_bnd, double* d_values, double* d_rhs,
                                    void* stream);

/* BSR view of the same reduced system (ReducedSystem.blocks maps
 * (interface edge, interface edge) pairs sharing an element to dense (p-2)x(p-2)
 * coupling blocks).  Block row i = interface edge i (active rows
 * i*q .. i*q+q-1, q = p-2 = *block_size), int64 brow_ptr (n_active/q + 1), int32
 * bcol_idx (nnzb, block columns = edge ids, ascending); call with brow_ptr == NULL
 * for block_size and nnzb only.  Values: nnzb blocks of q*q, row-major, holding
 * bit-for-bit the entries hps_gpu_assemble_reduced puts in CSR; rhs identical. */
int hps_gpu_reduced_bsr_pattern(hps_gpu_ctx* ctx, int32_t* block_size, int64_t* nnzb,
                                int64_t* brow_ptr, int32_t* bcol_idx);
int hps_gpu_assemble_reduced_bsr(hps_gpu_ctx* ctx, const double* T, const double* w,
                                 const double* g_bnd, double* bvalues, double* rhs);
int hps_gpu_assemble_reduced_bsr_device(hps_gpu_ctx* ctx, const double* d_T, const double* d_w,
                                        const double* d_g_bnd, double* d_bvalues, double* d_rhs,
                                        void* stream);

/* The reference's single-leaf operations on operators held as values,
 * batched over elements [e0, e1) (ids are used in error messages only):
 *   build_leaf_operator: from b samples (p*p per leaf) the dense
 *     A_loc = -(D (x) I)^2 - (I (x) D)^2 - kappa^2 diag(b)  (p^2 x p^2 row-major per leaf) and
 *     D_normal = the outward normal derivative maps of the S, E, N, W edges, each p x p^2
 *     (edge nodes ascending, corners on both edges; 4 p p^2 per leaf).
 *     Entries are bit-identical to the oracle's.
 *   condense_leaf of GIVEN operators: T, w, S (nullable) and status as
 *     hps_gpu_condense; interior/boundary blocks are gathered from A_loc, the flux rows from
 *     D_normal (a corner uses its owning edge).
 *   leaf_solve with a given A_loc: u (p*p per leaf) = [A_ii^{-1}(f_i -
 *     A_ib v) on the interior, v on the boundary].
 * Synchronous; the factors of the 'store' policy are not kept by these calls. */
int hps_gpu_build_leaf_operator(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* b, double* A_loc,
                                double* D_normal);
int hps_gpu_condense_operator(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* A_loc,
                              const double* D_normal, const double* f, double* T, double* w, double* S,
                              int32_t* status);
int hps_gpu_leaf_solve_operator(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* A_loc, const double* f,
                                const double* v, double* u, int32_t* status);

/* Kernel-path selection (results are the same to 1e-12; the default picks the faster one):
 *   HPS_OPT_SMALL_KERNEL  register-resident K2s for 4 <= p <= 12 (default on)
 *   HPS_OPT_LOCKSTEP      lock-step 4-leaf K2 CTAs for R <= 640, p <= 24 (default on)
 * value: -1 default, 0 off, 1 on.  For tests and A/B measurements. */
#define HPS_OPT_SMALL_KERNEL 1
#define HPS_OPT_LOCKSTEP 2
int hps_gpu_set_option(hps_gpu_ctx* ctx, int32_t option, int32_t value);

/* Test hook: zero interior row 0 of A_ii for these element
 * ids, which forces a zero pivot.  n = 0 clears. */
int hps_gpu_set_fault_injection(hps_gpu_ctx* ctx, const int32_t* elements, int32_t n);

/* ---- Leaf-range sharding over the GPUs of one box (parallel.hpp:21-24;
 * SPEC.md:291,317).  One ctx per entry of `devices` (a device may repeat), one host thread
 * per ctx, contiguous element ranges balanced to +-1 leaf (hps_shard_range), each shard
 * writing its disjoint leaf-major slots of the caller's host buffers.  No collective on the
 * data path.  Results are bitwise those of a single ctx.  assemble_reduced: each shard runs
 * K4 on the interface edges inside its range; edges cut by a shard boundary are summed on
 * the host in K4's operation order (hps_reduced_host_edges). ---- */
typedef struct hps_gpu_multi hps_gpu_multi;
int hps_gpu_multi_create(const int32_t* devices, int32_t n_devices, const hps_leaf_desc* desc,
                         hps_gpu_multi** out);
void hps_gpu_multi_destroy(hps_gpu_multi* m);
const char* hps_gpu_multi_last_error(const hps_gpu_multi* m);
/* Number of shards; lo/hi (nullable, length >= shards) receive each shard's leaf range. */
int hps_gpu_multi_shards(const hps_gpu_multi* m, int32_t* lo, int32_t* hi);
hps_gpu_ctx* hps_gpu_multi_ctx(hps_gpu_multi* m, int32_t shard);
int hps_gpu_multi_condense(hps_gpu_multi* m, int32_t e0, int32_t e1, const double* b, const double* f, double* T,
                           double* w, int32_t* status);
int hps_gpu_multi_leaf_solve(hps_gpu_multi* m, int32_t e0, int32_t e1, const double* b, const double* f,
                             const double* v, double* u, int32_t* status);
int hps_gpu_multi_assemble_reduced(hps_gpu_multi* m, const double* T, const double* w, const double* g_bnd,
                                   double* values, double* rhs);

/* Host-only pieces of the sharded path (no GPU involved). */
/* Leaf range [lo, hi) of shard i of k over n leaves (sizes n/k or n/k + 1, larger first). */
int hps_shard_range(int32_t n, int32_t k, int32_t i, int32_t* lo, int32_t* hi);
/* Interface edges whose two elements lie on different shards (shard_lo: first leaf of each
 * of the k shards, ascending); edges == NULL returns the count only. */
int hps_reduced_cut_edges(int32_t p, int32_t nx, int32_t ny, const int32_t* shard_lo, int32_t k, int32_t* edges,
                          int64_t* n_cut);
/* K4's values/rhs of the listed edges computed on the host in K4's operation order
 * (bit-identical), from all leaves' T and w (leaf-major) and g_bnd. */
int hps_reduced_host_edges(int32_t p, int32_t nx, int32_t ny, const int32_t* edges, int64_t n, const double* T,
                           const double* w, const double* g_bnd, double* values, double* rhs);

/* Pinned host memory helpers. */
void* hps_host_alloc(size_t bytes);
void hps_host_free(void* ptr);

/* FP64 tensor (DMMA) peak of `device` in TF/s, measured now with a register-only
 * mma.sync.m8n8k4.f64 loop (~0.1 s): the roofline denominator of K2/K3. */
double hps_gpu_fp64_peak_tflops(int device);

/* The same loop run back to back for `seconds` (<= 0: 3 s), rate of the last third: the
 * power-limited steady state, the denominator for kernels timed inside a long step (as
 * MEASURED_PEAKS.json's bf16_tflops_sustained). */
double hps_gpu_fp64_peak_tflops_sustained(int device, double seconds);

/* Library identity (for load checks). */
const char* hps_gpu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HPS_LEAF_GPU_H */
