/* ===========================================================================
 * hps_slablu.h — C-ABI of the GPU SlabLU reduced-system solver
 * (paper_2211_14969_b200/_lib/libhps_slablu_b200.so).
 *
 * Replaces the reference's slablu module:
 *   partition_slabs  contiguous element-column slabs of `slab_width`
 *                                      elements, the last absorbing the remainder; slab
 *                                      interiors = interfaces strictly inside a slab,
 *                                      slab interfaces = the vertical edge columns
 *                                      between slabs (in the active ordering, SPEC.md:154,
 *                                      the unknowns are [I_0 | B_0 | I_1 | ... | I_{S-1}]);
 *   factor           dense partial-pivoted LU of every slab interior,
 *                                      Schur complements onto its two bounding interfaces,
 *                                      block-tridiagonal forward sweep (block Thomas) over
 *                                      the interfaces without inter-block pivoting;
 *   solve            slab-interior solves, interface forward/backward
 *                                      sweep, interior back substitution.
 * Dense blocks are column-major in HBM; the dense LU / triangular solves / GEMMs are
 * cuSOLVER (getrf/getrs, 64-bit API) and cuBLAS (DGEMM/DGEMV) library calls, the gathers
 * from the reduced system's BSR view (hps_gpu_reduced_bsr_pattern) and the
 * pivot checks are this library's kernels.
 * Errors (errors.hpp): HPS_ERR_PARAM (ParameterError: widths leaving < 2 slabs,
 * SPEC.md:418), HPS_ERR_SINGULAR_BLOCK (SingularBlockError(block_index), errors.hpp:30-38:
 * a pivot below 1e-12 of the block's inf-norm; index = interface k, or -1 - s for the
 * interior of slab s), HPS_ERR_CUDA.  The factorization is immutable; solves may repeat.
 * =========================================================================== */
#ifndef HPS_SLABLU_H
#define HPS_SLABLU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_SLABLU_OK 0
#define HPS_ERR_SINGULAR_BLOCK 4   /* HPS_ERR_PARAM 2, HPS_ERR_CUDA 3 as in hps_leaf_gpu.h */

typedef struct hps_slablu hps_slablu;

typedef struct {
  int32_t slab_width;   /* elements per slab actually used */
  int32_t n_slabs;
  int64_t n_active;
  int64_t max_interior; /* largest slab-interior block */
  int64_t n_interface;  /* unknowns per slab interface (ny * (p-2)) */
  int64_t device_bytes; /* HBM held by the factorization */
  float ms_factor;      /* device time of the factorization (CUDA events) */
  float ms_solve;       /* device time of the last solve */
} hps_slablu_info_t;

/* SPEC.md:421 default slab width: ceil(n_active_per_element_column^(1/3)), clamped to
 * [1, nx/2]; then reduced while the factorization would exceed `device_budget_bytes`
 * (0: 70% of free HBM). */
int32_t hps_slablu_default_width(int32_t p, int32_t nx, int32_t ny, int64_t device_budget_bytes);

/* Factor the reduced system given in its BSR view (host arrays: brow_ptr n_edges+1,
 * bcol_idx nnzb, blocks nnzb*q*q row-major, q = p-2).  slab_width <= 0 picks the default. */
int hps_slablu_factor(int device, int32_t p, int32_t nx, int32_t ny, int32_t slab_width,
                      const int64_t* brow_ptr, const int32_t* bcol_idx, const double* blocks,
                      hps_slablu** out);
/* x = A^{-1} rhs (host vectors of n_active). */
int hps_slablu_solve(hps_slablu* s, const double* rhs, double* x);
int hps_slablu_get_info(const hps_slablu* s, hps_slablu_info_t* out);
/* Message of the last failure (s == NULL: of the last failed hps_slablu_factor on this
 * thread); the failing block index of a SingularBlockError. */
const char* hps_slablu_last_error(const hps_slablu* s);
int32_t hps_slablu_last_block(void);
void hps_slablu_destroy(hps_slablu* s);

#ifdef __cplusplus
}
#endif

#endif /* HPS_SLABLU_H */
