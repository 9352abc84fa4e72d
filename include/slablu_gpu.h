/*
 * slablu_gpu.h — C ABI of the B200-native SlabLU engine (libslablu_gpu.so).
 *
 * Drop-in boundary for the reference's dense-mode factorize/solve path
 * (arxiv/paper_2211_07572, /root/reference/proj/include/slablu/):
 *
 *   slablu_gpu_assemble_fd5*   <- assemble_fd5            (problem.hpp:78-132)
 *   slablu_gpu_assemble_canned_device, _sample_solution_device, _error_report(_device)
 *                              <- assemble_fd5 / sample_field / error_report on the device
 *                                                         (problem.hpp:78-132, 160-206; §8(f)2)
 *   slablu_gpu_choose_b        <- choose_b                (driver.hpp:55-66)
 *   slablu_gpu_partition       <- partition               (partition.hpp:70-91)
 *   slablu_gpu_factorize       <- factorize               (driver.hpp:115-167)
 *   slablu_gpu_solve           <- solve                   (driver.hpp:171-179)
 *   slablu_gpu_stats           <- Factorization fields    (driver.hpp:72-87)
 *   slablu_gpu_T_block         <- ReducedSystem blocks    (stage_one.hpp:303-338, staged parity)
 *   slablu_gpu_reduce_rhs      <- reduce_rhs              (stage_one.hpp:415-433, staged parity)
 *   slablu_gpu_sweep_solve     <- sweep_solve             (stage_two.hpp:245-248 -> 170-188, staged)
 *   slablu_gpu_recover         <- recover_interiors       (stage_one.hpp:438-462, staged)
 *   slablu_gpu_sweep_build     <- sweep_build / SweepFactorization(BlockTridiagonal)
 *                                                         (stage_two.hpp:41-56, 131-150, 241-243)
 *   slablu_gpu_destroy         <- ~Factorization
 *   slablu_gpu_save / _load / _export_sweep / _import_sweep
 *                              <- serialize / deserialize (stage_two.hpp:95-120, 200-232; dense.hpp:71-87)
 *   slablu_gpu_shard_*         <- (no reference counterpart: the multi-GPU split of
 *                                 factorize/solve designed in SURVEY.md §8(e))
 *
 * Conventions (mirroring the reference):
 *   - matrices are column major; the operator is the reference's CSR
 *     (Eigen RowMajor compressed: int32 row_ptr[n+1], int32 col_idx[nnz],
 *     double val[nnz]), unknown (i, j) at index i*n2 + j.
 *   - errors are returned as a status; code SLABLU_ERR_CONFIG maps to
 *     ConfigError, SLABLU_ERR_SINGULAR to SingularMatrixError(index), every
 *     other nonzero code to Error (common.hpp:32-60).
 *   - a factorization is immutable after slablu_gpu_factorize and owns all of
 *     its device memory; solves are const and may be issued repeatedly.
 *   - there is no CPU fallback: without a usable CUDA device every compute
 *     entry point returns SLABLU_ERR_CUDA.
 *   - device-pointer entry points run on the factorization's own stream: the
 *     caller's writes to their inputs must be complete before the call, and
 *     outputs are complete when the call returns.
 */
#ifndef SLABLU_GPU_H
#define SLABLU_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SLABLU_OK = 0,
  SLABLU_ERR_GENERIC = 1,     /* Error */
  SLABLU_ERR_CONFIG = 2,      /* ConfigError */
  SLABLU_ERR_SINGULAR = 3,    /* SingularMatrixError; index = strip or block */
  SLABLU_ERR_CUDA = 4,        /* CUDA runtime failure or no device */
  SLABLU_ERR_OOM = 5,         /* device memory exhausted */
  SLABLU_ERR_UNSUPPORTED = 6, /* valid input outside the engine's envelope */
  SLABLU_ERR_COMPRESSION = 7  /* CompressionError (common.hpp:55-60); residual estimate in .residual */
};

/* SolverConfig (driver.hpp:41-50). compression: 0 automatic, 1 dense, 2 hbs; automatic
 * resolves to hbs when n2 >= 512 and b >= 16, else dense (driver.hpp:125-130).  The hbs_*
 * fields follow the reference's defaults when left 0 (1e-11, 1e-13, 64). */
typedef struct {
  int64_t b;          /* explicit slab width; 0 derives it from c */
  double c;           /* b ~ c * n2^(2/3), c in (0, 2] */
  int compression;
  uint64_t seed;
  int threads;        /* accepted, unused (as in the reference) */
  int device;         /* CUDA device ordinal */
  int keep_T;         /* keep a copy of the reduced blocks for slablu_gpu_T_block */
  int refine;         /* iterative-refinement steps per solve (residual with the original CSR) */
  double hbs_tol;         /* per-block compression tolerance (0: 1e-11) */
  double hbs_trunc_rel;   /* generator truncation floor (0: 1e-13) */
  int64_t hbs_leaf_size;  /* cluster-tree leaf size (0: 64) */
} slablu_gpu_config;

typedef struct {
  int code;
  int64_t index;
  char msg[256];
  double residual;    /* SLABLU_ERR_COMPRESSION: the probe's residual estimate */
} slablu_gpu_status;

typedef struct {
  int64_t n1, n2, b;
  int64_t interfaces;     /* k */
  int64_t strips;
  int64_t padded_width;   /* Wp */
  int single_slab;        /* degenerate whole-grid path */
  int symmetric_strips;   /* strips that took the symmetric Schur shortcut */
  double t_stage1;        /* seconds, device time (CUDA events) */
  double t_stage2;
  int64_t storage_stage1; /* reference-equivalent scalars (driver.hpp:153-159) */
  int64_t storage_stage2; /* (stage_two.hpp:191-198) */
  int64_t device_bytes;   /* bytes held by the factorization */
  int64_t gpu_launches;   /* kernels launched by the last factorize */
  int64_t solve_launches; /* kernels launched by the last solve */
  double t_chain;         /* stage one: block band LU of all slabs (s, CUDA events) */
  double t_schur;         /* stage one: Schur sweep kernel (s, CUDA events) */
  double t_assemble;      /* stage one: T assembly + validation (s) */
  double t_solve_last;    /* device time of the last solve (s) */
  double t_solve_strips;  /* ... of which the two slab sweeps (reduce + recover) */
  int compression;        /* resolved: 1 dense, 2 hbs */
  int64_t hbs_max_rank;   /* Factorization::hbs_max_rank (driver.hpp:84) */
  double t_hbs;           /* stage one: HBS compression of the reduced blocks (s) */
} slablu_gpu_stats_t;

typedef struct slablu_gpu_fact slablu_gpu_fact;

/* ---- problem assembly (host) ------------------------------------------- */
typedef double (*slablu_field_fn)(double x, double y, void* user);
/* Generic ProblemSpec: coefficient b(x), Dirichlet data g, body load f. Fills
 * caller buffers row_ptr[n+1], col_idx[5n], val[5n], rhs[n]; *nnz receives
 * the entry count. */
slablu_gpu_status slablu_gpu_assemble_fd5(int64_t n1, int64_t n2, double h, double kappa,
                                          slablu_field_fn coefficient, slablu_field_fn dirichlet,
                                          slablu_field_fn load, void* user, int32_t* row_ptr,
                                          int32_t* col_idx, double* val, double* rhs,
                                          int64_t* nnz);
/* Canned problems (problem.hpp:210-261): 0 poisson_log, 1 helmholtz, 2 helmholtz_bump. */
slablu_gpu_status slablu_gpu_assemble_canned(int kind, int64_t n1, int64_t n2, double kappa,
                                             int32_t* row_ptr, int32_t* col_idx, double* val,
                                             double* rhs, int64_t* nnz);
/* Manufactured solution of a canned problem sampled on the grid (problem.hpp:199-206). */
slablu_gpu_status slablu_gpu_sample_solution(int kind, int64_t n1, int64_t n2, double kappa,
                                             double* out);
/* On-device assembly of a canned problem: CSR + rhs written to device memory of
 * `device` (d_rp[n+1], d_ci[5n], d_v[5n], d_rhs[n]).  Index arrays equal slablu_gpu_assemble_canned's;
 * values follow the same operation order (bit-identical except libm-level differences in exp, and in
 * the log / J0 Dirichlet data of the boundary rhs entries: ~1e-15 / ~1e-12 relative). */
slablu_gpu_status slablu_gpu_assemble_canned_device(int kind, int64_t n1, int64_t n2, double kappa, int device,
                                                    int32_t* d_rp, int32_t* d_ci, double* d_v, double* d_rhs,
                                                    int64_t* nnz);
slablu_gpu_status slablu_gpu_sample_solution_device(int kind, int64_t n1, int64_t n2, double kappa, int device,
                                                    double* d_out);
/* error_report (problem.hpp:160-196): out[0] relerr_res = ||A u - f|| / ||f||, out[1] relerr_true =
 * ||u - u_true|| / ||u_true|| (Frobenius over the nrhs columns; absolute if the norm vanishes, flagged
 * in out[2] / out[3]; u_true NULL gives NaN), vectors n x nrhs with ld n.  _device: device pointers. */
slablu_gpu_status slablu_gpu_error_report(int64_t n, const int32_t* row_ptr, const int32_t* col_idx,
                                          const double* val, const double* f, const double* u,
                                          const double* u_true, int64_t nrhs, int device, double* out);
slablu_gpu_status slablu_gpu_error_report_device(int64_t n, const int32_t* d_row_ptr, const int32_t* d_col_idx,
                                                 const double* d_val, const double* d_f, const double* d_u,
                                                 const double* d_u_true, int64_t nrhs, int device, double* out);
double slablu_gpu_kappa_from_ppw(double ppw, int64_t n2);
double slablu_gpu_bessel_j0(double t);
/* gaussian_matrix (common.hpp:72-79): mt19937_64(seed) + normal_distribution. */
void slablu_gpu_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out);

/* ---- geometry ---------------------------------------------------------------- */
slablu_gpu_status slablu_gpu_choose_b(int64_t n1, int64_t n2, int64_t b, double c, int64_t* out);
/* interior/interface strips as (first_col, width) pairs; cap = pairs available. */
slablu_gpu_status slablu_gpu_partition(int64_t n1, int64_t n2, int64_t b, int64_t* n_interiors,
                                       int64_t* interiors, int64_t* n_interfaces,
                                       int64_t* interfaces, int64_t cap);

/* ---- factorize / solve ------------------------------------------------------ */
/* Randomized HBS compression of one dense n x n operator (host buffers, column major), the
 * reference's hbs_compress (adaptive = 0, rank bound r_max) / hbs_compress_adaptive
 * (adaptive = 1, ranks r_start doubling to r_max) with the dense sampler of test_hbs.cpp:64-68
 * (hbs_compress.hpp:186-311).  out = the dense materialization of the compressed operator
 * (HbsMatrix::to_dense, hbs.hpp:150-154).  CompressionError -> SLABLU_ERR_COMPRESSION. */
typedef struct {
  int64_t products_normal, products_adjoint;
  int rounds;
  int64_t final_rank;
  double residual_estimate;
} slablu_gpu_hbs_stats;
slablu_gpu_status slablu_gpu_hbs_compress(int64_t n, const double* m, int64_t leaf_size, int64_t r_start,
                                          int64_t r_max, int adaptive, double tol, double trunc_rel,
                                          uint64_t seed, int device, double* out, slablu_gpu_hbs_stats* stats);

/* Host CSR. */
slablu_gpu_status slablu_gpu_factorize(int64_t n1, int64_t n2, const int32_t* row_ptr,
                                       const int32_t* col_idx, const double* val,
                                       const slablu_gpu_config* config, slablu_gpu_fact** out);
/* Device-resident CSR (pointers into device memory of config->device). */
slablu_gpu_status slablu_gpu_factorize_device(int64_t n1, int64_t n2, int64_t nnz,
                                              const int32_t* d_row_ptr, const int32_t* d_col_idx,
                                              const double* d_val, const slablu_gpu_config* config,
                                              slablu_gpu_fact** out);
/* u (n x nrhs, ld ldu) = A^{-1} f (n x nrhs, ld ldf); host buffers. */
slablu_gpu_status slablu_gpu_solve(const slablu_gpu_fact* fact, const double* f, int64_t ldf,
                                   int64_t nrhs, double* u, int64_t ldu);
/* Same with device buffers; stream 0 of the factorization's device. */
slablu_gpu_status slablu_gpu_solve_device(const slablu_gpu_fact* fact, const double* d_f,
                                          int64_t ldf, int64_t nrhs, double* d_u, int64_t ldu);
slablu_gpu_status slablu_gpu_stats(const slablu_gpu_fact* fact, slablu_gpu_stats_t* out);
/* Refinement steps of later solves (SolverConfig.refine); raising it above 0 needs a factorization
 * made with refine > 0 (the original operator is kept only then). */
slablu_gpu_status slablu_gpu_set_refine(slablu_gpu_fact* fact, int refine);
/* Reduced block before stage two (needs config.keep_T): which 0 diag[j], 1 super[j], 2 sub[j]. */
slablu_gpu_status slablu_gpu_T_block(const slablu_gpu_fact* fact, int which, int64_t j, double* out);
/* Staged reduce_rhs: out (k*n2 x nrhs) from host f (n x nrhs, ld n). */
slablu_gpu_status slablu_gpu_reduce_rhs(const slablu_gpu_fact* fact, const double* f, int64_t nrhs,
                                        double* out);
/* Staged sweep solve: u_ifc (k*n2 x nrhs) = T^{-1} red through the LU factors of S_j (host buffers). */
slablu_gpu_status slablu_gpu_sweep_solve(const slablu_gpu_fact* fact, const double* red, int64_t nrhs,
                                         double* u_ifc);
/* sweep_build on a caller's block-tridiagonal system (host): blocks = [diag 0..k-1 | super
 * 0..k-2 | sub 0..k-2], each m x m column major.  Rejects k < 1 (ConfigError) and non-finite
 * entries (Error); a singular S_j raises SingularMatrixError(j).  The handle serves
 * slablu_gpu_sweep_solve (m*k x nrhs) and slablu_gpu_stats; release with slablu_gpu_destroy. */
slablu_gpu_status slablu_gpu_sweep_build(int64_t m, int64_t k, const double* blocks, int device,
                                         slablu_gpu_fact** out);
/* Staged recover_interiors: u (n x nrhs, ld n) from f (n x nrhs, ld n) and u_ifc (k*n2 x nrhs);
 * interface entries of u are copied from u_ifc (host buffers). */
slablu_gpu_status slablu_gpu_recover(const slablu_gpu_fact* fact, const double* f, const double* u_ifc,
                                     int64_t nrhs, double* u);
void slablu_gpu_destroy(slablu_gpu_fact* fact);

/* ---- factor caching ---------------------------------------
 * save / load: the whole GPU factorization in a versioned file (magic SLBGPU01, named sections),
 * factor once, solve in another process.  export_sweep / import_sweep: stage two in the
 * reference's SweepFactorization layout (magic SLBSWP01, stage_two.hpp:200-232 with DenseLU
 * dense.hpp:71-87: write_dense blocks, int64 1-based pivots), so stage-two factors move between
 * the reference and the GPU engine; an imported handle serves slablu_gpu_sweep_solve. */
slablu_gpu_status slablu_gpu_save(const slablu_gpu_fact* fact, const char* path);
slablu_gpu_status slablu_gpu_load(const char* path, int device, slablu_gpu_fact** out);
slablu_gpu_status slablu_gpu_export_sweep(const slablu_gpu_fact* fact, const char* path);
slablu_gpu_status slablu_gpu_import_sweep(const char* path, int device, slablu_gpu_fact** out);

/* ---- multi-GPU: strip-sharded factorization and solve ----------------------
 * One process per GPU.  Rank r of G owns the contiguous global strips [s_begin, s_end)
 * (s_begin = r*S/G) and the interfaces [j_begin, j_end) (j_begin = s_begin - 1 for r > 0; the last
 * rank also owns a trailing interface).  For r > 0 interface j_begin is the rank's SEPARATOR; the
 * rest is its interior chain.  Stage one (band LU, Schur blocks) is local.  Stage two is a
 * partitioned (SPIKE-style) elimination: every rank eliminates its interior chain on its own, then
 * the G - 1 separators are swept in rank order with ONE message per rank boundary (the caller moves
 * it: ncclSend/ncclRecv over NVLink between processes, or a device copy between logical shards):
 *   factorize : shard_factorize_device; shard_eliminate (no communication);
 *               shard_sweep(in from r-1, out to r+1), messages n2 x n2 (ld n2)
 *   solve     : shard_solve_local (no communication);
 *               shard_solve_forward(in from r-1, out to r+1);
 *               shard_solve_backward(in from r+1, out to r-1), messages n2 x nrhs (ld n2)
 * NULL message pointers on the ends (rank 0 has no "from r-1" etc.).  All buffers are device
 * memory of the shard's device.  A sharded factorization is not usable with slablu_gpu_solve; the
 * sharded solve keeps per-solve state in the factorization (one solve at a time) and does no
 * refinement (slablu_gpu_residual serves a host-driven one). */
typedef struct {
  int rank, nranks;
  int64_t s_begin, s_end;     /* local strips (global indices) */
  int64_t j_begin, j_end;     /* owned interfaces */
  int64_t n_strips, n_interfaces;  /* global counts */
} slablu_gpu_shard_t;
slablu_gpu_status slablu_gpu_shard_plan(int64_t n1, int64_t n2, int64_t b, int rank, int nranks,
                                        slablu_gpu_shard_t* out);
slablu_gpu_status slablu_gpu_shard_factorize_device(int64_t n1, int64_t n2, int64_t nnz,
                                                    const int32_t* d_row_ptr, const int32_t* d_col_idx,
                                                    const double* d_val, const slablu_gpu_config* config,
                                                    int rank, int nranks, slablu_gpu_fact** out);
slablu_gpu_status slablu_gpu_shard_eliminate(slablu_gpu_fact* fact);
slablu_gpu_status slablu_gpu_shard_sweep(slablu_gpu_fact* fact, const double* d_in, double* d_out);
/* d_f: n x nrhs (ld ldf >= n) device; kept (copied) until the backward phase. */
slablu_gpu_status slablu_gpu_shard_solve_local(slablu_gpu_fact* fact, const double* d_f, int64_t ldf, int64_t nrhs);
slablu_gpu_status slablu_gpu_shard_solve_forward(slablu_gpu_fact* fact, const double* d_in, double* d_out);
/* d_u: n x nrhs with ldu == n; receives the shard's unknowns, other entries untouched. */
slablu_gpu_status slablu_gpu_shard_solve_backward(slablu_gpu_fact* fact, const double* d_in, double* d_out,
                                                  double* d_u, int64_t ldu);
/* r = f - A u over all n rows with the operator kept by a factorization made with
 * config.refine > 0 (device buffers, ld n); the host-driven refinement of the sharded solve. */
slablu_gpu_status slablu_gpu_residual(const slablu_gpu_fact* fact, const double* d_f, int64_t ldf, int64_t nrhs,
                                      const double* d_u, int64_t ldu, double* d_r);

/* Device count visible to the engine (0 when CUDA is unusable). */
int slablu_gpu_device_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SLABLU_GPU_H */
