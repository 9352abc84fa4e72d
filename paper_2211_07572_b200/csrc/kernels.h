// Internal launcher declarations for the SlabLU B200 engine.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace slb {

// ---- gemm.cu -------------------------------------------------------------
void dgemm_batched(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                   int64_t lda, int64_t sA, const double* B, int64_t ldb, int64_t sB, double beta,
                   double* C, int64_t ldc, int64_t sC, int64_t batch, bool transA = false);
// Batched triangular solve X = T^{-1} B in place, T m x m (m <= 160) stored
// ROW-major (T[r][c] at T[r * ldt + c]); lower => unit-lower forward,
// else upper (non-unit) backward.  B is m x ncols column major.
void trsm_small_batched(cudaStream_t st, bool lower, int m, const double* T, int64_t ldt, int64_t sT,
                        double* B, int64_t ldb, int64_t sB, int64_t ncols, int64_t batch, bool rowmajor = true);
void dscale_batched(cudaStream_t st, int64_t M, int64_t N, double beta, double* C, int64_t ldc,
                    int64_t sC, int64_t batch);

// ---- strips ----------------------------------------------------------------
// One interior strip (slab) of the partition, with its adjacent interfaces.
struct StripDesc {
  int32_t col0;       // first grid column
  int32_t w;          // real width (<= Wp)
  int32_t left;       // left interface id or -1
  int32_t right;      // right interface id or -1
  int64_t left_off;   // global index of the left interface's first unknown, -1
  int64_t right_off;  // same for the right interface
};

// Error flags raised by the extraction / factor kernels (bitmask).
enum ErrBits : int32_t {
  ERR_OUT_OF_BAND = 1,        // interior entry outside the kl=ku=w band
  ERR_PAST_INTERFACE = 2,     // interior couples past its adjacent interfaces
  ERR_COUPLING_LEVEL = 4,     // interior<->interface coupling across levels
  ERR_SINGULAR = 8,           // exactly singular pivot
  ERR_IFC_STRUCTURE = 16,     // interface row couples outside adjacent strips/interfaces
  ERR_NONFINITE = 32,         // non-finite reduced block entry
  ERR_CHAIN_TIMEOUT = 64,     // getrs_chain: a published block never arrived (bounded spin expired)
};
struct DevStatus {
  int32_t flags;
  int32_t singular_strip;  // lowest strip index with a singular pivot (or INT_MAX)
  int32_t singular_block;  // lowest sweep block index with a singular pivot
  int32_t singular_pos;    // single strip: lowest level * Wp + column of a zero pivot (or INT_MAX)
};

// ---- band_lu.cu --------------------------------------------------------------
struct CsrDev {
  const int32_t* rp;
  const int32_t* ci;
  const double* v;
  int64_t n;
};

// Extract per-level dense blocks [Lsub | D | Usup] (Wp x 3Wp, ld Wp) for levels
// [L0, L0+nl) of every strip into nx (stride per strip sNX, per level 3*Wp*Wp).
// Also records, per (strip, level L), the diagonal of Lsub_L into dsub[s][L-1][i] and whether
// Lsub_L has an off-diagonal entry into lnd[s][L] (the forward sweep shortcut needs diagonal Lsub).
void extract_levels(cudaStream_t st, CsrDev A, const StripDesc* strips, int nstrips, int64_t n2,
                    int Wp, int64_t L0, int64_t nl, double* nx, int64_t sNX, DevStatus* status, double* dsub,
                    uint8_t* lnd);
// Per-level coupling vectors fromL/fromR/toL/toR (n2 x Wp each per strip).
void extract_couplings(cudaStream_t st, CsrDev A, const StripDesc* strips, int nstrips, int64_t n2,
                       int Wp, double* cpl, int64_t sCPL, int32_t* sym_flags, DevStatus* status);
// SV(level 0) = [D_0 | Usup_0] from the level-0 extracted blocks.
void init_sv(cudaStream_t st, int nstrips, int Wp, const double* nx0, int64_t sNX, double* sv,
             int64_t sSV);
// One level step of the block band LU for all strips (see band_lu.cu).
struct LevelArgs {
  int Wp;
  int nstrips;
  int has_next;          // level l+1 exists
  const double* sv_in;   // Wp x 2Wp per strip  [S | V]
  int64_t sSV;
  const double* nx;      // Wp x 3Wp per strip  [Lsub | D | Usup] of level l+1
  int64_t sNX;
  double* sv_out;        // Wp x 2Wp per strip: receives R2 (prefill for the update)
  double* slot;          // level slot (4 Wp^2): [LU11 | L21 | U1213]
  int64_t sF;            // per-strip stride of factor storage
  int32_t* perm;         // 2Wp      (factor storage, level l)
  int64_t sP;
  uint8_t* u13;          // flags of this level (per strip stride n2): bit 0 U13 != 0 (a level-l+1
                         // row pivoted up), bit 1 Lsub_{l+1} not diagonal; 0 = Fbot t = -dsub * y
  int64_t sU13;
  const uint8_t* lnd;    // Lsub_{l+1} off-diagonal flag (per strip stride n2), level l+1
  DevStatus* status;
  int32_t level;
  int tw0 = 0;  // measurement knob of level_lu_la_kernel (first trailing warp beside the panel)
};
void level_lu(cudaStream_t st, const LevelArgs& a);
// U1213 = L11^{-1} R1 and [S|V]_{l+1} = R2 - L21 U1213 in one launch (trsm.cu).
void level_update(cudaStream_t st, const LevelArgs& a);
// perm: the chunk's first level (2 Wp per level); exc/excpos: that level's exceptional Fbot rows
void convert_levels(cudaStream_t st, int Wp, double* slots, int64_t lvl, int64_t nl, double* work,
                    const int32_t* perm, double* exc, int32_t* excpos, double* hcol, int32_t* hidx);

// ---- schur.cu --------------------------------------------------------------------
struct SchurArgs {
  int Wp;
  int64_t n2;
  int nstrips;
  const StripDesc* strips;
  const double* fac;      // factor storage base (per strip stride sF; per level 4*Wp*Wp)
  int64_t sF;
  const int32_t* perm;    // per strip stride sP; per level 2*Wp
  int64_t sP;
  const double* cpl;      // coupling vectors (per strip sCPL): fromL, fromR, toL, toR (n2 x Wp each)
  int64_t sCPL;
  const int32_t* sym;     // per-strip symmetric flag
  const uint8_t* u13;     // per (strip, level) flags: bit 0 U13 != 0, bit 1 Lsub_{l+1} not diagonal
  const double* dsub;     // per (strip, level) diag(Lsub_{l+1}) (Wp), per strip stride n2 * Wp
  int fsc;                // forward shortcut enabled (Lsub diagonal, <= 8 rows pivoted up)
  const double* exc;      // per (strip, level) up to 8 exceptional Fbot rows (8 x Wp), strip stride n2*8*Wp
  const int32_t* excpos;  // their bottom positions (8 per level, -1 unused), strip stride n2*8
  int bsc;                // backward shortcut: x_{l+2} half of H applied as <= 8 columns
  const double* hcol;     // per (strip, level) those columns (8 x Wp), strip stride n2*8*Wp
  const int32_t* hidx;    // their indices (8 per level, -1 unused), strip stride n2*8
  double* gbuf;           // per strip 4 * n2 * n2 (row-major [X][Y][p][q])
  int64_t sG;
  double* ybuf;           // per CTA slot: n2 * Wp * C
  int64_t sY;
  int32_t* task_counter;
  int ntasks;
  const int32_t* tasks;   // packed (strip, side, q0) triples (solve modes: side unused, q0 = rhs col0)
  int mode;               // SweepMode
  int chunk;              // RHS columns per task: 64 (Schur, batched solves) or 8 (small solves)
  // solve modes
  int64_t N, K, nrhs;
  const double* f;        // N x nrhs (ld N), natural ordering
  const double* u_ifc;    // K x nrhs (recover)
  double* out;            // reduce: contrib[s][X][nrhs][n2]; recover: u (N x nrhs)
};
enum SweepMode { SWEEP_SCHUR = 0, SWEEP_REDUCE = 1, SWEEP_RECOVER = 2 };
// 4-D TMA map {32 doubles, m tiles, k4 rows, level} over per-level operator blocks in DMMA fragment
// order [k4][m8][lane] (solve2.cu): base = first tile, tile_stride tiles per k4 row, box_mt x box_k.
CUtensorMap make_map(const double* base, int mt, int tile_stride, int k4rows, int64_t levels, int64_t lvl_doubles,
                     int box_mt, int box_k);
constexpr int kSweepChunk = 64;
void sweep(cudaStream_t st, const SchurArgs& a, int nslots);
// Solve-phase slab sweeps (8 RHS columns per task) on clusters of 4 CTAs (solve.cu);
// ybuf holds ntasks slabs of n2 * Wp * 8 doubles.
bool strip_solve_fits(int Wp, int64_t n2);
void strip_solve(cudaStream_t st, const SchurArgs& a, int ntasks);  // launches 2 kernels
// b_l of every (task, level) packed level-major into ybuf (8 columns per task), recover-mode
// couplings folded in.
void strip_rhs_pack(cudaStream_t st, const SchurArgs& a, int ntasks);
// Version 2 (solve2.cu): TMA tensor slices + st.async level exchange, cluster size chosen at run
// time (2..8 CTAs); ybuf as for strip_solve.
bool strip_solve2_fits(int Wp, int64_t n2, int G, bool dmma_only = false);
int strip_solve2_cluster(int Wp, int64_t n2, int ntasks, bool dmma = false);
void strip_solve2(cudaStream_t st, const SchurArgs& a, int ntasks);

// T block assembly from per-strip G buffers (reference order: direct, left strip, right strip).
// Interface-block ranges of a (possibly sharded) factorization: local strips are the global
// strips [sbase, sbase + nstrips); diag blocks [dlo, dhi) receive local strip terms, owned
// interfaces [olo, ohi) also their direct operator terms, super/sub [ulo, uhi) come from local strips.
struct TRanges {
  int sbase = 0, nstrips_global = 0;
  int dlo = 0, dhi = 0, olo = 0, ohi = 0, ulo = 0, uhi = 0;
};
void assemble_T(cudaStream_t st, int64_t n2, int nifc, int nstrips, const StripDesc* strips,
                const int32_t* sym, const double* gbuf, int64_t sG, double* Tdiag, double* Tsup,
                double* Tsub, CsrDev A, const int64_t* ifc_off, DevStatus* status, const TRanges& tr);

// ---- dense.cu (stage two) -------------------------------------------------------
// In-place LU with partial pivoting of an n x n column-major matrix (ld = n).
void dgetrf(cudaStream_t st, int64_t n, double* a, int32_t* ipiv, double* work, DevStatus* status,
            int block_index);
// dgetrf with columns [h, n) produced concurrently on another stream (event right_ready).
void dgetrf_split(cudaStream_t st, int64_t n, double* a, int32_t* ipiv, DevStatus* status, int block_index,
                  int64_t h, cudaEvent_t right_ready);
// Solve A X = B with the dgetrf factors, B is n x nrhs (ld ldb), in place.
void dgetrs(cudaStream_t st, int64_t n, int64_t nrhs, const double* lu, const int32_t* ipiv,
            double* b, int64_t ldb, double* work);
void check_finite(cudaStream_t st, const double* a, int64_t count, DevStatus* status);
// From the dgetrf factors: perm (n, source row of each row after the interchanges) and the
// inverses of the 64x64 diagonal blocks of L and U (dinv: cdiv(n,64) * 2 * 64 * 64).
void getrs_prepare(cudaStream_t st, int64_t n, const double* lu, const int32_t* ipiv, int32_t* perm,
                   double* dinv);
// x = beta*x + alpha * A^{-1} b with the dgetrf factors: chains of 8 columns, one launch
// (plus one for a remainder).  b and x must not alias.  yz: getrs_chain_scratch(n, nrhs)
// doubles, set up once by getrs_chain_init; epoch: 1, 2, 3, ... on consecutive calls that
// share yz (stream-ordered).
inline int64_t getrs_chain_scratch(int64_t n, int64_t nrhs) { return 2 * 16 * n * ((nrhs + 7) / 8); }
void getrs_chain_init(cudaStream_t st, int64_t n, int64_t nrhs, double* yz);
void getrs_chain(cudaStream_t st, int64_t n, int64_t nrhs, const double* lu, const double* dinv,
                 const int32_t* perm, const double* b, int64_t ldb, double* x, int64_t ldx, double alpha,
                 double beta, double* yz, int epoch, DevStatus* status);

// ---- solve.cu ---------------------------------------------------------------------

// y = beta*y + alpha * A x  (A m x n col-major, x n x nrhs); part: 8*m*nrhs scratch
void dgemv_batched_rhs(cudaStream_t st, int64_t m, int64_t n, int64_t nrhs, double alpha,
                       const double* A, int64_t lda, const double* x, int64_t ldx, double beta,
                       double* y, int64_t ldy, double* part);
void dset_identity(cudaStream_t st, double* a, int64_t n);

// ---- hbs.cu ------------------------------------------------------------------
// Randomized HBS compression of dense blocks (hbs_compress.hpp:90-311).
struct HbsOptions {
  double tol = 1e-11;        // probe tolerance (SolverConfig.hbs_tol)
  double trunc_rel = 1e-13;  // generator truncation floor (SolverConfig.hbs_trunc_rel)
  int leaf = 64;             // cluster-tree leaf size
  int64_t r_start = 0, r_max = 0;
  bool fixed_rank = false;   // hbs_compress with rank bound r_max instead of the adaptive loop
};
struct HbsStats {
  int64_t products_normal = 0, products_adjoint = 0;
  int rounds = 0;
  int64_t final_rank = 0;
  double residual = 0.0;
};
// Each of the nb dense n x n blocks (device, column major, ld n) is replaced in place by the
// dense materialization of its HBS approximation; seeds[i] = the block's CompressOptions.seed.
// Throws HostError (SLABLU_ERR_COMPRESSION with the residual, or SLABLU_ERR_CONFIG).
void hbs_compress_blocks(cudaStream_t st, int64_t n, int nb, double* const* blocks, const uint64_t* seeds,
                         const HbsOptions& o, HbsStats* stats);
struct HbsFootprint {
  double per_block, densify;  // bytes
};
HbsFootprint hbs_footprint(int64_t n, const HbsOptions& o);

}  // namespace slb
