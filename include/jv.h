/*
 * jv.h — C-ABI of the B200-native ILU / stri / spmv library (libjv.so).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `ilukit` (/root/reference/pkg/src/ilukit).  The reference's own seam is the
 * L3 -> L0 call from a Python wrapper into a numba kernel that takes flat
 * int64/float64 arrays plus scalars and mutates outputs in place
 * (SURVEY.md §1, §8b).  Each entry point below replaces one such kernel (or
 * a fused group); the replaced reference symbol is cited beside it.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless the name ends in `_h`.
 *  - Structure arrays are int32 (n, nnz < 2^31; the Python shim checks),
 *    values are IEEE binary64.
 *  - Every call is asynchronous on the caller's `stream` (a cudaStream_t
 *    passed as void*), never synchronises unless documented, and returns
 *    0 on success or a negative JV_E* code; jv_last_error() describes the
 *    last failure of the calling thread.
 *  - Error rows (zero pivot, missing diagonal) are reported through a
 *    DEVICE int32 slot that the kernels atomicMin into; the caller
 *    initialises it to INT32_MAX (jv_reset_row) and maps a final value
 *    < INT32_MAX to ZeroPivotError(row) / MissingDiagonalError(row), exactly
 *    as the reference raises the smallest bad row after its workers
 *    quiesce (factor.py:61-63, trisolve.py:54-57, symbolic.py:70-75).
 *  - Sync-free kernels need a per-plan `epoch` (uint32, strictly increasing
 *    per call on the same mailbox) so mailboxes never need clearing.
 */
#ifndef JV_H
#define JV_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  JV_OK = 0,
  JV_EINVAL = -1,     /* bad argument */
  JV_ECUDA = -2,      /* CUDA runtime error */
  JV_ENOMEM = -3,     /* workspace too small / allocation failed */
  JV_ECOOP = -4       /* cooperative launch not possible */
};

/* ---- context ---------------------------------------------------------- */
const char* jv_last_error(void);
int jv_version(void);
/* page-lock a caller's host buffer in place / release it; async copies on a
 * stream (kind 0 host->device, 1 device->host): the drop-in API's transfers */
int jv_host_register(void* ptr, int64_t bytes);
int jv_host_unregister(void* ptr);
int jv_memcpy_async(void* dst, const void* src, int64_t bytes, int kind, void* stream);
/* number of SMs and the persistent grid each sync-free kernel uses */
int jv_device_info(int device, int* sms_h, int* coop_h);
/* *row = INT32_MAX */
int jv_reset_row(int32_t* row, void* stream);

/* 1 in *hang_h if a sync-free wait gave up because a producer never
 * published (a schedule bug, never expected); clears it.  Synchronises. */
int jv_status(int* hang_h);
/* probes a single sync-free wait may spend before it gives up and flags
 * jv_status (default 2^26, ~10 s): a guard against schedule bugs. */
int jv_set_spin_limit(unsigned limit);
/* cap (ns) of the exponential __nanosleep backoff of the warp gates that
 * sync-free kernels use before touching their own mailbox packets
 * (default 64; 0 = busy poll). */
int jv_set_backoff(unsigned cap_ns);
/* which sync-free kernels wait at that gate (bit 0: factor, bit 1: forward
 * and backward solves; default 0: measured faster on configs 1, 2, 4).
 * Without it the converged probe loops wait on every needed packet
 * directly, with their own backoff capped at jv_set_poll (default 32 ns,
 * min 16). */
int jv_set_gate(unsigned mask);
int jv_set_poll(unsigned cap_ns);
/* lanes of a factor thread batch that wait and finish together (power of
 * 2, <= 32; default 32) */
int jv_set_sfp_group(unsigned g);
/* solve thread path: dependencies staged by cp.async in two round trips (1)
 * or probed in register rounds of 12 (0, default: measured faster) */
int jv_set_solve_staged(unsigned on);
/* diagnostics: record 4 globaltimer stamps per factor batch into buf
 * (device, 16*batches uint64; NULL disables) */
int jv_set_trace(unsigned long long* buf, long long batches);
/* test hook: out = a / b through the kernels' batched fast division */
int jv_test_ddiv(int32_t n, const double* a, const double* b, double* out, void* stream);

/* ---- spmv: y = A x ---------------------------------------------------
 * replaces _kernels.py:28-34 spmv_kernel (called by csr.py:251-260 spmv).
 * Row sums are accumulated in ascending column order without FMA, so the
 * result is bitwise equal to the reference for rows of any length.
 * Two kernels, same bits: a CTA-per-tile stream kernel (small matrices)
 * and a persistent kernel whose col/val tiles arrive by bulk copies (TMA)
 * in a shared-memory ring (from 2^20 nonzeros; col and val 16-byte
 * aligned, else its tiles are loaded directly; not for matrices with rows
 * spanning two whole tiles — power-law hubs — whose serial sums the
 * CTA-per-tile kernel spreads better: jv_spmv_plan notes that per plan
 * pointer and synchronises the stream once to do so).  jv_set_spmv_impl:
 * -1 by size and plan (default), 0 stream, 1 persistent.
 * tile_rows (nullable) is the jv_spmv_plan output, int32[2*(ntiles+1)]
 * (first row of each tile boundary and that row's first nonzero) with
 * ntiles = max(1, ceil(nnz / jv_spmv_tile())).                           */
int jv_spmv_tile(void);
int jv_set_spmv_impl(int impl);
int jv_spmv_impl_for(int32_t nnz, const int32_t* tile_rows);   /* 1 persistent, 0 stream */
int jv_spmv_plan(int32_t n, int32_t nnz, const int32_t* row_start, int32_t* tile_rows,
                 void* stream);
int jv_spmv(int32_t n, int32_t nnz, const int32_t* row_start, const int32_t* col,
            const double* val, const double* x, double* y, const int32_t* tile_rows,
            void* stream);
/* Row-mapped variant for the multi-GPU interior/boundary split: CSR row r is
 * written to y[row_map[r]] (row_map nullable = identity).                  */
int jv_spmv_rows(int32_t n, int32_t nnz, const int32_t* row_start, const int32_t* col,
                 const double* val, const double* x, double* y, const int32_t* tile_rows,
                 const int32_t* row_map, void* stream);
/* dst[i] = src[idx[i]], i < n — packs the halo entries a peer needs.      */
int jv_gather(int32_t n, const int32_t* idx, const double* src, double* dst, void* stream);
/* Batches of independent systems (config 5) are stored as ONE
 * block-diagonal CSR (column indices offset by each block's first row), so
 * every entry point below serves them unchanged and the level schedule of
 * the block-diagonal matrix interleaves all blocks automatically. */

/* ---- vector kernels of the device Krylov driver (krylov.py) -----------
 * replace the numpy vector ops of krylov.py:52-151 (pcg / gmres).  Dot
 * products are deterministic (fixed grid of partial sums, summed in order);
 * ws = device workspace of jv_dot_workspace() doubles; out / rr device
 * scalars.  Updates are explicitly rounded (no FMA), as numpy's.        */
int jv_dot_workspace(void);
int jv_dot(int64_t n, const double* x, const double* y, double* ws, double* out, int sqrt_out,
           void* stream);
/* y += a*x, with a = sign * (*coef_dev) when coef_dev is not NULL */
int jv_axpy(int64_t n, double a, const double* coef_dev, double sign, const double* x, double* y,
            void* stream);
int jv_xpby(int64_t n, const double* x, double b, double* y, void* stream);   /* y = x + b y */
int jv_scale(int64_t n, double a, const double* x, double* y, void* stream);  /* y = a x */
/* PCG step (krylov.py:72-79): x += alpha p ; r -= alpha ap ; *rr = r.r */
int jv_pcg_update(int64_t n, double alpha, const double* p, const double* ap, double* x,
                  double* r, double* ws, double* rr, void* stream);

/* ---- setup (bit-exact structure) ------------------------------------- */
/* Longest-path depth over the columns < r of each row (forward,
 * _kernels.py:37-48, whose input is already strictly lower) or the columns
 * > r swept backward (_kernels.py:51-62).  level_of: int32[n].  ws:
 * uint64[n] mailbox.
 * `*nlev_h` receives max level + 1 (this call synchronises the stream). */
int jv_levels(int backward, int32_t n, const int32_t* row_start, const int32_t* col,
              int32_t* level_of, uint64_t* ws, uint32_t epoch, int32_t* nlev_h,
              void* stream);
/* Stable counting sort by level (= np.argsort(level_of, kind="stable"),
 * ordering.py:86-94): order[n] and level_ptr[nlev+1] (int32). */
int jv_level_sort(int32_t n, int32_t nlev, const int32_t* level_of, int32_t* order,
                  int32_t* level_ptr, void* stream);
/* Partition rule (ordering.py:119-159) over levels given as level_ptr/order
 * with integer row nnz; results to host: cut level, n_upper. */
int jv_partition(int32_t n, int32_t nlev, const int32_t* level_ptr, const int32_t* order,
                 const int32_t* row_nnz, int32_t min_level_rows, double density_factor,
                 int suffix_only, int32_t* cut_h, int32_t* n_upper_h, void* stream);
/* Transpose (csr.py:203-211): out arrays sized n+1/nnz.  t_pos (nullable)
 * receives, per transposed entry, its source position, so values follow as
 * t_val[k] = val[t_pos[k]].  Stable: rows ascend within each column. */
int jv_transpose_pattern(int32_t n, const int32_t* row_start, const int32_t* col,
                         int32_t* t_row_start, int32_t* t_col, int32_t* t_pos, void* stream);
/* Pattern of A ∪ Aᵀ then strict lower, fused (csr.py:214-235).  Two-phase:
 * call with out_col == NULL to get *nnz_h (synchronises), then again. */
int jv_sym_lower(int32_t n, const int32_t* row_start, const int32_t* col,
                 const int32_t* t_row_start, const int32_t* t_col, int lower_only,
                 int32_t* out_row_start, int32_t* out_col, int64_t* nnz_h, void* stream);
/* B[inv[i], inv[j]] = A[i, j] with sorted rows (csr.py:238-243); val may be
 * NULL for patterns.  out arrays sized like the input. */
int jv_permute_symmetric(int32_t n, const int32_t* row_start, const int32_t* col,
                         const double* val, const int32_t* perm, const int32_t* inv,
                         int32_t* out_row_start, int32_t* out_col, double* out_val,
                         void* stream);
/* First row without a stored diagonal -> *row (atomicMin). symbolic.py:70-75 */
int jv_check_diagonal(int32_t n, const int32_t* row_start, const int32_t* col,
                      int32_t* row, void* stream);
/* ILU(1) fill pattern = A ∪ pattern(strict_lower(A)·strict_upper(A)) with
 * fill level 0/1 (symbolic.py:86-138 at k = 1).  Two-phase like
 * jv_sym_lower; out_lev may be NULL. */
int jv_iluk1_pattern(int32_t n, const int32_t* row_start, const int32_t* col,
                     int32_t* out_row_start, int32_t* out_col, int32_t* out_lev,
                     int64_t* nnz_h, void* stream);
/* ILU(k >= 2): one round of the level-of-fill closure on a levelled pattern
 * (symbolic.py:86-138): every strict-lower entry (m, a) of row i with every
 * strict-upper entry (j, b) of row m gives (j, a + b + 1) when that is <= K;
 * per column the smallest level wins.  K rounds from (A, level 0) give the
 * reference's ILU(K) pattern and level table.  Two-call protocol like
 * jv_iluk1_pattern (out_col NULL: only out_row_start and *nnz_h).          */
int jv_iluk_round(int32_t n, const int32_t* row_start, const int32_t* col, const int32_t* lev,
                  int32_t K, int32_t* out_row_start, int32_t* out_col, int32_t* out_lev,
                  int64_t* nnz_h, void* stream);
/* Values of the (already permuted) matrix into the factor pattern; fill
 * positions start at 0; diag_pos found; uncovered entries -> *bad_cover,
 * missing diagonals -> *bad_diag (both atomicMin rows).  symbolic.py:146-181 */
int jv_assemble(int32_t n, const int32_t* a_row_start, const int32_t* a_col,
                const double* a_val, const int32_t* f_row_start, const int32_t* f_col,
                double* f_val, int32_t* diag_pos, int32_t* bad_cover, int32_t* bad_diag,
                void* stream);
/* Row inf-norms of the assembled values, zeros when tau == 0 (factor.py:25) */
int jv_row_norms(int32_t n, const int32_t* row_start, const double* val, double tau,
                 double* norms, void* stream);
/* Host-side RCM (ordering.py:199-266) on a symmetrized int32 pattern (host
 * arrays).  Setup only; a device version is the next item. */
/* Reverse Cuthill-McKee on the device (reference ordering.py:199-266,
 * bit-exact with jv_rcm_host): symmetrized pattern on the device, perm
 * (new -> old) written on the device.  Returns 1 (nothing written) when the
 * graph has more than max_components components of >= 2 vertices: the
 * level-synchronous traversal would be launch-bound, use jv_rcm_host. */
int jv_rcm_device(int32_t n, const int32_t* row_start, const int32_t* col, int32_t* perm,
                  int32_t max_components, int32_t* ncomp_h, void* stream);
int jv_rcm_host(int32_t n, const int32_t* row_start_h, const int32_t* col_h, int32_t* perm_h);
/* Host-side level-of-fill ILU(k) for k >= 2 (symbolic.py:86-138); outputs
 * malloc'd (free with jv_free_host); returns nnz or < 0.  k = 1 is device. */
int64_t jv_iluk_host(int32_t n, const int32_t* row_start_h, const int32_t* col_h, int32_t k,
                     int32_t** out_row_start_h, int32_t** out_col_h, int32_t** out_lev_h);
void jv_free_host(void* p);
/* Hub-row gather plan (host; see host.cpp): the target-parallel schedule of
 * one heavy row's elimination list (piv_ptr[nL+1] absolute offsets of each
 * pivot's ops, op_q/op_w indexed from piv_ptr[0]; dslot[nL] = mailbox slot
 * of each pivot's diagonal).  stream: int32[2*(nops + nL)], meta:
 * int32[1 + 33*(nL + 2)] upper bounds; returns 0 or -1.                  */
int jv_hub_plan_host(int32_t len, int32_t nL, const int64_t* piv_ptr, const int32_t* op_q,
                     const int32_t* op_w, const int32_t* dslot, int32_t* stream,
                     int64_t* nstream, int32_t* meta, int64_t* nmeta);

/* ---- numeric factorization ------------------------------------------
 * Sync-free up-looking ILU(k,tau) over rows taken in `order` (a
 * topological order of the factor DAG cut into batches that never hold
 * two dependent rows: batch_ptr[nbatch+1] indexes order).  Bitwise equal
 * to factor_serial (_kernels.py:197-204): per-row elimination in ascending
 * pivot order, no FMA.  Replaces factor_serial_kernel, factor_p2p_kernel,
 * factor_er_kernel, factor_corner*_kernel and factor_sr_kernel
 * (_kernels.py:197-343): the upper/lower split changes the schedule, never
 * the arithmetic.  `mbox`: 16-byte mailbox per stored position (nnz*2
 * uint64).  `err_row`: min zero-pivot row.  `ticket`: two int32 words,
 * zero before the first call; batches are claimed through them in order and
 * the kernel leaves them zero again.                                      */
int jv_factor(int32_t n, const int32_t* row_start, const int32_t* col, double* val,
              const int32_t* diag_pos, const double* norms, double tau, int milu,
              const int32_t* order, const int32_t* batch_ptr, int32_t nbatch,
              int32_t ready_below, uint64_t* mbox, uint32_t epoch, int32_t* err_row,
              int32_t* ticket, const int8_t* heavy, const int64_t* elim_ptr,
              const int32_t* elim, const int8_t* batch_class, const int32_t* hub_stream,
              const int64_t* hub_sptr, const int32_t* hub_meta, const int64_t* hub_mptr,
              void* stream);
/* hub_* (nullable): gather plans of the rows flagged 4 in `heavy`
 * (jv_hub_plan_host, concatenated): hub_sptr[r] / hub_mptr[r] = offsets of
 * row r's stream entries (int2) and meta.  Used for full factorizations
 * with tau = 0 and no MILU; otherwise those rows take the heavy path.     */
/* batch_class (nullable): class of each batch of the schedule (0: up to 32
 * thread-path rows, 1: a pair of listed warp rows, 2: one warp row), i.e.
 * key % 3 of its first row under jv_build_schedule_n(nclass 3).          */
/* `ready_below`: rows with index < ready_below were factored by an earlier
 * call (the upper stage before the lower-tail call, lower.py:273-318) and are
 * read from val directly instead of the mailbox. */

/* ---- triangular solves -----------------------------------------------
 * forward (which=0): y = L^-1 b, unit L (_kernels.py:348-357);
 * backward (which=1): x = U^-1 y (_kernels.py:360-366).  Same sync-free
 * machinery; order/batch_ptr as in jv_factor for the solve's own DAG
 * (backward: rows of higher index first).  in and out may alias.
 * `mbox`: 16 bytes per row.  The backward diagonal check
 * (trisolve.py:54-57) is jv_check_zero_diag.                              */
int jv_solve(int which, int32_t n, const int32_t* row_start, const int32_t* col,
             const double* val, const int32_t* diag_pos, const int32_t* order,
             const int32_t* batch_ptr, int32_t nbatch, const double* in, double* out,
             uint64_t* mbox, uint32_t epoch, int32_t* ticket, void* stream);
/* ready_below analogue for solves is not needed: every solve path of the
 * reference (serial, csrls, ls, ls_lower; trisolve.py:60-182) produces the
 * same bits, so one sync-free sweep serves all of them. */
/* one level of the paper's CSR-LS baseline stri (trisolve.py:74-108):
 * rows order[lo:hi] of one level, thread per row, reference order; the host
 * launches the levels back to back (a CUDA graph) */
int jv_solve_level(int which, const int32_t* row_start, const int32_t* col, const double* val,
                   const int32_t* diag_pos, const int32_t* order, int32_t lo, int32_t hi,
                   const double* in, double* out, void* stream);
int jv_check_zero_diag(int32_t n, const double* val, const int32_t* diag_pos,
                       int32_t* row, void* stream);
/* Small systems: one sweep in ONE thread block with the vector, the sweep's
 * dependency entries, the diagonal and the level lists all in shared memory;
 * levels separated by __syncthreads, thread per row, the reference chain
 * (_kernels.py:348-366) — bitwise the other solve paths.  order: rows sorted
 * by level of the sweep's DAG; lptr[nlev + 1]: level bounds in it;
 * estart[n + 1]: prefix sum of the rows' dependency counts (forward: strict-
 * lower entries, backward: strict-upper), nent = estart[n]; width: rows of
 * the largest level (narrow levels run with fewer warps).  Fits when
 * jv_solve_small_bytes(...) <= jv_solve_small_max().                        */
int64_t jv_solve_small_bytes(int which, int32_t n, int32_t nlev, int64_t nent);
int64_t jv_solve_small_max(void);
int jv_solve_small(int which, int32_t n, const int32_t* row_start, const int32_t* col,
                   const double* val, const int32_t* diag_pos, const int32_t* order,
                   const int32_t* lptr, int32_t nlev, const int32_t* estart, int64_t nent,
                   int32_t width, const double* in, double* out, void* stream);
/* schedule builder: cut every level of a level_sort result into batches of
 * at most 32 rows (one warp; rows of a batch never depend on each other).
 * batch_ptr sized >= n/32 + nlev + 1; *nbatch_h returned (synchronises). */
int jv_build_batches(int32_t nlev, const int32_t* level_ptr, int32_t* batch_ptr,
                     int32_t* nbatch_h, void* stream);
/* Elimination lists (setup, once per pattern): the structural matches of
 * every pivot of a row — what _factor_row (_kernels.py:165-194) finds by
 * search — precomputed so the numeric kernel does no searching.
 * Rows with pivots get a list when their candidate count
 * sum_k min(|U(c_k)|, entries after k) exceeds min_cand (MILU: sum |U(c_k)|)
 * or, with cls (nullable: jv_classify_factor classes), when they are
 * warp-path rows.  A listed row is heavy (flag 2, the power-law path) when
 * one of its 32-pivot chunks holds more than 256 ops (the warp op list) —
 * or always when min_cand < 256 (diagnostic setting); otherwise flag 1 (the
 * warp path reads its op list instead of searching): 1 when the row is
 * also pairable (length <= 64, no pivot with more than 160 ops: two such
 * rows of one level share a warp, a half each), else 3.  Thread-path
 * rows (cls 0) get none (flag 0).  heavy[n] (int8) holds the flags;
 * elim_ptr[nnz+1] gives each strict-lower entry p of a listed row its ops
 * [elim_ptr[p], elim_ptr[p+1]) (0-length for every other entry);
 * elim[2*nops] holds (q, w) pairs: q = index of the matching U entry of the
 * pivot row, w = target position in the row (MILU: w = diag offset | 1<<30
 * for an out-of-pattern q), ascending.  Call with elim = NULL to get
 * *nops_h (synchronises), then again to fill.  jv_factor takes (heavy,
 * elim_ptr, elim) or three NULLs.                                          */
int jv_elim_lists(int32_t n, const int32_t* row_start, const int32_t* col,
                  const int32_t* diag_pos, int milu, int64_t min_cand, const int32_t* cls,
                  int8_t* heavy, int64_t* elim_ptr, int32_t* elim, int64_t* nops_h, void* stream);

/* Class-aware schedule used by jv_factor / jv_solve: rows (nullable = 0..m-1)
 * stably sorted by key = 2*level + class; class-0 rows of a level go 32 to a
 * batch (thread path), class-1 rows one per batch (warp path).
 * order[m], batch_ptr sized >= m + nkeys + 1; *nbatch_h (synchronises). */
int jv_build_schedule(int32_t m, const int32_t* rows, const int32_t* keys, int32_t nkeys,
                      int32_t* order, int32_t* batch_ptr, int32_t* nbatch_h, void* stream);
/* General form: key = nclass * level + class (nclass <= 4), class c rows
 * `steps[c]` (host array) to a batch.  jv_build_schedule = nclass 2, steps
 * {32, 1}; the factor uses nclass 3, steps {32, 2, 1} (thread rows, pairs
 * of listed warp rows, single warp rows).                                */
int jv_build_schedule_n(int32_t m, const int32_t* rows, const int32_t* keys, int32_t nkeys,
                        int32_t nclass, const int32_t* steps, int32_t* order, int32_t* batch_ptr,
                        int32_t* nbatch_h, void* stream);
/* row classes: factor (thread path iff <= 8 entries, <= 4 pivots, pivots'
 * U rows <= 4 entries, no MILU) and solve (thread path iff <= 32 deps) */
int jv_classify_factor(int32_t n, const int32_t* row_start, const int32_t* col,
                       const int32_t* diag_pos, int milu, int32_t* cls, void* stream);
int jv_classify_solve(int which, int32_t n, const int32_t* row_start, const int32_t* diag_pos,
                      int32_t* cls, void* stream);

/* ---- CTA-resident region kernels (csrc/region.cu, regions_host.cpp) ---
 * One co-resident CTA per region of an acyclic box-like partition of the
 * lower DAG; in-region dependencies through shared memory, cross-region
 * ones through the 16-byte mailboxes.  Same results as the ticket kernels
 * (bitwise).  Setup on the host:
 *   jv_region_partition_host  region id per row (returns #regions or -1);
 *   jv_rstream_build          wave stream of one direction (kind 0 factor of
 *                             a stencil-class matrix, 1 forward, 2 backward);
 *                             sizes[13] = {static bytes, waves, nreg,
 *                             slot ring, max_waves, S, D, CS, CD, remote
 *                             deps, packed values, packed vector,
 *                             most rows in a wave};
 *                             returns a handle > 0, -1 (a row does not
 *                             qualify) or -2 (shared memory too small);
 *   jv_rstream_export         copies the stream out and frees the handle.
 * jv_region_run replaces factor_serial_kernel (_kernels.py:197-204) for
 * kind 0 and the solve kernels (_kernels.py:348-366) for kinds 1/2. */
int32_t jv_region_partition_host(int32_t n, const int32_t* row_start_h, const int32_t* col_h,
                                 const int32_t* diag_h, int32_t nreg_max, int32_t max_rows,
                                 int32_t dims_max, int32_t* region_of_h);
int64_t jv_rstream_build(int32_t kind, int32_t n, const int32_t* row_start_h,
                         const int32_t* col_h, const int32_t* diag_h, const int32_t* region_of_h,
                         int32_t nreg, int32_t threads, int64_t smem_budget, int32_t tau_norms,
                         int64_t* sizes_h);
int jv_rstream_export(int64_t handle, int32_t* words_h, int32_t* table_h, int32_t* reg_wave_h,
                      int32_t* sidx_h, int32_t* vidx_h);
/* dst[e] = src[sidx[e]] (0 where sidx < 0): a sweep's wave-ordered values */
int jv_pack_values(int64_t m, const int32_t* sidx, const double* src, double* dst, void* stream);
/* two such gathers in one launch (either length may be 0) and, when
 * reset_row is not NULL, *reset_row = "no row": what runs in front of a
 * region sweep */
int jv_pack_values2(int64_t m1, const int32_t* sidx1, const double* src1, double* dst1,
                    int64_t m2, const int32_t* sidx2, const double* src2, double* dst2,
                    int32_t* reset_row, void* stream);
int jv_region_threads(void);
/* timing diagnostics of the region kernels (results become wrong): 4 skips
 * the value bulk copies, 8 the remote-dependency waits; 0 in production */
int jv_set_region_flags(unsigned flags);
int64_t jv_region_smem_fixed(int32_t max_region, int32_t max_waves);
/* max_rows: low 16 bits = most rows in a wave (picks 128 / 256 / 512 compute
 * threads), high bits = most dependencies of a row in any wave (0 = unknown;
 * <= 3 picks the three-dependency instances) */
int jv_region_run(int32_t kind, int32_t nreg, int32_t max_rows, const void* words,
                  const int32_t* table,
                  const int32_t* reg_wave, int32_t max_region, int32_t max_waves, int32_t S,
                  int32_t D, int32_t CS, int32_t CD, double* val, const double* pack,
                  const double* vpack, double* out,
                  const double* norms, double tau, uint64_t* mbox, uint32_t epoch,
                  int32_t* err_row, void* stream);

/* ---- lower-tail two-stage factorization (a20) ------------------------
 * Replaces the reference's SR / ER lower stage (lower.py:273-318 ->
 * factor_sr_kernel _kernels.py:326-343, factor_er_kernel :221-228) and the
 * corner (factor_corner_kernel :231-240).  Rows [n_upper, n) of the
 * level-ordered factor storage; the upper rows must be factored.
 *
 * jv_tail_plan_build: pattern-only plan (device), returns a handle > 0 or a
 *   negative status.  MILU changes the update lists, tau does not.
 * jv_tail_plan_info: info[6] = {tail rows, upper-pivot L positions,
 *   updates, groups, segments, corner entries}.
 * jv_tail_upper: stage 1, every tail row eliminates its upper-stage
 *   pivots (warp per row; DIVIDE per group of independent pivots, UPDATE as
 *   a segmented reduction, one lane per target in pivot order: bitwise the
 *   reference's sequence).  norms: row inf-norms of the ORIGINAL tail
 *   values (needed when tau > 0).
 * jv_tail_corner: the corner (tail rows x columns >= n_upper) as a compact
 *   CSR (columns shifted by -n_upper) plus the storage position of each
 *   entry, for the sync-free factor of the corner and the scatter back.
 * jv_scatter: dst[idx[i]] = src[i]. */
int64_t jv_tail_plan_build(int32_t n, int32_t n_upper, const int32_t* row_start,
                           const int32_t* col, const int32_t* diag_pos, int milu, void* stream);
int jv_tail_plan_info(int64_t handle, int64_t* info_h);
int jv_tail_upper(int64_t handle, const int32_t* col, const int32_t* diag_pos, double* val,
                  const double* norms, double tau, void* stream);
int jv_tail_corner(int64_t handle, int32_t* row_start, int32_t* col, int32_t* diag_pos,
                   int32_t* pos, void* stream);
int jv_tail_plan_free(int64_t handle);
/* ---- single-CTA level-synchronous kernels (small systems, the corner) --
 * One thread block walks the levels of a sweep's DAG with __syncthreads
 * between them (no cross-SM hops): factor_serial semantics
 * (_kernels.py:165-204; thread per row, pivots ascending, updates in
 * (pivot, q) order, tau / MILU as _factor_row) and the serial sweeps
 * (_kernels.py:348-366).  Per level a precomputed program block
 * (jv_cta_program_host, from the device update lists of jv_cta_plan_build
 * exported by jv_cta_plan_export) is prefetched two levels ahead and the
 * level's row data one level ahead with cp.async.  kind: 0 factor,
 * 1 forward, 2 backward.  rb: depth of the row-data ring (2..6; the
 * program ring is 2 rb - 1 deep); maxrows: rows of the widest level (sets the
 * block width).  resident: values (factor) / the vector (solves)
 * in shared memory for the whole sweep; jv_cta_smem gives the bytes a
 * launch needs or -1 when it does not fit.  err_row: smallest zero-pivot
 * row (atomicMin).  in may equal out. */
int jv_cta_max_rows(void);
int64_t jv_cta_plan_build(int32_t n, const int32_t* row_start, const int32_t* col,
                          const int32_t* diag_pos, int milu, void* stream);
int jv_cta_plan_export(int64_t handle, int32_t* lstart_h, int64_t* off_h, int32_t* otgt_h,
                       int32_t* oq_h, int8_t* ok_h, int64_t* info_h);
int jv_cta_plan_free(int64_t handle);
int jv_cta_program_host(int kind, int32_t n, const int32_t* row_start_h, const int32_t* col_h,
                        const int32_t* diag_h, const int32_t* order_h, const int32_t* level_ptr_h,
                        int32_t nlev, const int32_t* lstart_h, const int64_t* off_h,
                        const int32_t* otgt_h, const int32_t* oq_h, const int8_t* ok_h, int milu,
                        int32_t* prog_h, int32_t* lbase_h, int64_t* sizes_h);
int64_t jv_cta_smem(int kind, int32_t n, int64_t nnz, int32_t nlev, int64_t maxblk,
                    int64_t maxstage, int resident, int rb);
int jv_cta_run(int kind, int32_t n, int64_t nnz, int32_t nlev, const int32_t* prog,
               const int32_t* lbase, int64_t maxblk, int64_t maxstage, int resident, int rb,
               int32_t maxrows, double* val,
               const double* norms, double tau, int milu, const double* in, double* out,
               int32_t* err_row, void* stream);
/* latency of one dependent cross-SM mailbox hop (ns), measured by a chain of
 * `hops` steps on consecutive SMs (synchronous; diagnostics for the bench's
 * depth x t_hop bound) */
int jv_hop_latency(int32_t hops, double* ns_per_hop_h);
int jv_scatter(int64_t n, const int32_t* idx, const double* src, double* dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* JV_H */
