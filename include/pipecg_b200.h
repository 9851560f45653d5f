/*
 * pipecg_b200.h -- C ABI of the B200-native PIPECG solve path.
 *
 * Drop-in boundary for the reference package `pipecg`
 * (/root/reference/pkg/src/pipecg).  The reference has no FFI of its own: its
 * Python functions call numba-compiled loops directly.  Each entry point
 * below replaces one of those calls; the citation says which.  The Python
 * mirror (paper_2105_06176_b200/) binds these with ctypes and keeps the
 * reference's names, argument meaning and exceptions; INTEGRATION.md shows
 * the binding a maintainer of the reference would add.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless the name ends in `_host`.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - Every function returns 0 on success, otherwise a PCG_E* code or a
 *     cudaError_t value (>= 1); pipecg_b200_last_error() gives the text.
 *     Nothing throws across the ABI; caller memory is never freed here.
 *   - Row pointers are int32 (rp64 = 0) or int64 (rp64 = 1); column indices
 *     are int32 (a device matrix never has >= 2^31 columns).
 *   - Arithmetic is fp64 with separate multiply/add roundings (no FMA), so
 *     every per-element / per-row result is bitwise equal to the reference.
 *     Dot products use either a deterministic block tree ("tree", fast) or
 *     the reference's strict left-to-right order ("seq", bitwise).
 */
#ifndef PIPECG_B200_H
#define PIPECG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PCG_OK = 0,
  PCG_EINVAL = 1001,    /* bad argument (shape, null, size) */
  PCG_ENOMEM = 1002,    /* device allocation failed */
  PCG_ESTATE = 1003,    /* call out of order (e.g. iterate before init) */
  PCG_ERANGE = 1004,    /* index out of int32 range / out of bounds */
  PCG_EDIAG = 1005,     /* missing or zero diagonal (jacobi_setup) */
  PCG_ECOMM = 1006,     /* distributed exchange timed out (peer stalled / died) */
  PCG_EPARSE = 1007,    /* malformed Matrix Market input (see pipecg_b200_mm_error_line) */
  PCG_EIO = 1008        /* file cannot be opened / read */
};

/* dot-product modes */
enum { PCG_DOT_TREE = 0, PCG_DOT_SEQ = 1 };

/* solver status (pcg_result.status) */
enum {
  PCG_RUNNING = 0,
  PCG_STOPPED = 1,  /* loop condition false: converged or max_iterations */
  PCG_BREAKDOWN = 2 /* SolverBreakdown raised (solvers.py:61-71) */
};
/* pcg_result.breakdown_quantity: matches SolverBreakdown.quantity */
enum { PCG_BD_NONE = 0, PCG_BD_ALPHA = 1, PCG_BD_GAMMA = 2, PCG_BD_DELTA = 3 };

const char* pipecg_b200_last_error(void);
const char* pipecg_b200_version(void);

/* ---------------------------------------------------------------------- */
/* Operators (the reference's kernels.py surface)                          */
/* ---------------------------------------------------------------------- */

/* y = A x, each row accumulated left to right in storage order.
 * Replaces kernels.py:152-164 (spmv) -> kernels.py:64-70 (_spmv).
 * long_rows (n_long entries, may be NULL) lists rows handled by the
 * warp-per-row path (deterministic tree order; used for rows > 32 nnz). */
int pipecg_b200_spmv(int64_t n_rows, int rp64, const void* rowptr, const int32_t* col,
                     const double* val, const double* x, double* y,
                     const int32_t* long_rows, int64_t n_long, void* stream);

/* r = b - A x (the two roundings of solvers.py:307 / :191). */
int pipecg_b200_residual(int64_t n_rows, int rp64, const void* rowptr, const int32_t* col,
                         const double* val, const double* x, const double* b, double* r,
                         const int32_t* long_rows, int64_t n_long, void* stream);

/* out = inv_diag * v.  Replaces kernels.py:240-247 (jacobi_apply). */
int pipecg_b200_jacobi_apply(int64_t n, const double* inv_diag, const double* v, double* out,
                             void* stream);

/* inv_diag = 1/diag(A).  Replaces kernels.py:218-237 (jacobi_setup).  On a
 * missing / zero diagonal returns PCG_EDIAG with *bad_row_host = the first
 * such row and *bad_kind_host = 1 (missing) or 2 (zero).  Synchronous. */
int pipecg_b200_jacobi_setup(int64_t n_rows, int rp64, const void* rowptr, const int32_t* col,
                             const double* val, double* inv_diag, int64_t* bad_row_host,
                             int* bad_kind_host, void* stream);

/* The eight PIPECG recurrences in one pass (z,q,s,p,x,r,u,w in place).
 * Replaces kernels.py:250-267 (fused_pipecg_update) -> :100-111. */
int pipecg_b200_fused_update(int64_t n, double* z, double* q, double* s, double* p, double* x,
                             double* r, double* u, double* w, const double* m,
                             const double* nvec, double alpha, double beta, void* stream);

/* fused_update + m = inv_diag*w + the three dots (r,u), (w,u), (u,u) in one
 * HBM pass (solvers.py:350-358 in one kernel).  dots_out: device double[3].
 * workspace: >= pipecg_b200_dots_workspace_bytes() bytes. */
int pipecg_b200_fused_update_pc_dots(int64_t n, double* z, double* q, double* s, double* p,
                                     double* x, double* r, double* u, double* w, double* m,
                                     const double* nvec, const double* inv_diag, double alpha,
                                     double beta, int dot_mode, double* dots_out,
                                     void* workspace, void* stream);

/* Up to 4 dot products sum_i a_k[i]*b_k[i] (k < npairs) -> out[k] (device).
 * Replaces kernels.py:192-201 (dot / norm2).  mode = PCG_DOT_SEQ gives the
 * reference's bitwise left-to-right order. */
int pipecg_b200_dots(int64_t n, int npairs, const double* const* a, const double* const* b,
                     int mode, double* out, void* workspace, void* stream);
int64_t pipecg_b200_dots_workspace_bytes(void);

/* int64 host-layout indices -> int32 device indices; *overflow_host = 1 if any
 * value is outside [0, 2^31).  Synchronous. */
int pipecg_b200_narrow_i64(int64_t n, const int64_t* src, int32_t* dst, int* overflow_host,
                           void* stream);

/* Host <-> device transfer pipeline for the reference's pageable host
 * arrays (csrc/hostio.cu): a pool of host threads converts chunks into a
 * pinned staging ring while earlier chunks cross PCIe on `stream`.
 * kind PCG_H2D_I64_TO_I32 narrows int64 indices (sparse.py:59-71 layout) to
 * the device's int32 (PCG_ERANGE if any value does not fit); PCG_H2D_COPY64
 * copies 8-byte elements.  h2d returns once every chunk is enqueued (the
 * source may be reused then); d2h returns when dst_host holds the data. */
enum { PCG_H2D_COPY64 = 0, PCG_H2D_I64_TO_I32 = 1 };
int pipecg_b200_h2d(void* dst_dev, const void* src_host, int64_t count, int kind, void* stream);
/* Several arrays in one pass (e.g. a CSR's row offsets, column indices and
 * values), their chunks interleaved so that host-bound narrowing overlaps
 * PCIe-bound copies; same kinds and semantics as pipecg_b200_h2d. */
int pipecg_b200_h2d_multi(int n_arrays, void* const* dst_dev, const void* const* src_host,
                          const int64_t* count, const int* kind, void* stream);
int pipecg_b200_d2h(void* dst_host, const void* src_dev, int64_t bytes, void* stream);
/* Touch every page of a freshly allocated host buffer (host threads): the
 * first-touch page faults of a new numpy array otherwise cap a following
 * pipecg_b200_d2h at ~15 GB/s (~38 GB/s into touched pages).  Run while the
 * GPU solves.  Contents become unspecified. */
int pipecg_b200_host_prefault(void* host, int64_t bytes);

/* Matrix Market ingestion (replaces sparse.py:195-326
 * parse_matrix_market / load_matrix_market).  Same accepted subset
 * (`matrix coordinate real general|symmetric`), checks, messages and
 * 1-based line numbers; PCG_EPARSE + pipecg_b200_mm_error_line() on bad
 * input.  Parsing is multi-threaded host code; mm_to_csr builds the CSR on
 * the device (stable key sort, duplicates summed in document order):
 * rowptr has n_rows+1 entries (int32, or int64 if rp64), col/val need
 * n_coo entries of capacity, *nnz_out receives the distinct count. */
typedef struct pcg_mm pcg_mm;
int pipecg_b200_mm_parse(const char* data, int64_t len, int universal_newlines, pcg_mm** out);
int pipecg_b200_mm_read(const char* path, pcg_mm** out);
int64_t pipecg_b200_mm_error_line(void);
int pipecg_b200_mm_info(const pcg_mm* m, int64_t* n_rows, int64_t* n_cols, int64_t* n_coo);
int pipecg_b200_mm_to_csr(const pcg_mm* m, int rp64, void* rowptr, int32_t* col, double* val,
                          int64_t* nnz_out, void* stream);
void pipecg_b200_mm_free(pcg_mm* m);

/* Rows with more than `threshold` entries -> long_rows (device int32[cap]);
 * *n_long_host receives the count.  Synchronous. */
int pipecg_b200_find_long_rows(int64_t n_rows, int rp64, const void* rowptr, int64_t threshold,
                               int32_t* long_rows, int64_t cap, int64_t* n_long_host,
                               void* stream);

/* Lossless row-pattern dictionary (csrc/patterns.cu; what fused variants
 * E/F read instead of the CSR): row i's entries are (i + off_k, v_k) for one
 * of *n_pat distinct lists, *n_entries entries in all.  *n_pat = 0: the rows
 * are too diverse (> 256 lists or > 8192 entries).  codes (device uint8[n_rows],
 * optional) receives each row's list index, lists numbered by first row.
 * Synchronous.  No reference counterpart (a storage format of sparse.py's CSR). */
int pipecg_b200_row_patterns(int64_t n_rows, int rp64, const void* rowptr, const int32_t* col,
                             const double* val, int64_t* n_pat, int64_t* n_entries,
                             unsigned char* codes, void* stream);

/* ---------------------------------------------------------------------- */
/* On-device problem generators                   */
/* kind: 5 = 2D 5-point, 7 = 3D 7-point, 27 = 3D 27-point (diag 26),      */
/*       125 = the reference's 125-point stencil (kernels.py:35-61).      */
/* Natural x-fastest order, ascending columns (sparse.py:350).             */
/* ---------------------------------------------------------------------- */
int pipecg_b200_stencil_shape(int kind, int64_t n, int64_t* n_rows, int64_t* nnz);
/* number of entries in rows [0, row) (closed form, 0 <= row <= n_rows) */
int pipecg_b200_stencil_prefix(int kind, int64_t n, int64_t row, int64_t* count);
/* rows [row_begin, row_end) of the matrix; rowptr is local (starts at 0),
 * columns are global.  rp64 selects the rowptr width. */
int pipecg_b200_stencil_fill(int kind, int64_t n, int64_t row_begin, int64_t row_end, int rp64,
                             void* rowptr, int32_t* col, double* val, void* stream);

/* ---------------------------------------------------------------------- */
/* Solver (solvers.py:297-387 pipecg_init + pipecg_solve)                  */
/* ---------------------------------------------------------------------- */
typedef struct pcg_solver pcg_solver;

typedef struct {
  int64_t n_rows;      /* local rows (= N on one GPU) */
  int64_t n_cols;      /* columns of the local [owned | halo] vector space */
  int64_t nnz;
  int rp64;
  const void* rowptr;  /* n_rows+1 entries, padded by >= 16 entries */
  const int32_t* col;  /* nnz entries, padded by >= 16 entries */
  const double* val;   /* nnz entries, padded by >= 16 entries */
  const double* inv_diag; /* n_cols entries (owned + halo) */
} pcg_matrix;

typedef struct {
  int dot_mode;        /* PCG_DOT_TREE (default) or PCG_DOT_SEQ */
  int engine;          /* 0 auto (autotuned for >= 64K rows), 1 fused (variant autotuned),
                          2 two-kernel, 3..9 fused variant A/B/C/D/P/E/F
                          (E/F: A/C reading the matrix's row-pattern dictionary;
                          only for matrices that have one), 10 fused-g (one
                          SELL-C-sigma kernel per iteration for irregular rows,
                          hub rows as chunks inside it) */
  int chunk;           /* iterations per CUDA-graph chunk (0 = auto) */
  int use_graphs;      /* 1 (default) or 0 (plain launches, debugging) */
  int max_sms;         /* size persistent grids for at most this many SMs (0 = all) */
} pcg_options;

typedef struct {
  int status;          /* PCG_STOPPED / PCG_BREAKDOWN / PCG_RUNNING */
  int converged;       /* final_norm < tolerance */
  int64_t iterations;
  double final_norm;
  double norm0;        /* history[0] */
  int breakdown_quantity;
  int64_t breakdown_iteration;
  double breakdown_value;
  int64_t n_history;   /* entries written to history_host */
  int64_t n_drift;     /* samples written to drift_*_host */
  int engine;          /* engine used: 2 two-kernel, 3..9 fused variant A/B/C/D/P/E/F,
                          10 fused-g */
  int64_t graph_launches;  /* iteration chunks launched (CUDA graphs, or directly) */
  double tune_ms[9];   /* autotune ms/iteration: fused A, B, C, D, P, E, F, two-kernel,
                          fused-g
                          (0 = not run) */
  int pattern_flags;   /* row-pattern dictionary in use by E/F: 1 dictionary, 2 windows,
                          4 dinv a function of the row's code, 8 ... one dinv for all rows,
                          16 deferred x update (x read + written every other iteration),
                          32 E's stages without the streamed vectors (the consumers
                          load them) */
} pcg_result;

int pipecg_b200_solver_create(const pcg_matrix* A, const pcg_options* opts, pcg_solver** out);
int pipecg_b200_solver_destroy(pcg_solver* s);

/* pipecg_init (solvers.py:297-321): x = x0, r = b - Ax, u = M^-1 r, w = Au,
 * m = M^-1 w, n = Am, gamma/delta/norm, z=q=s=p=0.  Waits on `stream`
 * before starting; the solver runs on its own stream afterwards. */
int pipecg_b200_solver_init(pcg_solver* s, const double* b, const double* x0, double tolerance,
                            int64_t max_iterations, int64_t drift_check_interval,
                            void* stream);

/* The loop of solvers.py:346-372 until the loop condition fails, a
 * breakdown occurs or the iteration budget is spent.  history_host
 * (capacity hist_cap, may be NULL) receives report.history; drift_*_host
 * receive report.drift_history.  Returns when the solve has finished. */
int pipecg_b200_solver_run(pcg_solver* s, pcg_result* res, double* history_host,
                           int64_t hist_cap, int64_t* drift_it_host, double* drift_val_host,
                           int64_t drift_cap);

/* Capture + instantiate the CUDA graphs that a following
 * pipecg_b200_solver_enqueue(s, count) will launch (both record parities),
 * so that graph construction stays out of a timed region.  Optional. */
int pipecg_b200_solver_prepare(pcg_solver* s, int64_t count);
/* Enqueue exactly `count` more iterations (no host synchronisation; used by
 * the benchmark to time a fixed number of iterations with CUDA events). */
int pipecg_b200_solver_enqueue(pcg_solver* s, int64_t count);
void* pipecg_b200_solver_stream(pcg_solver* s);
/* Poll the result after pipecg_b200_solver_enqueue (synchronises). */
int pipecg_b200_solver_poll(pcg_solver* s, pcg_result* res);
/* Forget the process-wide autotuning cache (engine / variant picked per
 * matrix shape and row profile): the next solver_create re-tunes.  Used to
 * measure a first call including its autotuning. */
void pipecg_b200_tune_cache_clear(void);

/* Device pointer of the iterate x (valid after solver_run / poll).  With the
 * row-pattern variants E/F, x is updated every other iteration (both updates
 * in order, bitwise the reference's) and is final once the solve has STOPPED
 * (convergence or max_iterations); after a solver_enqueue that ends with the
 * solve still RUNNING it may lag one update. */
double* pipecg_b200_solver_x(pcg_solver* s);

/* Device pointers of the state vectors in PipecgState field order
 * x r u w m n z q s p (solvers.py:74-101).  m and n are materialised first
 * (the fused engine keeps them implicit).  ptrs: void*[10]. */
int pipecg_b200_solver_state(pcg_solver* s, double** ptrs);

/* ---------------------------------------------------------------------- */
/* Multi-GPU row-block sharding; one process per GPU.    */
/* Each rank creates a solver for its row block with local column indices */
/* ([owned rows | halo], halo sorted by global index) and inv_diag over    */
/* n_cols entries; the ranks exchange CUDA IPC handles of their vector     */
/* block and comm block, then connect.  Per iteration the fused kernel is  */
/* followed by an exchange kernel that stores the boundary rows of w into  */
/* the neighbours' halo and this rank's dot partial into every rank's slot */
/* over NVLink, then signals; the next iteration's prologue waits on that  */
/* signal in-kernel.  No host synchronisation, no NCCL on the data path.   */
/* ---------------------------------------------------------------------- */
/* vector block base (vectors at base + k*ld, w0 = 7, w1 = 8), ld, comm block */
int pipecg_b200_solver_comm_info(pcg_solver* s, void** vbuf, int64_t* ld, void** comm);
/* cudaIpcMemHandle_t (64 bytes) of a device allocation, and its mapping */
int pipecg_b200_ipc_get_handle(void* dev_ptr, void* handle_out);
int pipecg_b200_ipc_open(const void* handle, void** dev_ptr_out);
int pipecg_b200_ipc_close(void* dev_ptr);
/* One process driving several GPUs (pipecg_solve(..., devices=[...])): let
 * `device` load/store `peer`'s memory (idempotent). */
int pipecg_b200_enable_peer_access(int device, int peer);
/* peer_*: world entries (this rank's own at [rank]); send_*: device arrays
 * of n_send entries: local row, destination rank, destination local column */
int pipecg_b200_solver_connect(pcg_solver* s, int rank, int world, void* const* peer_vbuf,
                               const int64_t* peer_ld, void* const* peer_comm, int64_t n_send,
                               const int32_t* send_row, const int32_t* send_peer,
                               const int64_t* send_dst);

/* ---------------------------------------------------------------------- */
/* One-call host-buffer drop-in for pipecg_solve (solvers.py:324-387).     */
/* Host CSR in the reference layout (int64 offsets and indices, float64).  */
/* Uploads, solves on cuda device 0 (current device), downloads x.         */
/* ---------------------------------------------------------------------- */
int pipecg_b200_solve_host(int64_t n_rows, const int64_t* row_offsets_host,
                           const int64_t* col_indices_host, const double* values_host,
                           const double* b_host, const double* x0_host,
                           const double* inv_diag_host, double tolerance,
                           int64_t max_iterations, int64_t drift_check_interval, int dot_mode,
                           double* x_host, double* history_host, int64_t hist_cap,
                           int64_t* drift_it_host, double* drift_val_host, int64_t drift_cap,
                           pcg_result* res);

#ifdef __cplusplus
}
#endif
#endif /* PIPECG_B200_H */
