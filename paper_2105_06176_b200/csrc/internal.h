// internal.h -- declarations shared by the translation units of the library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pcg {

constexpr int kNumSMs = 148;               // B200
constexpr int kDotGrid = 4 * kNumSMs;      // fixed grid for deterministic dots
constexpr int64_t kGridCap = 64 * kNumSMs; // grid-stride cap for row kernels
constexpr int64_t kLongRow = 256;          // rows longer than this use the block path

int set_error(int code, const char* what);

// Setup-time device allocations come from the device's stream-ordered pool
// (cudaMallocAsync on the solver's stream, set for the calling thread with
// AllocStream): creating and destroying solvers call after call (the
// reference-facing API builds one per matrix) then costs no cudaMalloc /
// cudaFree round trips.  Memory exported over CUDA IPC stays on cudaMalloc.
struct AllocStream {
  explicit AllocStream(cudaStream_t st);
  ~AllocStream();
  cudaStream_t prev;
};
cudaError_t pool_malloc_bytes(void** p, size_t bytes);
template <typename T>
inline cudaError_t pool_malloc(T** p, size_t bytes) {
  return pool_malloc_bytes(reinterpret_cast<void**>(p), bytes);
}
void pool_free(void* p);
void pool_init();  // once per device: keep up to 2 GB cached in the pool
int cuda_status(cudaError_t e, const char* where);

inline unsigned elementwise_grid(int64_t n) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > kGridCap) blocks = kGridCap;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

int spmv_any(int64_t n_rows, int rp64, const void* rowptr, const int* col, const double* val,
             const double* x, const double* b, double* y, const int* long_rows, int64_t n_long,
             int mode, cudaStream_t st);
int preload_ops();

// Row-pattern dictionary of a CSR matrix (patterns.cu): row i's entries are
// (i + off[k], val[k]) for k in [start[code[i]], start[code[i] + 1]), in
// the CSR order, bit for bit.  n_pat == 0: the matrix has no dictionary.
constexpr int kPatMax = 256;          // codes are one byte
constexpr int kPatMaxEntries = 8192;  // dictionary entries (shared memory: 16 B each; the
                                      // plans check what fits -- 125-pt: 6,859)
struct RowPatterns {
  int n_pat = 0, n_entries = 0, max_len = 0;
  unsigned char* code = nullptr;  // [n + 256]
  int* start = nullptr;           // [n_pat + 1]
  int* rep = nullptr;             // [n_pat] first row of each code
  int* off = nullptr;             // [n_entries] column - row
  double* val = nullptr;          // [n_entries]
};
int build_row_patterns(long long n, int rp64, const void* rp, const int* col, const double* val,
                       cudaStream_t st, RowPatterns* out);
void free_row_patterns(RowPatterns* p);
// pdinv[k] = dinv[rep[k]]; *ok = dinv[i] == pdinv[code[i]] bitwise for every row;
// *uniform: ok and every pdinv[k] == *value bitwise
int check_dinv_by_code(const RowPatterns& p, long long n, const double* dinv, double* pdinv,
                       bool* ok, bool* uniform, double* value, cudaStream_t st);
int preload_patterns();
int dots_any(int64_t n, int npairs, const double* const* a, const double* const* b, int mode,
             double* out, double* workspace, cudaStream_t st);

}  // namespace pcg
