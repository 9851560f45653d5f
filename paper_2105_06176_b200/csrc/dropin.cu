// dropin.cu -- one-call host-buffer entry point (pipecg_b200_solve_host).
//
// This is the C-ABI form of the reference's pipecg_solve(A, b, x0, pc, cfg)
// (solvers.py:324-387) for callers that hold the reference's host layout:
// int64 row offsets / column indices and float64 values (sparse.py:59-71).
// It uploads the CSR through the pinned transfer pipeline (hostio.cu;
// indices narrowed to int32 on the host side), solves with the autotuned
// engine and downloads x.  See INTEGRATION.md for the ctypes
// binding a maintainer of the reference would add.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>

#include "../../include/pipecg_b200.h"
#include "internal.h"

using namespace pcg;

namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  int alloc(size_t bytes) {
    return cudaMalloc(&p, bytes ? bytes : 16) == cudaSuccess ? PCG_OK
                                                            : set_error(PCG_ENOMEM, "solve_host: cudaMalloc");
  }
};
}  // namespace

extern "C" int pipecg_b200_solve_host(int64_t n, const int64_t* ro_h, const int64_t* ci_h,
                                      const double* va_h, const double* b_h, const double* x0_h,
                                      const double* dinv_h, double tol, int64_t max_it,
                                      int64_t drift_k, int dot_mode, double* x_h,
                                      double* hist_h, int64_t hist_cap, int64_t* dit_h,
                                      double* dval_h, int64_t drift_cap, pcg_result* res) {
  if (n <= 0 || !ro_h || !b_h || !x0_h || !dinv_h || !x_h || !res)
    return set_error(PCG_EINVAL, "solve_host: bad arguments");
  const int64_t nnz = ro_h[n];
  const int rp64 = nnz >= (1LL << 31) ? 1 : 0;
  cudaStream_t st = nullptr;
  int rc = cuda_status(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "solve_host stream");
  if (rc) return rc;
  DevBuf rp, ci, va, dinv, b, x0;
  const size_t pad = 16;
  if ((rc = rp.alloc((n + 1 + pad) * (rp64 ? 8 : 4))) || (rc = ci.alloc((nnz + pad) * 4)) ||
      (rc = va.alloc((nnz + pad) * 8)) || (rc = dinv.alloc(n * 8)) || (rc = b.alloc(n * 8)) ||
      (rc = x0.alloc(n * 8))) {
    cudaStreamDestroy(st);
    return rc;
  }
  // pageable host arrays -> device through the pinned pipeline (hostio.cu),
  // indices narrowed to int32 on the host side
  cudaMemsetAsync((char*)va.p + nnz * 8, 0, pad * 8, st);
  cudaMemsetAsync((char*)ci.p + nnz * 4, 0, pad * 4, st);
  rc = pipecg_b200_h2d(rp.p, ro_h, n + 1, rp64 ? PCG_H2D_COPY64 : PCG_H2D_I64_TO_I32, st);
  if (!rc && nnz) rc = pipecg_b200_h2d(ci.p, ci_h, nnz, PCG_H2D_I64_TO_I32, st);
  if (!rc && nnz) rc = pipecg_b200_h2d(va.p, va_h, nnz, PCG_H2D_COPY64, st);
  if (!rc) rc = pipecg_b200_h2d(dinv.p, dinv_h, n, PCG_H2D_COPY64, st);
  if (!rc) rc = pipecg_b200_h2d(b.p, b_h, n, PCG_H2D_COPY64, st);
  if (!rc) rc = pipecg_b200_h2d(x0.p, x0_h, n, PCG_H2D_COPY64, st);
  // pad the row pointers with nnz so staged reads past the end stay in range
  for (size_t k = 0; k < pad && !rc; ++k) {
    if (rp64)
      cudaMemcpyAsync((int64_t*)rp.p + n + 1 + k, (int64_t*)rp.p + n, 8, cudaMemcpyDeviceToDevice, st);
    else
      cudaMemcpyAsync((int32_t*)rp.p + n + 1 + k, (int32_t*)rp.p + n, 4, cudaMemcpyDeviceToDevice, st);
  }
  pcg_solver* S = nullptr;
  if (!rc) {
    pcg_matrix A;
    A.n_rows = n;
    A.n_cols = n;
    A.nnz = nnz;
    A.rp64 = rp64;
    A.rowptr = rp.p;
    A.col = (const int32_t*)ci.p;
    A.val = (const double*)va.p;
    A.inv_diag = (const double*)dinv.p;
    pcg_options o;
    o.dot_mode = dot_mode;
    o.engine = 0;
    o.chunk = 0;
    o.use_graphs = 1;
    o.max_sms = 0;
    rc = cuda_status(cudaStreamSynchronize(st), "solve_host upload");
    if (!rc) rc = pipecg_b200_solver_create(&A, &o, &S);
  }
  if (!rc) rc = pipecg_b200_solver_init(S, (const double*)b.p, (const double*)x0.p, tol, max_it,
                                        drift_k, st);
  if (!rc) rc = pipecg_b200_solver_run(S, res, hist_h, hist_cap, dit_h, dval_h, drift_cap);
  if (!rc) rc = pipecg_b200_d2h(x_h, pipecg_b200_solver_x(S), n * 8, st);
  if (S) pipecg_b200_solver_destroy(S);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return rc;
}
