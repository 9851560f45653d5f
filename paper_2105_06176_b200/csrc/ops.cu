// ops.cu -- operator kernels behind the C ABI (include/pipecg_b200.h).
//
// These are the B200 replacements of the reference's kernels.py surface:
//   spmv           kernels.py:152-164 / _spmv :64-70
//   jacobi_apply   kernels.py:240-247
//   jacobi_setup   kernels.py:218-237
//   fused update   kernels.py:250-267 / _fused_update :100-111
//   dot / norm2    kernels.py:192-201 / _dot :92-97
// plus the fused update+PC+dots kernel (solvers.py:350-358 in one pass) and
// setup helpers (index narrowing, long-row detection, stencil generators).
//
// All of them are HBM-bandwidth kernels (no tensor-core work exists on this
// path): grids are sized as a multiple of the 148 SMs, loads are coalesced,
// and reductions are deterministic fixed-order trees.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/pipecg_b200.h"
#include "common.cuh"
#include "internal.h"

namespace pcg {

thread_local std::string g_last_error;

int set_error(int code, const char* what) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s (code %d)", what, code);
  g_last_error = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return PCG_OK;
  char buf[512];
  snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
  g_last_error = buf;
  return static_cast<int>(e);
}

// ---------------------------------------------------------------------------
// SpMV: thread per row, sequential in CSR order (bitwise = _spmv) for rows
// with <= kLongRow entries; longer rows are left to spmv_long_kernel
// (one block per row, deterministic tree) when a long-row list exists.
// MODE 0: y = Ax ; MODE 1: y = b - Ax (solvers.py:307).
// ---------------------------------------------------------------------------
template <typename RP, int MODE>
__global__ void __launch_bounds__(256) spmv_rows_kernel(int64_t n_rows, const RP* __restrict__ rp,
                                                         const int* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ y,
                                                         int64_t long_threshold) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = rp[i], hi = rp[i + 1];
    if (hi - lo > long_threshold) continue;
    double acc = 0.0;
    for (int64_t k = lo; k < hi; ++k) acc = add(acc, mul(ldg_nc(val + k), ldg_nc(x + ldg_nc(col + k))));
    y[i] = MODE == 0 ? acc : sub(b[i], acc);
  }
}

template <typename RP, int MODE>
__global__ void __launch_bounds__(256) spmv_long_kernel(const int* __restrict__ rows,
                                                         const RP* __restrict__ rp,
                                                         const int* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ y) {
  __shared__ double red[8];
  const int64_t i = rows[blockIdx.x];
  const int64_t lo = rp[i], hi = rp[i + 1];
  double v[1] = {0.0};
  for (int64_t k = lo + threadIdx.x; k < hi; k += 256)
    v[0] = add(v[0], mul(ldg_nc(val + k), ldg_nc(x + ldg_nc(col + k))));
  group_sum<1, 256>(v, threadIdx.x, red, 1);
  if (threadIdx.x == 0) y[i] = MODE == 0 ? v[0] : sub(b[i], v[0]);
}

template <typename RP, int MODE>
static int spmv_launch(int64_t n_rows, const RP* rp, const int* col, const double* val,
                       const double* x, const double* b, double* y, const int* long_rows,
                       int64_t n_long, cudaStream_t st) {
  if (n_rows <= 0) return PCG_OK;
  const int64_t thr = long_rows && n_long > 0 ? kLongRow : INT64_MAX;
  int64_t blocks = (n_rows + 255) / 256;
  if (blocks > kGridCap) blocks = kGridCap;
  spmv_rows_kernel<RP, MODE><<<(unsigned)blocks, 256, 0, st>>>(n_rows, rp, col, val, x, b, y, thr);
  if (long_rows && n_long > 0)
    spmv_long_kernel<RP, MODE><<<(unsigned)n_long, 256, 0, st>>>(long_rows, rp, col, val, x, b, y);
  return cuda_status(cudaGetLastError(), "spmv launch");
}

int spmv_any(int64_t n_rows, int rp64, const void* rowptr, const int* col, const double* val,
             const double* x, const double* b, double* y, const int* long_rows, int64_t n_long,
             int mode, cudaStream_t st) {
  if (rp64) {
    auto rp = static_cast<const long long*>(rowptr);
    return mode == 0 ? spmv_launch<long long, 0>(n_rows, rp, col, val, x, b, y, long_rows, n_long, st)
                     : spmv_launch<long long, 1>(n_rows, rp, col, val, x, b, y, long_rows, n_long, st);
  }
  auto rp = static_cast<const int*>(rowptr);
  return mode == 0 ? spmv_launch<int, 0>(n_rows, rp, col, val, x, b, y, long_rows, n_long, st)
                   : spmv_launch<int, 1>(n_rows, rp, col, val, x, b, y, long_rows, n_long, st);
}

// ---------------------------------------------------------------------------
// elementwise kernels
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) jacobi_kernel(int64_t n, const double* __restrict__ d,
                                                      const double* __restrict__ v,
                                                      double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mul(d[i], v[i]);
}

// kernels.py:100-111, one element per thread-iteration, lanes in reference order
__global__ void __launch_bounds__(256) fused_update_kernel(int64_t n, double* z, double* q, double* s,
                                                            double* p, double* x, double* r,
                                                            double* u, double* w,
                                                            const double* __restrict__ m,
                                                            const double* __restrict__ nv,
                                                            double alpha, double beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = add(nv[i], mul(beta, z[i]));
    const double qi = add(m[i], mul(beta, q[i]));
    const double wi = w[i], ui = u[i];
    const double si = add(wi, mul(beta, s[i]));
    const double pi = add(ui, mul(beta, p[i]));
    z[i] = zi;
    q[i] = qi;
    s[i] = si;
    p[i] = pi;
    x[i] = add(x[i], mul(alpha, pi));
    r[i] = sub(r[i], mul(alpha, si));
    u[i] = sub(ui, mul(alpha, qi));
    w[i] = sub(wi, mul(alpha, zi));
  }
}

// fused update + m = inv_diag*w + partial dots (r,u), (w,u), (u,u)
__global__ void __launch_bounds__(256) fused_update_pc_dots_kernel(
    int64_t n, double* z, double* q, double* s, double* p, double* x, double* r, double* u,
    double* w, double* m, const double* __restrict__ nv, const double* __restrict__ d,
    double alpha, double beta, double* __restrict__ partials) {
  __shared__ double red[3 * 8];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = add(nv[i], mul(beta, z[i]));
    const double qi = add(m[i], mul(beta, q[i]));
    const double wi = w[i], ui = u[i];
    const double si = add(wi, mul(beta, s[i]));
    const double pi = add(ui, mul(beta, p[i]));
    const double xi = add(x[i], mul(alpha, pi));
    const double ri = sub(r[i], mul(alpha, si));
    const double un = sub(ui, mul(alpha, qi));
    const double wn = sub(wi, mul(alpha, zi));
    z[i] = zi;
    q[i] = qi;
    s[i] = si;
    p[i] = pi;
    x[i] = xi;
    r[i] = ri;
    u[i] = un;
    w[i] = wn;
    m[i] = mul(d[i], wn);
    acc[0] = add(acc[0], mul(ri, un));
    acc[1] = add(acc[1], mul(wn, un));
    acc[2] = add(acc[2], mul(un, un));
  }
  group_sum<3, 256>(acc, threadIdx.x, red, 1);
  if (threadIdx.x == 0) {
    partials[blockIdx.x * 4 + 0] = acc[0];
    partials[blockIdx.x * 4 + 1] = acc[1];
    partials[blockIdx.x * 4 + 2] = acc[2];
    partials[blockIdx.x * 4 + 3] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// dots: fixed kDotGrid x 256 grid-stride partials -> one-block fixed-order
// finish (deterministic, independent of the device), or a single-warp
// strictly sequential pass (bitwise = kernels.py:92-97).
// ---------------------------------------------------------------------------
struct DotPairs {
  const double* a[4];
  const double* b[4];
};

template <int NP>
__global__ void __launch_bounds__(256) dots_partial_kernel(int64_t n, DotPairs pr,
                                                            double* __restrict__ partials) {
  __shared__ double red[4 * 8];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < NP; ++k) acc[k] = add(acc[k], mul(pr.a[k][i], pr.b[k][i]));
  }
  group_sum<4, 256>(acc, threadIdx.x, red, 1);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) partials[blockIdx.x * 4 + k] = acc[k];
  }
}

// Sum `count` partial quadruples in a fixed order into out[0..3].
__global__ void __launch_bounds__(256) dots_finish_kernel(const double* __restrict__ partials,
                                                           int count, int npairs,
                                                           double* __restrict__ out) {
  __shared__ double red[4 * 8];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j = threadIdx.x; j < count; j += 256) {
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] = add(acc[k], partials[j * 4 + k]);
  }
  group_sum<4, 256>(acc, threadIdx.x, red, 1);
  if (threadIdx.x < npairs) out[threadIdx.x] = acc[threadIdx.x];
}

// Strictly sequential left-to-right sums: the warp stages 32*8 products per
// step in shared memory, lane 0 accumulates them in index order.
template <int NP>
__global__ void __launch_bounds__(32) dots_seq_kernel(int64_t n, DotPairs pr,
                                                       double* __restrict__ out) {
  constexpr int CH = 256;
  __shared__ double prod[NP][CH];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int lane = threadIdx.x;
  for (int64_t base = 0; base < n; base += CH) {
#pragma unroll
    for (int j = 0; j < CH / 32; ++j) {
      const int64_t i = base + j * 32 + lane;
#pragma unroll
      for (int k = 0; k < NP; ++k) prod[k][j * 32 + lane] = i < n ? mul(pr.a[k][i], pr.b[k][i]) : 0.0;
    }
    __syncwarp();
    if (lane == 0) {
      const int cnt = (int)((n - base) < CH ? (n - base) : CH);
      for (int j = 0; j < cnt; ++j) {
#pragma unroll
        for (int k = 0; k < NP; ++k) acc[k] = add(acc[k], prod[k][j]);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NP; ++k) out[k] = acc[k];
  }
}

int dots_any(int64_t n, int npairs, const double* const* a, const double* const* b, int mode,
             double* out, double* workspace, cudaStream_t st) {
  if (npairs < 1 || npairs > 4) return set_error(PCG_EINVAL, "dots: npairs must be 1..4");
  DotPairs pr;
  for (int k = 0; k < 4; ++k) {
    pr.a[k] = k < npairs ? a[k] : a[0];
    pr.b[k] = k < npairs ? b[k] : b[0];
  }
  if (mode == PCG_DOT_SEQ) {
    switch (npairs) {
      case 1: dots_seq_kernel<1><<<1, 32, 0, st>>>(n, pr, out); break;
      case 2: dots_seq_kernel<2><<<1, 32, 0, st>>>(n, pr, out); break;
      case 3: dots_seq_kernel<3><<<1, 32, 0, st>>>(n, pr, out); break;
      default: dots_seq_kernel<4><<<1, 32, 0, st>>>(n, pr, out); break;
    }
  } else {
    switch (npairs) {
      case 1: dots_partial_kernel<1><<<kDotGrid, 256, 0, st>>>(n, pr, workspace); break;
      case 2: dots_partial_kernel<2><<<kDotGrid, 256, 0, st>>>(n, pr, workspace); break;
      case 3: dots_partial_kernel<3><<<kDotGrid, 256, 0, st>>>(n, pr, workspace); break;
      default: dots_partial_kernel<4><<<kDotGrid, 256, 0, st>>>(n, pr, workspace); break;
    }
    dots_finish_kernel<<<1, 256, 0, st>>>(workspace, kDotGrid, npairs, out);
  }
  return cuda_status(cudaGetLastError(), "dots launch");
}

// ---------------------------------------------------------------------------
// setup helpers
// ---------------------------------------------------------------------------
template <typename RP>
__global__ void jacobi_setup_kernel(int64_t n, const RP* __restrict__ rp, const int* __restrict__ col,
                                    const double* __restrict__ val, double* __restrict__ inv_diag,
                                    unsigned long long* bad /* [0]=first missing, [1]=first zero */) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = rp[i], hi = rp[i + 1];
    bool found = false;
    double dv = 0.0;
    for (int64_t k = lo; k < hi; ++k) {
      if (col[k] == i) {
        found = true;
        dv = val[k];
        break;
      }
    }
    if (!found) {
      atomicMin(bad + 0, (unsigned long long)i);
      inv_diag[i] = 0.0;
    } else {
      if (dv == 0.0) atomicMin(bad + 1, (unsigned long long)i);
      inv_diag[i] = 1.0 / dv;  // correctly rounded division, as numpy's 1.0/diag
    }
  }
}

__global__ void narrow_kernel(int64_t n, const long long* __restrict__ src, int* __restrict__ dst,
                              int* overflow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const long long v = src[i];
    if (v < 0 || v > 0x7fffffffLL) *overflow = 1;
    dst[i] = (int)v;
  }
}

template <typename RP>
__global__ void long_rows_kernel(int64_t n, const RP* __restrict__ rp, int64_t thr, int* out,
                                 int64_t cap, unsigned long long* count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (rp[i + 1] - rp[i] > thr) {
      unsigned long long slot = atomicAdd(count, 1ull);
      if ((int64_t)slot < cap) out[slot] = (int)i;
    }
  }
}

// Force-load every operator kernel.  Under CUDA lazy module loading the
// first launch of a kernel loads it, and loading can wait for the device to
// go idle; a kernel spinning on a peer's signal would then deadlock with a
// peer whose first launch is stuck the same way.  Loading everything up front
// removes that coupling (solver_create calls this once).
int preload_ops() {
  cudaFuncAttributes a;
  cudaError_t e = cudaSuccess;
#define PCG_LOAD(k) if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void*)(k))
  PCG_LOAD((spmv_rows_kernel<int, 0>)); PCG_LOAD((spmv_rows_kernel<int, 1>));
  PCG_LOAD((spmv_rows_kernel<long long, 0>)); PCG_LOAD((spmv_rows_kernel<long long, 1>));
  PCG_LOAD((spmv_long_kernel<int, 0>)); PCG_LOAD((spmv_long_kernel<int, 1>));
  PCG_LOAD((spmv_long_kernel<long long, 0>)); PCG_LOAD((spmv_long_kernel<long long, 1>));
  PCG_LOAD(jacobi_kernel); PCG_LOAD(fused_update_kernel); PCG_LOAD(fused_update_pc_dots_kernel);
  PCG_LOAD(dots_partial_kernel<1>); PCG_LOAD(dots_partial_kernel<2>);
  PCG_LOAD(dots_partial_kernel<3>); PCG_LOAD(dots_partial_kernel<4>);
  PCG_LOAD(dots_finish_kernel);
  PCG_LOAD(dots_seq_kernel<1>); PCG_LOAD(dots_seq_kernel<2>);
  PCG_LOAD(dots_seq_kernel<3>); PCG_LOAD(dots_seq_kernel<4>);
#undef PCG_LOAD
  return cuda_status(e, "preload operator kernels");
}

}  // namespace pcg

using namespace pcg;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* pipecg_b200_last_error(void) { return pcg::g_last_error.c_str(); }
const char* pipecg_b200_version(void) { return "pipecg_b200 0.1.0 sm_100a"; }

int pipecg_b200_spmv(int64_t n_rows, int rp64, const void* rowptr, const int32_t* col,
                     const double* val, const double* x, double* y, const int32_t* long_rows,
                     int64_t n_long, void* stream) {
  if (n_rows < 0 || (n_rows > 0 && (!rowptr || !x || !y)))
    return set_error(PCG_EINVAL, "spmv: bad arguments");
  return spmv_any(n_rows, rp64, rowptr, col, val, x, nullptr, y, long_rows, n_long, 0,
                  (cudaStream_t)stream);
}

int pipecg_b200_residual(int64_t n_rows, int rp64, const void* rowptr, const int32_t* col,
                         const double* val, const double* x, const double* b, double* r,
                         const int32_t* long_rows, int64_t n_long, void* stream) {
  if (n_rows < 0 || (n_rows > 0 && (!rowptr || !x || !b || !r)))
    return set_error(PCG_EINVAL, "residual: bad arguments");
  return spmv_any(n_rows, rp64, rowptr, col, val, x, b, r, long_rows, n_long, 1,
                  (cudaStream_t)stream);
}

int pipecg_b200_jacobi_apply(int64_t n, const double* inv_diag, const double* v, double* out,
                             void* stream) {
  if (n < 0) return set_error(PCG_EINVAL, "jacobi_apply: n < 0");
  if (n == 0) return PCG_OK;
  jacobi_kernel<<<elementwise_grid(n), 256, 0, (cudaStream_t)stream>>>(n, inv_diag, v, out);
  return cuda_status(cudaGetLastError(), "jacobi_apply launch");
}

int pipecg_b200_fused_update(int64_t n, double* z, double* q, double* s, double* p, double* x,
                             double* r, double* u, double* w, const double* m, const double* nvec,
                             double alpha, double beta, void* stream) {
  if (n < 0) return set_error(PCG_EINVAL, "fused_update: n < 0");
  if (n == 0) return PCG_OK;
  fused_update_kernel<<<elementwise_grid(n), 256, 0, (cudaStream_t)stream>>>(
      n, z, q, s, p, x, r, u, w, m, nvec, alpha, beta);
  return cuda_status(cudaGetLastError(), "fused_update launch");
}

int64_t pipecg_b200_dots_workspace_bytes(void) { return (int64_t)kDotGrid * 4 * sizeof(double); }

int pipecg_b200_fused_update_pc_dots(int64_t n, double* z, double* q, double* s, double* p,
                                     double* x, double* r, double* u, double* w, double* m,
                                     const double* nvec, const double* inv_diag, double alpha,
                                     double beta, int dot_mode, double* dots_out, void* workspace,
                                     void* stream) {
  if (n < 0 || !workspace || !dots_out) return set_error(PCG_EINVAL, "fused_update_pc_dots: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  double* ws = static_cast<double*>(workspace);
  if (dot_mode == PCG_DOT_SEQ) {
    int rc = pipecg_b200_fused_update(n, z, q, s, p, x, r, u, w, m, nvec, alpha, beta, stream);
    if (rc) return rc;
    rc = pipecg_b200_jacobi_apply(n, inv_diag, w, m, stream);
    if (rc) return rc;
    const double* a[3] = {r, w, u};
    const double* b[3] = {u, u, u};
    return dots_any(n, 3, a, b, PCG_DOT_SEQ, dots_out, ws, st);
  }
  fused_update_pc_dots_kernel<<<kDotGrid, 256, 0, st>>>(n, z, q, s, p, x, r, u, w, m, nvec,
                                                        inv_diag, alpha, beta, ws);
  dots_finish_kernel<<<1, 256, 0, st>>>(ws, kDotGrid, 3, dots_out);
  return cuda_status(cudaGetLastError(), "fused_update_pc_dots launch");
}

int pipecg_b200_dots(int64_t n, int npairs, const double* const* a, const double* const* b,
                     int mode, double* out, void* workspace, void* stream) {
  if (n < 0 || !a || !b || !out || (mode != PCG_DOT_SEQ && !workspace))
    return set_error(PCG_EINVAL, "dots: bad arguments");
  return dots_any(n, npairs, a, b, mode, out, static_cast<double*>(workspace),
                  (cudaStream_t)stream);
}

int pipecg_b200_jacobi_setup(int64_t n_rows, int rp64, const void* rowptr, const int32_t* col,
                             const double* val, double* inv_diag, int64_t* bad_row_host,
                             int* bad_kind_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (bad_row_host) *bad_row_host = -1;
  if (bad_kind_host) *bad_kind_host = 0;
  if (n_rows <= 0) return PCG_OK;
  unsigned long long* bad = nullptr;
  cudaError_t e = cudaMallocAsync(&bad, 2 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return cuda_status(e, "jacobi_setup alloc");
  cudaMemsetAsync(bad, 0xff, 2 * sizeof(unsigned long long), st);
  if (rp64)
    jacobi_setup_kernel<long long><<<elementwise_grid(n_rows), 256, 0, st>>>(
        n_rows, static_cast<const long long*>(rowptr), col, val, inv_diag, bad);
  else
    jacobi_setup_kernel<int><<<elementwise_grid(n_rows), 256, 0, st>>>(
        n_rows, static_cast<const int*>(rowptr), col, val, inv_diag, bad);
  unsigned long long h[2];
  cudaMemcpyAsync(h, bad, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(bad, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e, "jacobi_setup");
  if (h[0] != ~0ull) {
    if (bad_row_host) *bad_row_host = (int64_t)h[0];
    if (bad_kind_host) *bad_kind_host = 1;
    return set_error(PCG_EDIAG, "jacobi_setup: missing diagonal entry");
  }
  if (h[1] != ~0ull) {
    if (bad_row_host) *bad_row_host = (int64_t)h[1];
    if (bad_kind_host) *bad_kind_host = 2;
    return set_error(PCG_EDIAG, "jacobi_setup: zero diagonal entry");
  }
  return PCG_OK;
}

int pipecg_b200_narrow_i64(int64_t n, const int64_t* src, int32_t* dst, int* overflow_host,
                           void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (overflow_host) *overflow_host = 0;
  if (n <= 0) return PCG_OK;
  int* flag = nullptr;
  cudaError_t e = cudaMallocAsync(&flag, sizeof(int), st);
  if (e != cudaSuccess) return cuda_status(e, "narrow alloc");
  cudaMemsetAsync(flag, 0, sizeof(int), st);
  narrow_kernel<<<elementwise_grid(n), 256, 0, st>>>(n, reinterpret_cast<const long long*>(src), dst,
                                                      flag);
  int h = 0;
  cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(flag, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e, "narrow");
  if (overflow_host) *overflow_host = h;
  return h ? set_error(PCG_ERANGE, "narrow: index outside int32 range") : PCG_OK;
}

int pipecg_b200_find_long_rows(int64_t n_rows, int rp64, const void* rowptr, int64_t threshold,
                               int32_t* long_rows, int64_t cap, int64_t* n_long_host,
                               void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *n_long_host = 0;
  if (n_rows <= 0) return PCG_OK;
  unsigned long long* cnt = nullptr;
  cudaError_t e = cudaMallocAsync(&cnt, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return cuda_status(e, "long_rows alloc");
  cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st);
  if (rp64)
    long_rows_kernel<long long><<<elementwise_grid(n_rows), 256, 0, st>>>(
        n_rows, static_cast<const long long*>(rowptr), threshold, long_rows, cap, cnt);
  else
    long_rows_kernel<int><<<elementwise_grid(n_rows), 256, 0, st>>>(
        n_rows, static_cast<const int*>(rowptr), threshold, long_rows, cap, cnt);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(cnt, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e, "long_rows");
  *n_long_host = (int64_t)h;
  return PCG_OK;
}

}  // extern "C"
