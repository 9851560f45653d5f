// generators.cu -- on-device stencil matrices.
//
// The reference builds its 125-point matrix on the host with a numba filler
// (kernels.py:35-61, sparse.py:347-375) under a 2 GiB cap; the 2D/3D Poisson
// configs of BASELINE.json (and the 1.5B-row sharded config) cannot be built
// on the host at all.  Here every row is generated independently on the GPU:
// its offset comes from a closed-form prefix count, so any row range (a
// shard) can be generated without a scan.  Ordering is natural x-fastest
// with ascending columns, identical to the oracle's / reference's matrices.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pipecg_b200.h"
#include "common.cuh"
#include "internal.h"

namespace pcg {

// f(c) = sum_{k<c} min(k, R)
__host__ __device__ inline long long fmin_sum(long long c, long long R) {
  if (c <= 0) return 0;
  if (c <= R + 1) return c * (c - 1) / 2;
  return R * (R + 1) / 2 + (c - R - 1) * R;
}
// span of axis coordinate c (entries along that axis, incl. itself)
__host__ __device__ inline long long span1(long long c, long long n, long long R) {
  return (c < R ? c : R) + ((n - 1 - c) < R ? (n - 1 - c) : R) + 1;
}
// S(c) = sum_{k<c} span1(k)
__host__ __device__ inline long long span_prefix(long long c, long long n, long long R) {
  return fmin_sum(c, R) + fmin_sum(n, R) - fmin_sum(n - c, R) + c;
}

struct StencilGeom {
  int kind;  // 5, 7, 27, 125
  long long n;
  long long R;
  int dims;
  bool product;  // 27/125: len = product of spans; 5/7: 1 + sum(span-1)
};

__host__ __device__ inline StencilGeom geom(int kind, long long n) {
  StencilGeom g;
  g.kind = kind;
  g.n = n;
  g.R = kind == 125 ? 2 : 1;
  g.dims = kind == 5 ? 2 : 3;
  g.product = kind == 27 || kind == 125;
  return g;
}

// number of entries in rows [0, row)
__host__ __device__ inline long long row_offset(const StencilGeom& g, long long row) {
  const long long n = g.n, R = g.R;
  if (g.dims == 2) {
    const long long iy = row / n, ix = row % n;
    const long long T1n = span_prefix(n, n, R) - n;  // sum (span-1) over a full axis
    // full rows before iy: each row n points: n + T1n (x) + n*(s(ky)-1) (y)
    long long cnt = iy * (n + T1n) + n * (span_prefix(iy, n, R) - iy);
    // points before ix in row iy
    cnt += ix + (span_prefix(ix, n, R) - ix) + ix * (span1(iy, n, R) - 1);
    return cnt;
  }
  const long long n2 = n * n;
  const long long iz = row / n2, rem = row % n2, iy = rem / n, ix = rem % n;
  const long long SN = span_prefix(n, n, R);
  if (g.product) {
    return span_prefix(iz, n, R) * SN * SN +
           span1(iz, n, R) * (span_prefix(iy, n, R) * SN + span1(iy, n, R) * span_prefix(ix, n, R));
  }
  const long long T1n = SN - n;
  long long cnt = iz * (n2 + 2 * n * T1n) + n2 * (span_prefix(iz, n, R) - iz);
  cnt += iy * (n + T1n) + n * (span_prefix(iy, n, R) - iy) + iy * n * (span1(iz, n, R) - 1);
  cnt += ix + (span_prefix(ix, n, R) - ix) + ix * (span1(iy, n, R) - 1) + ix * (span1(iz, n, R) - 1);
  return cnt;
}

__host__ __device__ inline long long total_rows(const StencilGeom& g) {
  return g.dims == 2 ? g.n * g.n : g.n * g.n * g.n;
}

template <typename RP>
__global__ void stencil_fill_kernel(StencilGeom g, long long row_begin, long long row_end,
                                    long long off0, RP* __restrict__ rp, int* __restrict__ col,
                                    double* __restrict__ val) {
  const long long n = g.n, n2 = n * n;
  const long long count = row_end - row_begin;
  for (long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x; li <= count;
       li += (long long)gridDim.x * blockDim.x) {
    const long long row = row_begin + li;
    const long long pos0 = row_offset(g, row) - off0;
    rp[li] = (RP)pos0;
    if (li == count) continue;
    long long pos = pos0;
    if (g.dims == 2) {
      const long long iy = row / n, ix = row % n;
      if (iy > 0) { col[pos] = (int)(row - n); val[pos++] = -1.0; }
      if (ix > 0) { col[pos] = (int)(row - 1); val[pos++] = -1.0; }
      col[pos] = (int)row; val[pos++] = 4.0;
      if (ix < n - 1) { col[pos] = (int)(row + 1); val[pos++] = -1.0; }
      if (iy < n - 1) { col[pos] = (int)(row + n); val[pos++] = -1.0; }
      continue;
    }
    const long long iz = row / n2, rem = row % n2, iy = rem / n, ix = rem % n;
    if (!g.product) {
      if (iz > 0) { col[pos] = (int)(row - n2); val[pos++] = -1.0; }
      if (iy > 0) { col[pos] = (int)(row - n); val[pos++] = -1.0; }
      if (ix > 0) { col[pos] = (int)(row - 1); val[pos++] = -1.0; }
      col[pos] = (int)row; val[pos++] = 6.0;
      if (ix < n - 1) { col[pos] = (int)(row + 1); val[pos++] = -1.0; }
      if (iy < n - 1) { col[pos] = (int)(row + n); val[pos++] = -1.0; }
      if (iz < n - 1) { col[pos] = (int)(row + n2); val[pos++] = -1.0; }
      continue;
    }
    const long long R = g.R;
    const long long lz = iz >= R ? -R : -iz, hz = iz + R <= n - 1 ? R : n - 1 - iz;
    const long long ly = iy >= R ? -R : -iy, hy = iy + R <= n - 1 ? R : n - 1 - iy;
    const long long lx = ix >= R ? -R : -ix, hx = ix + R <= n - 1 ? R : n - 1 - ix;
    const double diag =
        g.kind == 27 ? 26.0 : (double)((hz - lz + 1) * (hy - ly + 1) * (hx - lx + 1));
    for (long long dz = lz; dz <= hz; ++dz)
      for (long long dy = ly; dy <= hy; ++dy)
        for (long long dx = lx; dx <= hx; ++dx) {
          const long long c = row + dz * n2 + dy * n + dx;
          col[pos] = (int)c;
          val[pos++] = c == row ? diag : -1.0;
        }
  }
}

}  // namespace pcg

using namespace pcg;

extern "C" {

int pipecg_b200_stencil_shape(int kind, int64_t n, int64_t* n_rows, int64_t* nnz) {
  if (!(kind == 5 || kind == 7 || kind == 27 || kind == 125) || n < 1 || (kind == 125 && n < 5))
    return set_error(PCG_EINVAL, "stencil_shape: kind must be 5/7/27/125 (125 needs n >= 5)");
  const StencilGeom g = geom(kind, n);
  const long long N = total_rows(g);
  if (n_rows) *n_rows = N;
  if (nnz) *nnz = row_offset(g, N);
  return PCG_OK;
}

int pipecg_b200_stencil_prefix(int kind, int64_t n, int64_t row, int64_t* count) {
  int64_t N = 0;
  int rc = pipecg_b200_stencil_shape(kind, n, &N, nullptr);
  if (rc) return rc;
  if (row < 0 || row > N || !count) return set_error(PCG_EINVAL, "stencil_prefix: bad row");
  *count = row_offset(geom(kind, n), row);
  return PCG_OK;
}

int pipecg_b200_stencil_fill(int kind, int64_t n, int64_t row_begin, int64_t row_end, int rp64,
                             void* rowptr, int32_t* col, double* val, void* stream) {
  int64_t N = 0;
  int rc = pipecg_b200_stencil_shape(kind, n, &N, nullptr);
  if (rc) return rc;
  if (row_begin < 0 || row_end > N || row_begin > row_end || !rowptr || !col || !val)
    return set_error(PCG_EINVAL, "stencil_fill: bad row range or null pointer");
  if (N >= (1LL << 31)) return set_error(PCG_ERANGE, "stencil_fill: column index exceeds int32");
  const StencilGeom g = geom(kind, n);
  const long long off0 = row_offset(g, row_begin);
  const long long local_nnz = row_offset(g, row_end) - off0;
  if (!rp64 && local_nnz >= (1LL << 31))
    return set_error(PCG_ERANGE, "stencil_fill: nnz >= 2^31 needs rp64");
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = elementwise_grid(row_end - row_begin + 1);
  if (rp64)
    stencil_fill_kernel<long long><<<grid, 256, 0, st>>>(g, row_begin, row_end, off0,
                                                         static_cast<long long*>(rowptr), col, val);
  else
    stencil_fill_kernel<int><<<grid, 256, 0, st>>>(g, row_begin, row_end, off0,
                                                   static_cast<int*>(rowptr), col, val);
  return cuda_status(cudaGetLastError(), "stencil_fill launch");
}

}  // extern "C"
