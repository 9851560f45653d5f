// Microbenchmark: random fp64 gathers from an L2-resident vector (4M
// doubles, the power-law m) -- LSU loads vs TMA 1-D bulk copies (16 B per
// element) vs TMA tile::gather4 (4 x 16 B rows per op).  Question: can the
// TMA engine serve the SELL SpMV's gathers faster than the L1TEX
// wavefront rate (one 128 B line per cycle per SM)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_mb gather_mb.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}

// A: LSU gathers, lane per element, 4 in flight per lane
__global__ void k_lsu(const double* __restrict__ x, const int* __restrict__ idx, long long M, double* out) {
  double s = 0.0;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x, T = (long long)gridDim.x * blockDim.x;
  for (long long k = t; k < M; k += 4 * T) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = k + u * T < M ? __ldg(x + idx[k + u * T]) : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) s += v[u];
  }
  if (s == 12345.678) out[0] = s;
}

// C: gather4 -- each lane issues one op for 4 consecutive elements of its
// batch; D-deep per-warp ring of 32 x 64 B
template <int D>
__global__ void k_g4(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, long long M, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + warp * D;
  unsigned char* ring = sm + 1024 + (size_t)warp * D * 4096;  // 128 B-aligned op slots
  if (lane == 0) for (int q = 0; q < D; ++q) mbar_init(&bar[q], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long gw = blockIdx.x * (long long)nw + warp, GW = (long long)gridDim.x * nw;
  const long long nb = M / 128;  // batches of 128 elements
  double s = 0.0;
  int4 keep[D];
  long long b = gw;
  auto issue = [&](long long bb, int q) {
    const int4 ii = *reinterpret_cast<const int4*>(idx + bb * 128 + lane * 4);
    keep[q] = ii;
    if (lane == 0) mbar_expect(&bar[q], 32 * 64);
    __syncwarp();
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(ring + q * 4096 + lane * 128)),
        "l"(&tm), "r"(su32(&bar[q])), "r"(0), "r"(ii.x >> 1), "r"(ii.y >> 1), "r"(ii.z >> 1),
        "r"(ii.w >> 1)
        : "memory");
  };
  long long k = 0;
  for (; k < D && b + k * GW < nb; ++k) issue(b + k * GW, (int)k);
  for (long long j = 0; b + j * GW < nb; ++j) {
    const int q = (int)(j % D);
    mbar_wait(&bar[q], (uint32_t)((j / D) & 1));
    const double* r = reinterpret_cast<const double*>(ring + q * 4096 + lane * 128);
    const int4 ii = keep[q];
    s += r[0 + (ii.x & 1)] + r[2 + (ii.y & 1)] + r[4 + (ii.z & 1)] + r[6 + (ii.w & 1)];
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (b + (j + D) * GW < nb) issue(b + (j + D) * GW, q);
  }
  if (s == 12345.678) out[0] = s;
}

// B: 1-D bulk copies, 16 B per element, one per lane per batch
template <int D>
__global__ void k_b1(const double* __restrict__ x, const int* __restrict__ idx, long long M, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + warp * D;
  unsigned char* ring = sm + 1024 + (size_t)warp * D * 512;
  if (lane == 0) for (int q = 0; q < D; ++q) mbar_init(&bar[q], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long gw = blockIdx.x * (long long)nw + warp, GW = (long long)gridDim.x * nw;
  const long long nb = M / 32;
  double s = 0.0;
  int keep[D];
  auto issue = [&](long long bb, int q) {
    const int i = idx[bb * 32 + lane];
    keep[q] = i;
    if (lane == 0) mbar_expect(&bar[q], 32 * 16);
    __syncwarp();
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                     su32(ring + q * 512 + lane * 16)),
                 "l"(x + (i & ~1)), "r"(su32(&bar[q]))
                 : "memory");
  };
  for (long long k = 0; k < D && gw + k * GW < nb; ++k) issue(gw + k * GW, (int)k);
  for (long long j = 0; gw + j * GW < nb; ++j) {
    const int q = (int)(j % D);
    mbar_wait(&bar[q], (uint32_t)((j / D) & 1));
    const double* r = reinterpret_cast<const double*>(ring + q * 512 + lane * 16);
    s += r[keep[q] & 1];
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (gw + (j + D) * GW < nb) issue(gw + (j + D) * GW, q);
  }
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
  const long long N = 1LL << 22, M = 50LL << 20;
  double* x; int* idx; double* out;
  CK(cudaMalloc(&x, N * 8)); CK(cudaMalloc(&idx, M * 4)); CK(cudaMalloc(&out, 8));
  std::vector<int> h(M);
  std::mt19937_64 g(7);
  for (long long k = 0; k < M; ++k) h[k] = (int)(g() % N);
  CK(cudaMemcpy(idx, h.data(), M * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(x, 0, N * 8));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CUtensorMap tm;
  cuuint64_t dims[2] = {2, (cuuint64_t)(N / 2)};
  cuuint64_t strides[1] = {16};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("tensor map encode: %d\n", (int)cr);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%-28s %8.1f us  %6.2f Ggather/s  %.2f gathers/clk/SM@1.92GHz\n", name, ms * 1e3, M / (ms * 1e6),
           M / (ms * 1e-3) / sms / 1.92e9);
  };
  for (int bpsm : {4, 8})
    timeit(bpsm == 4 ? "lsu 4x256/SM" : "lsu 8x256/SM", [&] { k_lsu<<<sms * bpsm, 256>>>(x, idx, M, out); });
  for (int thr : {256, 512, 1024}) {
    char nm[64];
    snprintf(nm, 64, "bulk16 D4 %d thr", thr);
    const size_t smb = 1024 + (size_t)(thr / 32) * 4 * 512;
    CK(cudaFuncSetAttribute(k_b1<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
    timeit(nm, [&] { k_b1<4><<<sms, thr, smb>>>(x, idx, M, out); });
  }
  if (cr == CUDA_SUCCESS) {
    for (int thr : {256, 512, 1024}) {
      for (int d : {2, 4}) {
        char nm[64];
        snprintf(nm, 64, "gather4 D%d %d thr", d, thr);
        const size_t smb = 1024 + (size_t)(thr / 32) * d * 4096;
        if (smb > 227 * 1024) continue;
        if (d == 2) {
          CK(cudaFuncSetAttribute(k_g4<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
          timeit(nm, [&] { k_g4<2><<<sms, thr, smb>>>(tm, idx, M, out); });
        } else {
          CK(cudaFuncSetAttribute(k_g4<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
          timeit(nm, [&] { k_g4<4><<<sms, thr, smb>>>(tm, idx, M, out); });
        }
      }
    }
  }
  return 0;
}
