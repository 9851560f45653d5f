// patterns.cu -- lossless row-pattern dictionary of a CSR matrix (setup).
//
// The reference solves with the CSR matrix it is given (sparse.py:43-132)
// and its SpMV walks every row's (column, value) pairs in storage order
// (kernels.py:64-70).  Matrices from constant-coefficient discretisations
// -- every BASELINE config except the power-law graph -- have only a
// handful of distinct rows once a row is written relative to its own index:
// row i's entries are (i + off_k, v_k) for one of a few (off, v) lists (the
// 3D 7-point Laplacian has 27: interior, faces, edges, corners).  The fused
// pattern variants (E/F, solver.cu) then read ONE byte per row instead of
// 12 bytes per nonzero + 4 per row; each row's sum still runs over exactly
// the same (column, value) pairs in exactly the same order, so every
// rounding is the reference's.
//
// Build (all on the device, ~2 passes over the CSR):
//   1. hash each row's (length, col - i, value bits) sequence and insert the
//      hash into a small open-addressing table (kPatTable slots); remember
//      the lowest row of each slot (its representative);
//   2. on the host: order the slots by representative row -> codes
//      0..U-1 (deterministic), copy the representatives' entries into the
//      dictionary (start / off / val);
//   3. verify EVERY row against its dictionary entry bit for bit and write
//      its code byte.  Any mismatch (a hash collision) or more than
//      kPatMax patterns / kPatMaxEntries dictionary entries -> no dictionary
//      (the CSR variants run).  Correctness never depends on the hash.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/pipecg_b200.h"
#include "internal.h"

namespace pcg {
namespace {

constexpr int kPatTable = 1024;  // hash slots (power of two, > kPatMax)

__device__ __forceinline__ unsigned long long mix64(unsigned long long h, unsigned long long x) {
  h ^= x + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdULL;
  return h ^ (h >> 33);
}

template <typename RP>
__device__ unsigned long long row_hash(long long i, const RP* rp, const int* col, const double* val) {
  const long long e0 = rp[i], e1 = rp[i + 1];
  unsigned long long h = mix64(0x243f6a8885a308d3ULL, (unsigned long long)(e1 - e0));
  for (long long k = e0; k < e1; ++k) {
    h = mix64(h, (unsigned long long)(unsigned)(col[k] - (int)i));
    h = mix64(h, (unsigned long long)__double_as_longlong(val[k]));
  }
  return h | 1ULL;  // 0 marks an empty slot
}

__device__ __forceinline__ int probe(const unsigned long long* tab, unsigned long long key) {
  int s = (int)(key >> 20) & (kPatTable - 1);
  for (int p = 0; p < kPatTable; ++p, s = (s + 1) & (kPatTable - 1)) {
    const unsigned long long cur = tab[s];
    if (cur == key) return s;
    if (cur == 0) return -1;
  }
  return -1;
}

template <typename RP>
__global__ void __launch_bounds__(256) pat_hash_kernel(long long n, const RP* __restrict__ rp,
                                                       const int* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       unsigned long long* tab, int* rep, int* fail) {
  int* used = fail + 1;  // distinct keys inserted so far
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (*reinterpret_cast<volatile int*>(fail)) return;  // too diverse: give up early
    const unsigned long long key = row_hash(i, rp, col, val);
    int s = (int)(key >> 20) & (kPatTable - 1);
    int slot = -1;
    for (int p = 0; p < kPatTable; ++p, s = (s + 1) & (kPatTable - 1)) {
      unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(&tab[s]);
      if (cur == 0) {
        cur = atomicCAS(&tab[s], 0ULL, key);
        if (cur == 0 && atomicAdd(used, 1) >= kPatMax) *fail = 1;
      }
      if (cur == 0 || cur == key) {
        slot = s;
        break;
      }
    }
    if (slot < 0) {
      *fail = 1;  // table full: far more distinct rows than a dictionary holds
      continue;
    }
    // lowest row per slot; rows of one warp with the same slot combine first
    const unsigned same = __match_any_sync(__activemask(), slot);
    if ((threadIdx.x & 31) == __ffs(same) - 1 && *reinterpret_cast<volatile int*>(&rep[slot]) > i)
      atomicMin(&rep[slot], (int)i);
  }
}

template <typename RP>
__global__ void pat_len_kernel(int u, const int* reps, const RP* rp, int* len) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < u; k += gridDim.x * blockDim.x)
    len[k] = (int)(rp[reps[k] + 1] - rp[reps[k]]);
}

template <typename RP>
__global__ void pat_extract_kernel(int u, const int* reps, const RP* rp, const int* col,
                                   const double* val, const int* start, int* off, double* pv) {
  for (int k = blockIdx.x; k < u; k += gridDim.x) {
    const long long i = reps[k], e0 = rp[i];
    const int len = start[k + 1] - start[k];
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      off[start[k] + j] = col[e0 + j] - (int)i;
      pv[start[k] + j] = val[e0 + j];
    }
  }
}

template <typename RP>
__global__ void __launch_bounds__(256) pat_verify_kernel(
    long long n, const RP* __restrict__ rp, const int* __restrict__ col,
    const double* __restrict__ val, const unsigned long long* __restrict__ tab,
    const int* __restrict__ slot_code, const int* __restrict__ start, const int* __restrict__ off,
    const double* __restrict__ pv, unsigned char* code, int* fail) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = probe(tab, row_hash(i, rp, col, val));
    const int c = s < 0 ? -1 : slot_code[s];
    bool ok = c >= 0;
    if (ok) {
      const long long e0 = rp[i], e1 = rp[i + 1];
      const int p0 = start[c];
      ok = e1 - e0 == start[c + 1] - p0;
      for (long long k = e0; ok && k < e1; ++k) {
        const int j = p0 + (int)(k - e0);
        ok = col[k] - (int)i == off[j] &&
             __double_as_longlong(val[k]) == __double_as_longlong(pv[j]);
      }
    }
    if (!ok) {
      *fail = 1;
      continue;
    }
    code[i] = (unsigned char)c;
  }
}

template <typename RP>
int build(long long n, const RP* rp, const int* col, const double* val, cudaStream_t st,
          RowPatterns* out) {
  *out = RowPatterns{};
  unsigned long long* tab = nullptr;
  int *rep = nullptr, *fail = nullptr, *dev_small = nullptr;
  int rc = PCG_OK;
  if (pool_malloc(&tab, kPatTable * 8) != cudaSuccess || pool_malloc(&rep, kPatTable * 4) != cudaSuccess ||
      pool_malloc(&fail, 8) != cudaSuccess)
    rc = set_error(PCG_ENOMEM, "row patterns: workspace");
  std::vector<unsigned long long> h_tab(kPatTable);
  std::vector<int> h_rep(kPatTable);
  int h_fail = 0;
  if (!rc) {
    cudaMemsetAsync(tab, 0, kPatTable * 8, st);
    cudaMemsetAsync(rep, 0x7f, kPatTable * 4, st);
    cudaMemsetAsync(fail, 0, 8, st);
    pat_hash_kernel<RP><<<elementwise_grid(n), 256, 0, st>>>(n, rp, col, val, tab, rep, fail);
    cudaMemcpyAsync(h_tab.data(), tab, kPatTable * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(h_rep.data(), rep, kPatTable * 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&h_fail, fail, 4, cudaMemcpyDeviceToHost, st);
    rc = cuda_status(cudaStreamSynchronize(st), "row patterns: hash");
  }
  // slots in order of their first row -> codes
  std::vector<int> slots;
  for (int s = 0; s < kPatTable && !rc; ++s)
    if (h_tab[s]) slots.push_back(s);
  const int u = (int)slots.size();
  bool usable = !rc && !h_fail && u >= 1 && u <= kPatMax;
  std::vector<int> h_len(u), h_start(u + 1, 0), slot_code(kPatTable, -1), reps(u);
  if (usable) {
    std::sort(slots.begin(), slots.end(), [&](int a, int b) { return h_rep[a] < h_rep[b]; });
    for (int k = 0; k < u; ++k) {
      slot_code[slots[k]] = k;
      reps[k] = h_rep[slots[k]];
    }
    if (pool_malloc(&dev_small, (size_t)(3 * u + 1 + kPatTable) * 4) != cudaSuccess)
      rc = set_error(PCG_ENOMEM, "row patterns: dictionary");
  }
  int* d_reps = dev_small;
  int* d_len = dev_small + u;
  int* d_start = dev_small + 2 * u;
  int* d_slot_code = dev_small + 3 * u + 1;
  if (usable && !rc) {
    cudaMemcpyAsync(d_reps, reps.data(), u * 4, cudaMemcpyHostToDevice, st);
    pat_len_kernel<RP><<<1, 256, 0, st>>>(u, d_reps, rp, d_len);
    cudaMemcpyAsync(h_len.data(), d_len, u * 4, cudaMemcpyDeviceToHost, st);
    rc = cuda_status(cudaStreamSynchronize(st), "row patterns: lengths");
    for (int k = 0; k < u; ++k) h_start[k + 1] = h_start[k] + h_len[k];
    usable = !rc && h_start[u] <= kPatMaxEntries;
  }
  if (usable && !rc) {
    const int ne = h_start[u];
    if (pool_malloc(&out->code, (size_t)n + 256) != cudaSuccess ||
        pool_malloc(&out->start, (size_t)(u + 1) * 4) != cudaSuccess ||
        pool_malloc(&out->rep, (size_t)u * 4) != cudaSuccess ||
        pool_malloc(&out->off, (size_t)std::max(ne, 1) * 4) != cudaSuccess ||
        pool_malloc(&out->val, (size_t)std::max(ne, 1) * 8) != cudaSuccess)
      rc = set_error(PCG_ENOMEM, "row patterns: codes");
  }
  if (usable && !rc) {
    cudaMemsetAsync(out->code + n, 0, 256, st);  // bulk-copy overrun of the last tile
    cudaMemcpyAsync(out->start, h_start.data(), (u + 1) * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(out->rep, reps.data(), u * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_start, h_start.data(), (u + 1) * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_slot_code, slot_code.data(), kPatTable * 4, cudaMemcpyHostToDevice, st);
    pat_extract_kernel<RP><<<std::min(u, 256), 128, 0, st>>>(u, d_reps, rp, col, val, d_start,
                                                              out->off, out->val);
    pat_verify_kernel<RP><<<elementwise_grid(n), 256, 0, st>>>(n, rp, col, val, tab, d_slot_code,
                                                               d_start, out->off, out->val,
                                                               out->code, fail);
    cudaMemcpyAsync(&h_fail, fail, 4, cudaMemcpyDeviceToHost, st);
    rc = cuda_status(cudaStreamSynchronize(st), "row patterns: verify");
    usable = !rc && !h_fail;
    if (usable) {
      out->n_pat = u;
      out->n_entries = h_start[u];
      out->max_len = *std::max_element(h_len.begin(), h_len.end());
    }
  }
  pool_free(tab);
  pool_free(rep);
  pool_free(fail);
  pool_free(dev_small);
  if (!usable || rc) free_row_patterns(out);
  return rc;
}

__global__ void pat_dinv_gather_kernel(int u, const int* rep, const double* dinv, double* pdinv) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < u; k += gridDim.x * blockDim.x)
    pdinv[k] = dinv[rep[k]];
}

__global__ void __launch_bounds__(256) pat_dinv_check_kernel(long long n, const unsigned char* code,
                                                             const double* dinv, const double* pdinv,
                                                             int* bad) {
  bool ok = true;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    ok &= __double_as_longlong(dinv[i]) == __double_as_longlong(pdinv[code[i]]);
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) *bad = 1;
}

}  // namespace

int check_dinv_by_code(const RowPatterns& p, long long n, const double* dinv, double* pdinv,
                       bool* ok, bool* uniform, double* value, cudaStream_t st) {
  *ok = false;
  *uniform = false;
  *value = 0.0;
  if (p.n_pat == 0) return PCG_OK;
  int* bad = nullptr;
  if (cudaMallocAsync(&bad, sizeof(int), st) != cudaSuccess)
    return set_error(PCG_ENOMEM, "dinv check");
  cudaMemsetAsync(bad, 0, sizeof(int), st);
  pat_dinv_gather_kernel<<<1, 256, 0, st>>>(p.n_pat, p.rep, dinv, pdinv);
  pat_dinv_check_kernel<<<elementwise_grid(n), 256, 0, st>>>(n, p.code, dinv, pdinv, bad);
  int h = 1;
  std::vector<double> pd(p.n_pat);
  cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(pd.data(), pdinv, p.n_pat * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(bad, st);
  const int rc = cuda_status(cudaStreamSynchronize(st), "dinv check");
  *ok = !rc && h == 0;
  bool same = *ok;
  for (int k = 1; k < p.n_pat && same; ++k)
    same = std::memcmp(&pd[k], &pd[0], sizeof(double)) == 0;
  *uniform = same;
  *value = same ? pd[0] : 0.0;
  return rc;
}

int build_row_patterns(long long n, int rp64, const void* rp, const int* col, const double* val,
                       cudaStream_t st, RowPatterns* out) {
  if (n >= (1LL << 31)) {
    *out = RowPatterns{};
    return PCG_OK;
  }
  return rp64 ? build<long long>(n, static_cast<const long long*>(rp), col, val, st, out)
              : build<int>(n, static_cast<const int*>(rp), col, val, st, out);
}

void free_row_patterns(RowPatterns* p) {
  pool_free(p->code);
  pool_free(p->start);
  pool_free(p->rep);
  pool_free(p->off);
  pool_free(p->val);
  *p = RowPatterns{};
}

int preload_patterns() {
  cudaFuncAttributes a;
  cudaError_t e = cudaSuccess;
#define PCG_LOAD(k) if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void*)(k))
  PCG_LOAD(pat_hash_kernel<int>); PCG_LOAD(pat_hash_kernel<long long>);
  PCG_LOAD(pat_len_kernel<int>); PCG_LOAD(pat_len_kernel<long long>);
  PCG_LOAD(pat_extract_kernel<int>); PCG_LOAD(pat_extract_kernel<long long>);
  PCG_LOAD(pat_verify_kernel<int>); PCG_LOAD(pat_verify_kernel<long long>);
  PCG_LOAD(pat_dinv_gather_kernel); PCG_LOAD(pat_dinv_check_kernel);
#undef PCG_LOAD
  return cuda_status(e, "preload pattern kernels");
}

}  // namespace pcg

extern "C" int pipecg_b200_row_patterns(int64_t n_rows, int rp64, const void* rowptr, const int* col,
                                        const double* val, int64_t* n_pat, int64_t* n_entries,
                                        unsigned char* codes, void* stream) {
  if (n_rows <= 0 || !rowptr || !n_pat || !n_entries)
    return pcg::set_error(PCG_EINVAL, "row_patterns: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  pcg::RowPatterns p;
  int rc = pcg::build_row_patterns(n_rows, rp64, rowptr, col, val, st, &p);
  if (rc) return rc;
  *n_pat = p.n_pat;
  *n_entries = p.n_entries;
  if (codes && p.n_pat > 0)
    rc = pcg::cuda_status(cudaMemcpyAsync(codes, p.code, (size_t)n_rows, cudaMemcpyDeviceToDevice, st),
                          "row_patterns: codes");
  if (!rc) rc = pcg::cuda_status(cudaStreamSynchronize(st), "row_patterns");
  pcg::free_row_patterns(&p);
  return rc;
}
