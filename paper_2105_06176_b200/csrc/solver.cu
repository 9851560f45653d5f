// solver.cu -- the PIPECG iteration on B200 (solvers.py:297-387).
//
// Two engines share one device-side control block (Ctrl) and one prologue:
//
//  Engine 1 ("fused", the hot path): ONE persistent kernel per iteration.
//    Iteration `it` of the reference does
//        scalars(it) -> fused update -> 3 dots -> guards -> m = M^-1 w -> n = A m
//    and iteration it+1 consumes n and m.  Kernel F(it) therefore computes,
//    per row i, n_i = sum_k a_ik * (dinv[c_k] * w_old[c_k]) on the fly from
//    the *previous* w (ping-pong buffers, so neighbours' w is never
//    overwritten in flight), m_i = dinv_i * w_old_i, and then the eight
//    recurrences and the three dot partials.  m and n never touch HBM:
//    17 vector streams + CSR per iteration instead of the canonical 22.
//    Every rounding matches the reference (mul/add separately, CSR order).
//    CSR tiles and the 7 streamed vectors are staged into shared memory by
//    the bulk-copy (TMA) engine from a producer warp, S-stage mbarrier ring.
//
//  Engine 2 ("two-kernel", general matrices, e.g. hub rows): K1 = fused
//    update + Jacobi + dot partials, K2 = SpMV n = A m (thread-per-row for
//    rows <= 256 nnz, block-per-row tree for longer rows).
//
// Control: no host synchronisation per iteration.  Each kernel reads the
// iteration index from Ctrl (base + graph step), re-derives gamma, delta and
// norm from the previous kernel's block partials in a fixed order (every
// block computes identical values), applies the reference's guards and stop
// test in the reference's order, and block 0 records history / status.
// Kernels after a stop are no-ops.  Iterations are launched as CUDA-graph
// chunks; the host reads one small record per chunk while the next chunk
// is already queued.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include "../../include/pipecg_b200.h"
#include "common.cuh"
#include "internal.h"

namespace pcg {

constexpr int kHistRing = 1024;
constexpr int kMaxRanks = 8;
constexpr long long kTuneRows = 1LL << 16;  // autotune engines for >= 64K rows
constexpr int kXchgBlocks = 16;    // exchange-kernel grid (identical on every rank)
constexpr int PCG_ECOMM_STATUS = 3; // Ctrl.status: peer exchange timed out  // history / drift ring (power of two)
constexpr int kMaxChunk = 256;   // 2*kMaxChunk <= kHistRing

struct Slot {
  double gamma, delta, alpha, norm;
};

struct Ctrl {
  // solve constants (set by init)
  double tol;
  long long max_it;
  long long drift_k;
  double b_norm;
  Slot init;  // gamma0, delta0, -, norm0
  // progress
  long long base_it;
  int status;
  int bd_code;
  long long bd_it;
  double bd_val;
  long long final_it;
  double final_norm;
  Slot slot[2];
  unsigned long long arrive_base;  // distributed: arrivals before this solve
  int comm_error;                  // a setup exchange timed out
  int diag_where;                  // 1 = iteration wait, 2 = setup wait timed out
  unsigned long long diag_seen;    // counter value at the timeout
  unsigned long long diag_target;  // value waited for
  int x_final;                     // deferred x: pending update applied after the stop
  int pad_;
  unsigned long long darrive_base;  // distributed drift: x-halo pushes before this solve
  unsigned long long dsum_base;     // ... and drift partials before this solve
};
static_assert(sizeof(Ctrl) <= 256, "Ctrl must fit its 256-byte record slot");

// host-visible record = Ctrl | hist ring | drift-value ring | drift-it ring
constexpr size_t kRecCtrl = 256;
constexpr size_t kRecBytes = kRecCtrl + 3 * kHistRing * sizeof(double);

struct Record {
  Ctrl* C;
  double* hist;
  double* dval;
  long long* dit;
};

__host__ __device__ inline Record record_at(char* base) {
  Record r;
  r.C = reinterpret_cast<Ctrl*>(base);
  r.hist = reinterpret_cast<double*>(base + kRecCtrl);
  r.dval = r.hist + kHistRing;
  r.dit = reinterpret_cast<long long*>(r.dval + kHistRing);
  return r;
}

struct Step {
  int go;
  double alpha, beta;
  double alpha_prev;  // alpha of iteration it-1 (it >= 1)
};

// What the prologue of iteration `it` reduces: pin[(it-1)&1][0..n_pin)[0..2]
// (block partials on one GPU; one partial per rank in distributed mode,
// pushed by the peers' exchange kernels).  In distributed mode `arrive`
// counts the peers' exchange-kernel arrivals (monotonic); iteration it may
// start once arrive >= arrive_base + it * arrive_per_it.
struct ReduceIn {
  const double* pin;
  int n_pin;
  const unsigned long long* arrive;
  unsigned long long arrive_per_it;
};

constexpr long long kSpinTimeoutNs = 10LL * 1000 * 1000 * 1000;  // 10 s

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// spin until *p >= target; false on timeout (a peer died or diverged)
__device__ bool spin_until(const unsigned long long* p, unsigned long long target, Ctrl* C,
                           int where) {
  if (ld_acquire_sys(p) >= target) return true;
  const unsigned long long t0 = globaltimer();
  unsigned long long v;
  while ((v = ld_acquire_sys(p)) < target) {
    if (globaltimer() - t0 > (unsigned long long)kSpinTimeoutNs) {
      C->diag_where = where;
      C->diag_seen = v;
      C->diag_target = target;
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

__device__ __forceinline__ int read_status(const Ctrl* C) {
  return *reinterpret_cast<const volatile int*>(&C->status);
}

// CTA-uniform "is the solve still running?" plus the iteration index: ONE
// thread reads the control block and the whole CTA acts on that value (a
// per-thread read could straddle block 0's status write and split a CTA
// across a later bar.sync).  Returns -1 when the CTA must exit.
// `slot` is a shared-memory word (kernels with a dynamic-smem header pass a
// header slot: static __shared__ would eat into their 227 KB dynamic budget).
__device__ __forceinline__ long long cta_iteration(const Ctrl* C, int step, long long* slot) {
  if (threadIdx.x == 0) *slot = read_status(C) == PCG_RUNNING ? C->base_it + step : -1;
  __syncthreads();
  return *reinterpret_cast<volatile long long*>(slot);
}
__device__ __forceinline__ long long cta_iteration(const Ctrl* C, int step) {
  __shared__ long long s_it;
  return cta_iteration(C, step, &s_it);
}

// The reference's loop head + tail, solvers.py:346-372, for iteration `it`.
// NT threads (local id lt) participate; `leader` is one thread of block 0.
template <int NT>
__device__ Step prologue(Ctrl* C, double* hist, const ReduceIn& R, long long it, int lt,
                         double* red, int bar_id, bool leader) {
  Step st{0, 0.0, 0.0, 0.0};
  double gamma, delta, norm, gamma_prev = 0.0, alpha_prev = 0.0;
  if (it == 0) {
    gamma = C->init.gamma;
    delta = C->init.delta;
    norm = C->init.norm;
  } else {
    if (R.arrive) {  // distributed: wait for every rank's exchange of it-1
      if (lt == 0)
        red[0] = spin_until(R.arrive, C->arrive_base + (unsigned long long)it * R.arrive_per_it,
                            C, 1) ? 1.0 : -1.0;
      bar_sync(bar_id, NT);
      const bool ok = red[0] > 0.0;
      bar_sync(bar_id, NT);
      if (!ok) {
        if (leader || lt == 0) {
          C->bd_code = PCG_BD_NONE;
          C->bd_it = it;
          C->status = PCG_ECOMM_STATUS;
        }
        return st;
      }
    }
    const double* P = R.pin + (size_t)((it - 1) & 1) * (size_t)R.n_pin * 4;
    const int n_partials = R.n_pin;
    double v[3] = {0.0, 0.0, 0.0};
    for (int j = lt; j < n_partials; j += NT) {
      // L2-coherent loads: in the persistent kernel these were written by
      // other CTAs of the same launch (an L1 line could be stale)
      v[0] = add(v[0], __ldcg(P + j * 4 + 0));
      v[1] = add(v[1], __ldcg(P + j * 4 + 1));
      v[2] = add(v[2], __ldcg(P + j * 4 + 2));
    }
    group_sum<3, NT>(v, lt, red, bar_id);
    gamma = v[0];
    delta = v[1];
    norm = sqrt(v[2]);
    const Slot* prev = &C->slot[(it - 1) & 1];
    gamma_prev = __ldcg(&prev->gamma);
    alpha_prev = __ldcg(&prev->alpha);
    st.alpha_prev = alpha_prev;
    // solvers.py:354-357 (iteration it-1's guards)
    if (gamma < 0.0 || !isfinite(gamma)) {
      if (leader) {
        C->bd_code = PCG_BD_GAMMA;
        C->bd_it = it - 1;
        C->bd_val = gamma;
        C->status = PCG_BREAKDOWN;
      }
      return st;
    }
    if (!isfinite(delta)) {
      if (leader) {
        C->bd_code = PCG_BD_DELTA;
        C->bd_it = it - 1;
        C->bd_val = delta;
        C->status = PCG_BREAKDOWN;
      }
      return st;
    }
    if (leader) hist[it & (kHistRing - 1)] = norm;  // solvers.py:369-370
  }
  // solvers.py:346 loop condition (NaN norm exits unconverged)
  if (!(norm >= C->tol && it < C->max_it)) {
    if (leader) {
      C->final_it = it;
      C->final_norm = norm;
      C->status = PCG_STOPPED;
    }
    return st;
  }
  // solvers.py:276-294 pipecg_scalars
  double beta, denom;
  if (it == 0) {
    beta = 0.0;
    denom = delta;
  } else {
    beta = gamma / gamma_prev;
    denom = sub(delta, mul(beta, gamma) / alpha_prev);
  }
  if (denom == 0.0 || !isfinite(denom)) {
    if (leader) {
      C->bd_code = PCG_BD_ALPHA;
      C->bd_it = it;
      C->bd_val = denom;
      C->status = PCG_BREAKDOWN;
    }
    return st;
  }
  const double alpha = gamma / denom;
  if (leader) C->slot[it & 1] = Slot{gamma, delta, alpha, norm};
  st.go = 1;
  st.alpha = alpha;
  st.beta = beta;
  return st;
}

// Distributed comm buffer layout (identical on every rank, IPC-exported):
//   [0] u64 arrive, [8] u64 xarrive, [16] u64 darrive, [24] u64 dsum,
//   [256] slots[2][kMaxRanks][4], [768] islots[kMaxRanks][4],
//   [1024] dslots[2][kMaxRanks]  (see the exchange section below)
constexpr size_t kCommBytes = 2048;
constexpr size_t kCommSlots = 256;
constexpr size_t kCommISlots = 768;
constexpr size_t kCommDSlots = 1024;

// Peer-memory exchange fused into the iteration kernel (distributed mode,
// fused variants A/C/D): after a tile's rows are final the CTA stores the
// tile's halo rows of the gathered vector (w for A, the stored m for C/D)
// straight into the neighbours' HBM over NVLink; the grid's last block then
// pushes this rank's dot partial into every rank's slot and signals every
// rank's arrival counter.  ptr == nullptr: not connected / separate kernel.
struct FusedXchg {
  const int* ptr;        // [n_tiles + 1] send entries of each tile (sorted by row)
  const int* row;        // local row to send
  const int* peer;       // destination rank
  const long long* dst;  // index in the destination's local column space
  char* peer_vbuf[kMaxRanks];
  long long peer_ld[kMaxRanks];
  char* peer_comm[kMaxRanks];
  int rank, world;
};

// The block's (r,u),(w,u),(u,u) partial -> pout; the last block of the grid
// to finish (atomic ticket) sums all partials in a fixed order into fin, so
// the next prologue reads 3 numbers instead of every block's partial.
// Used for large grids only (kFinGrid): for small grids the serial tail
// costs more than every block reducing a few hundred partials itself.
// Deterministic: the sum order does not depend on which block is last.
// red needs 3*NT/32 + 1 doubles.
template <int NT>
__device__ __forceinline__ void publish_partials(double (&acc)[3], int lt, double* red, int bar_id,
                                                 double* pout, double* fin, unsigned* counter,
                                                 long long it, const FusedXchg* X = nullptr) {
  constexpr int NW = NT / PCG_WARP;
  group_sum<3, NT>(acc, lt, red, bar_id);
  double* part = pout + (size_t)(it & 1) * (size_t)gridDim.x * 4;
  if (lt == 0) {
    double* out = part + (size_t)blockIdx.x * 4;
    out[0] = acc[0];
    out[1] = acc[1];
    out[2] = acc[2];
    out[3] = 0.0;
    if (!counter) return;
    // fused exchange: this CTA's halo stores (all consumer threads, ordered
    // before this point by group_sum's barrier) reach the peers before the
    // ticket, hence before the last block's signal
    if (X) __threadfence_system();
    else __threadfence();
    const unsigned ticket = atomicAdd(counter + (it & 1), 1u);
    red[3 * NW] = ticket == gridDim.x - 1 ? 1.0 : 0.0;
  }
  if (!counter) return;  // small grids: the next prologue reduces the partials itself
  bar_sync(bar_id, NT);
  if (red[3 * NW] == 0.0) return;
  __threadfence();
  double v[3] = {0.0, 0.0, 0.0};
  for (int j = lt; j < (int)gridDim.x; j += NT) {
    v[0] = add(v[0], __ldcg(part + j * 4 + 0));
    v[1] = add(v[1], __ldcg(part + j * 4 + 1));
    v[2] = add(v[2], __ldcg(part + j * 4 + 2));
  }
  group_sum<3, NT>(v, lt, red, bar_id);
  if (lt == 0) {
    double* f = fin + (size_t)(it & 1) * 4;
    f[0] = v[0];
    f[1] = v[1];
    f[2] = v[2];
    f[3] = 0.0;
    counter[it & 1] = 0u;  // reused by iteration it + 2 (stream-ordered)
  }
  if (X && lt < X->world) {  // this rank's partial into every rank's slot
    double* slot = reinterpret_cast<double*>(X->peer_comm[lt] + kCommSlots) +
                   ((size_t)(it & 1) * kMaxRanks + X->rank) * 4;
    slot[0] = v[0];
    slot[1] = v[1];
    slot[2] = v[2];
    slot[3] = 0.0;
  }
  if (X) {
    bar_sync(bar_id, NT);
    if (lt == 0) {
      __threadfence_system();
      for (int q = 0; q < X->world; ++q)
        atomicAdd_system(reinterpret_cast<unsigned long long*>(X->peer_comm[q]), 1ull);
    }
  }
}

// Halo rows of tile t -> the peers (see FusedXchg); consumers only (named
// barrier `bar_id` makes the tile's new values visible CTA-wide first).
template <int NT>
__device__ __forceinline__ void tile_exchange_range(const FusedXchg& X, int e0, int e1, int lt,
                                                    const double* src, int vec, int bar_id) {
  if (e1 <= e0) return;  // uniform across the CTA
  bar_sync(bar_id, NT);
  bool sent = false;
  for (int e = e0 + lt; e < e1; e += NT) {
    const int q = X.peer[e];
    double* dst = reinterpret_cast<double*>(X.peer_vbuf[q]) + (size_t)vec * X.peer_ld[q] + X.dst[e];
    *dst = __ldcg(src + X.row[e]);  // written by this CTA (L2-coherent read)
    sent = true;
  }
  if (sent) __threadfence_system();  // before this CTA's ticket (publish_partials)
}
template <int NT>
__device__ __forceinline__ void tile_exchange(const FusedXchg& X, long long t, int lt,
                                              const double* src, int vec, int bar_id) {
  tile_exchange_range<NT>(X, X.ptr[t], X.ptr[t + 1], lt, src, vec, bar_id);
}

// ===========================================================================
// Engine 1: fused iteration kernel
// ===========================================================================
template <typename RP>
struct FusedParams {
  long long n;
  long long n_tiles;
  const RP* rp;
  const int* col;
  const double* val;
  const double* dinv;
  double* vec[7];  // z q s p x r u (in place)
  double* w[2];    // ping-pong: read w[it&1], write w[(it+1)&1]
  double* m[2];    // variant C: stored m = M^-1 w, ping-pong like w
  Ctrl* C;
  double* hist;
  ReduceIn rin;   // what the prologue reduces
  double* pout;   // block partials [2][gridDim.x][4]
  double* fin;    // [2][4] their fixed-order sum (written by the last block)
  unsigned* counter;  // [2] blocks done per iteration parity
  int stages;
  int cap_val;  // doubles per stage
  int cap_col;  // ints per stage
  int flags;    // experiment switches (PIPECG_B200_FLAGS): 2 = contiguous tile ranges per CTA
  FusedXchg X;                // fused peer exchange (X.ptr == nullptr: off)
  // variant D (nnz-balanced tiles)
  const int* tile_row;        // [n_tiles + 1] first row of each tile
  const long long* tile_e;    // [n_tiles + 1] first nonzero of each tile
  long long hub_len;          // rows longer than this are single-row hub tiles
  // variants E/F (row-pattern dictionary, patterns.cu)
  const unsigned char* pcode;  // [n] pattern code per row
  const int* pstart;           // [n_pat + 1]
  const int* poff;             // [n_pat_e] column - row
  const double* pval;          // [n_pat_e]
  const unsigned char* pwin;   // [n_pat_e] window of each entry (WinTable)
  const double* pdinv;         // [n_pat] dinv of each code (valid when WinTable.dinv_by_code)
  const unsigned short* tile_runs;  // [n_tiles] runs the tile's rows use (WinTable bit w)
  int defer_x;                 // E/F: x updated every other iteration (see pipecg_fused_kernel_s)
  int l2_prefetch;             // E/F: prefetch the streams of the tile this many stages ahead into L2 (0: off)
  int n_pat, n_pat_e;
};

template <typename RP, int TR>
struct FusedLayout {
  static constexpr int kGatherWarps = TR / 64;  // 4 / 2 / 1 for TR = 256 / 128 / 64
  static constexpr int kThreads = 32 + 32 * kGatherWarps + TR;
  static constexpr int kRpBytes = (int)(((TR + 1) * sizeof(RP) + 15) / 16 * 16);
  static constexpr int kVecBytes = TR * 8;
  static constexpr int kVecs = 9;  // z q s p x r u (streams) + w_old + dinv (own rows)
  // stage: row pointers | 9 vectors | values | columns | m per nonzero
  __host__ __device__ static int stage_bytes(int cap_val, int cap_col) {
    return kRpBytes + kVecs * kVecBytes + cap_val * 8 + (cap_col * 4 + 15) / 16 * 16 +
           cap_val * 8;
  }
  // barriers + reduction scratch + decision, in front of the stages
  static constexpr int kHeader = 1024;
};

// Warp-specialised CTA:
//   warp 0            producer: bulk-copies (TMA engine) each tile's row
//                     pointers, the 7 streamed vectors, w_old and dinv of the
//                     tile rows, CSR values and columns into an S-stage ring;
//   warps 1..GW       gather: m_k = dinv[c_k] * w_old[c_k] for every nonzero
//                     of the tile into shared memory (the only scattered
//                     global loads, issued in batches, running ahead of the
//                     consumers by up to S-1 tiles);
//   warps GW+1..      consumers: one row per thread, everything from shared
//                     memory: n_i = sum a_k m_k in CSR order, m_i, the eight
//                     recurrences, streaming stores, dot partials.
// Barriers per stage: full (TMA bytes landed), gdone (m written by all
// gather threads), empty (all consumer warps done with the stage).
template <typename RP, int TR>
__global__ void __launch_bounds__(FusedLayout<RP, TR>::kThreads) pipecg_fused_kernel(FusedParams<RP> P,
                                                                                     int step) {
  using L = FusedLayout<RP, TR>;
  constexpr int NT = TR;                          // consumer threads
  constexpr int NG = 32 * L::kGatherWarps;        // gather threads
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [stages]
  uint64_t* gdone = full + 8;                          // [stages]
  uint64_t* empty = full + 16;                         // [stages]
  double* red = reinterpret_cast<double*>(smem + 256);  // 3*8 (+)
  volatile int* decision = reinterpret_cast<volatile int*>(smem + 512);
  double* sc = reinterpret_cast<double*>(smem + 768);  // alpha, beta
  unsigned char* stage0 = smem + L::kHeader;
  const int SB = L::stage_bytes(P.cap_val, P.cap_col);
  const int S = P.stages;

  Ctrl* C = P.C;
  pdl_trigger();
  pdl_wait();  // everything below reads what the previous kernel wrote
  const long long it = cta_iteration(C, step, reinterpret_cast<long long*>(smem + 896));
  if (it < 0) return;
  const double* w_old = P.w[it & 1];
  double* w_new = P.w[(it + 1) & 1];

  const int tid = threadIdx.x;
  const int role = tid < 32 ? 0 : (tid < 32 + NG ? 1 : 2);  // producer / gather / consumer
  // tile ownership: round-robin (tile t -> CTA t % grid) keeps the whole GPU
  // sweeping one narrow window of rows, so the far (+-n^2) gathers of every
  // CTA hit the same L2-resident planes; contiguous ranges per CTA (flag 2)
  // measured 28% slower at 256^3 (far gathers re-read from HBM).
  const bool contiguous = (P.flags & 2) != 0;
  const long long t_lo = contiguous ? (long long)blockIdx.x * P.n_tiles / gridDim.x : blockIdx.x;
  const long long t_hi = contiguous ? (long long)(blockIdx.x + 1) * P.n_tiles / gridDim.x : P.n_tiles;
  const long long t_step = contiguous ? 1 : gridDim.x;
  const long long my_tiles = t_hi > t_lo ? (t_hi - t_lo + t_step - 1) / t_step : 0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&gdone[s], NG);
      mbar_init(&empty[s], NT / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // ---- producer: stage tile j of this block into stage j % S -------------
  uint64_t pol = 0;
  auto issue = [&](long long j) {
    const int s = (int)(j % S);
    const long long t = t_lo + j * t_step;
    const long long t0 = t * TR;
    const long long rows = min((long long)TR, P.n - t0);
    const long long e0 = P.rp[t0], e1 = P.rp[t0 + rows];
    const long long cb = e0 & ~3LL, ce = (e1 + 3) & ~3LL;
    const long long vb = e0 & ~1LL, ve = (e1 + 1) & ~1LL;
    const uint32_t b_rp = (uint32_t)((((rows + 1) * sizeof(RP)) + 15) / 16 * 16);
    const uint32_t b_vec = (uint32_t)((rows * 8 + 15) / 16 * 16);
    const uint32_t b_val = (uint32_t)((ve - vb) * 8);
    const uint32_t b_col = (uint32_t)((ce - cb) * 4);
    unsigned char* sb = stage0 + (size_t)s * SB;
    mbar_arrive_expect_tx(&full[s], b_rp + L::kVecs * b_vec + b_val + b_col);
    bulk_g2s(sb, P.rp + t0, b_rp, &full[s], pol);
#pragma unroll
    for (int k = 0; k < 7; ++k)
      bulk_g2s(sb + L::kRpBytes + k * L::kVecBytes, P.vec[k] + t0, b_vec, &full[s], pol);
    // w_old and dinv of the tile rows: default L2 policy (neighbours gather them)
    bulk_g2s_nohint(sb + L::kRpBytes + 7 * L::kVecBytes, w_old + t0, b_vec, &full[s]);
    bulk_g2s_nohint(sb + L::kRpBytes + 8 * L::kVecBytes, P.dinv + t0, b_vec, &full[s]);
    unsigned char* sval = sb + L::kRpBytes + L::kVecs * L::kVecBytes;
    if (b_val) bulk_g2s(sval, P.val + vb, b_val, &full[s], pol);
    if (b_col) bulk_g2s(sval + (size_t)P.cap_val * 8, P.col + cb, b_col, &full[s], pol);
  };

  if (tid == 0) {
    pol = policy_evict_first();
    for (long long j = 0; j < my_tiles && j < S; ++j) issue(j);
  }

  // ---- prologue (consumers): entry scalars, guards, stop test ------------
  if (role == 2) {
    const int lt = tid - 32 - NG;
    const Step stp = prologue<NT>(C, P.hist, P.rin, it, lt, red, 1, blockIdx.x == 0 && lt == 0);
    if (lt == 0) {
      sc[0] = stp.alpha;
      sc[1] = stp.beta;
      *decision = stp.go;
    }
  }
  __syncthreads();
  const int go = *decision;
  if (!go) {
    // drain the copies already in flight before the CTA retires
    if (tid == 0)
      for (long long j = 0; j < my_tiles && j < S; ++j) mbar_wait(&full[j], 0);
    return;
  }

  if (role == 0) {
    if (tid == 0) {
      for (long long j = S; j < my_tiles; ++j) {
        const int s = (int)(j % S);
        mbar_wait(&empty[s], (uint32_t)((j / S - 1) & 1));
        issue(j);
      }
    }
    return;
  }

  if (role == 1) {
    // ---- gather warps: m_k = dinv[c_k] * w_old[c_k] for the whole tile ----
    const int gt = tid - 32;
    constexpr int U = 8;
    for (long long j = 0; j < my_tiles; ++j) {
      const int s = (int)(j % S);
      const long long t = t_lo + j * t_step;
      const long long rows = min((long long)TR, P.n - t * TR);
      unsigned char* sb = stage0 + (size_t)s * SB;
      const RP* rp_s = reinterpret_cast<const RP*>(sb);
      const double* val_s = reinterpret_cast<const double*>(sb + L::kRpBytes + L::kVecs * L::kVecBytes);
      const int* col_s = reinterpret_cast<const int*>(val_s + P.cap_val);
      double* m_s = const_cast<double*>(val_s) + P.cap_val + (P.cap_col * 4 + 15) / 16 * 2;
      mbar_wait(&full[s], (uint32_t)((j / S) & 1));
      const long long e0 = rp_s[0], e1 = rp_s[rows];
      const long long cb = e0 & ~3LL, vb = e0 & ~1LL;
      for (long long k0 = e0 + gt; k0 < e1; k0 += (long long)NG * U) {
        double dv[U], wv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const long long k = k0 + (long long)u * NG;
          if (k < e1) {
            const int c = col_s[k - cb];
            dv[u] = ldg_nc(P.dinv + c);
            wv[u] = ldg_nc(w_old + c);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const long long k = k0 + (long long)u * NG;
          if (k < e1) m_s[k - vb] = mul(dv[u], wv[u]);  // m = M^-1 w (jacobi_apply)
        }
      }
      mbar_arrive(&gdone[s]);
    }
    return;
  }

  // ---- consumers ----------------------------------------------------------
  const int lt = tid - 32 - NG;
  const double alpha = sc[0], beta = sc[1];
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long j = 0; j < my_tiles; ++j) {
    const int s = (int)(j % S);
    const long long t = t_lo + j * t_step;
    const long long t0 = t * TR;
    const long long rows = min((long long)TR, P.n - t0);
    unsigned char* sb = stage0 + (size_t)s * SB;
    const RP* rp_s = reinterpret_cast<const RP*>(sb);
    const double* v_s = reinterpret_cast<const double*>(sb + L::kRpBytes);
    const double* val_s = reinterpret_cast<const double*>(sb + L::kRpBytes + L::kVecs * L::kVecBytes);
    const double* m_s = val_s + P.cap_val + (P.cap_col * 4 + 15) / 16 * 2;
    const long long i = t0 + lt;
    mbar_wait(&full[s], (uint32_t)((j / S) & 1));
    mbar_wait(&gdone[s], (uint32_t)((j / S) & 1));
    if (lt < rows) {
      const long long e0 = rp_s[0];
      const long long vb = e0 & ~1LL;
      const long long lo = rp_s[lt] - vb, hi = rp_s[lt + 1] - vb;
      // n_i = sum_k a_ik * m_ck in CSR order (kernels.py:64-70 on m)
      double nacc = 0.0;
      for (long long k = lo; k < hi; ++k) nacc = add(nacc, mul(val_s[k], m_s[k]));
      const double wi = v_s[7 * TR + lt], di = v_s[8 * TR + lt];
      const double mi = mul(di, wi);
      const double zi = add(nacc, mul(beta, v_s[0 * TR + lt]));
      const double qi = add(mi, mul(beta, v_s[1 * TR + lt]));
      const double si = add(wi, mul(beta, v_s[2 * TR + lt]));
      const double ui = v_s[6 * TR + lt];
      const double pi = add(ui, mul(beta, v_s[3 * TR + lt]));
      const double xi = add(v_s[4 * TR + lt], mul(alpha, pi));
      const double ri = sub(v_s[5 * TR + lt], mul(alpha, si));
      const double un = sub(ui, mul(alpha, qi));
      const double wn = sub(wi, mul(alpha, zi));
      st_stream(P.vec[0] + i, zi);
      st_stream(P.vec[1] + i, qi);
      st_stream(P.vec[2] + i, si);
      st_stream(P.vec[3] + i, pi);
      st_stream(P.vec[4] + i, xi);
      st_stream(P.vec[5] + i, ri);
      st_stream(P.vec[6] + i, un);
      w_new[i] = wn;  // default policy: the next iteration gathers it
      acc[0] = add(acc[0], mul(ri, un));
      acc[1] = add(acc[1], mul(wn, un));
      acc[2] = add(acc[2], mul(un, un));
    }
    __syncwarp();
    if ((lt & 31) == 0) mbar_arrive(&empty[s]);
  }
  publish_partials<NT>(acc, lt, red, 1, P.pout, P.fin, P.counter, it);
}

template <typename RP, int TR>
struct FusedLayoutA {
  static constexpr int kRpBytes = (int)(((TR + 1) * sizeof(RP) + 15) / 16 * 16);
  static constexpr int kVecBytes = TR * 8;
  __host__ __device__ static int stage_bytes(int cap_val, int cap_col) {
    return kRpBytes + 7 * kVecBytes + cap_val * 8 + (cap_col * 4 + 15) / 16 * 16;
  }
  // barriers + reduction scratch + decision, in front of the stages
  static constexpr int kHeader = 1024;
};

// Variants A and C (consumer warps gather themselves; no gather warps, 7
// staged vectors, L1 serves part of the gathers).
//   A (MG = false): gathers dinv[c] and w_old[c] and forms m_c on the fly
//                   (17 vector streams, 2 gather loads per nonzero);
//   C (MG = true):  gathers a stored m_old[c] and writes m_new = dinv*w_new
//                   beside w_new (19 vector streams, 1 gather load per
//                   nonzero -- better for wide rows).
// Both round exactly like the reference (m is the same rounded product).
// Selected per matrix by the setup-time autotuner.
// XG: the distributed fused exchange is compiled in (a separate
// instantiation: its presence in the tile loop costs ~30% at 256^3 even
// when not taken, measured).
template <typename RP, int TR, bool MG, bool XG = false>
__global__ void __launch_bounds__(TR + 32) pipecg_fused_kernel_a(FusedParams<RP> P, int step) {
  using L = FusedLayoutA<RP, TR>;
  constexpr int NT = TR;  // consumer threads
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);       // [stages]
  uint64_t* empty = full + 8;                                // [stages]
  double* red = reinterpret_cast<double*>(smem + 256);       // 3*8 (+)
  volatile int* decision = reinterpret_cast<volatile int*>(smem + 512);
  double* sc = reinterpret_cast<double*>(smem + 768);        // alpha, beta
  unsigned char* stage0 = smem + L::kHeader;
  const int SB = L::stage_bytes(P.cap_val, P.cap_col);
  const int S = P.stages;

  Ctrl* C = P.C;
  const int tid = threadIdx.x;
  const bool producer = tid < 32;
  // tile ownership: round-robin (tile t -> CTA t % grid) keeps the whole GPU
  // sweeping one narrow window of rows, so the far (+-n^2) gathers of every
  // CTA hit the same L2-resident planes; contiguous ranges per CTA (flag 2)
  // measured 28% slower at 256^3 (far gathers re-read from HBM).
  const bool contiguous = (P.flags & 2) != 0;
  const long long t_lo = contiguous ? (long long)blockIdx.x * P.n_tiles / gridDim.x : blockIdx.x;
  const long long t_hi = contiguous ? (long long)(blockIdx.x + 1) * P.n_tiles / gridDim.x : P.n_tiles;
  const long long t_step = contiguous ? 1 : gridDim.x;
  const long long my_tiles = t_hi > t_lo ? (t_hi - t_lo + t_step - 1) / t_step : 0;

  pdl_trigger();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    fence_barrier_init();
  }
  pdl_wait();  // everything below reads what the previous kernel wrote

  // ---- producer: stage tile j of this block into stage j % S -------------
  uint64_t pol = 0;
  auto issue = [&](long long j) {
    const int s = (int)(j % S);
    const long long t = t_lo + j * t_step;
    const long long t0 = t * TR;
    const long long rows = min((long long)TR, P.n - t0);
    const long long e0 = P.rp[t0], e1 = P.rp[t0 + rows];
    const long long cb = e0 & ~3LL, ce = (e1 + 3) & ~3LL;
    const long long vb = e0 & ~1LL, ve = (e1 + 1) & ~1LL;
    const uint32_t b_rp = (uint32_t)((((rows + 1) * sizeof(RP)) + 15) / 16 * 16);
    const uint32_t b_vec = (uint32_t)((rows * 8 + 15) / 16 * 16);
    const uint32_t b_val = (uint32_t)((ve - vb) * 8);
    const uint32_t b_col = (uint32_t)((ce - cb) * 4);
    unsigned char* sb = stage0 + (size_t)s * SB;
    mbar_arrive_expect_tx(&full[s], b_rp + 7 * b_vec + b_val + b_col);
    bulk_g2s(sb, P.rp + t0, b_rp, &full[s], pol);
#pragma unroll
    for (int k = 0; k < 7; ++k)
      bulk_g2s(sb + L::kRpBytes + k * L::kVecBytes, P.vec[k] + t0, b_vec, &full[s], pol);
    unsigned char* sval = sb + L::kRpBytes + 7 * L::kVecBytes;
    if (b_val) bulk_g2s(sval, P.val + vb, b_val, &full[s], pol);
    if (b_col) bulk_g2s(sval + (size_t)P.cap_val * 8, P.col + cb, b_col, &full[s], pol);
  };

  // The first S tiles are requested before the control block is even read
  // (tile addresses do not depend on the iteration): the status load of
  // thread 32 and the CTA barrier overlap the first bulk copies.  One
  // thread reads the status, so the whole CTA takes the same exit.
  long long* s_it = reinterpret_cast<long long*>(smem + 896);
  if (producer && tid == 0) {
    pol = policy_evict_first();
    for (long long j = 0; j < my_tiles && j < S; ++j) issue(j);
  }
  if (tid == 32) *s_it = read_status(C) == PCG_RUNNING ? C->base_it + step : -1;
  __syncthreads();
  const long long it = *reinterpret_cast<volatile long long*>(s_it);
  if (it < 0) {
    if (tid == 0)  // drain the copies in flight before the CTA retires
      for (long long j = 0; j < my_tiles && j < S; ++j) mbar_wait(&full[j], 0);
    return;
  }
  const double* w_old = P.w[it & 1];
  double* w_new = P.w[(it + 1) & 1];

  // ---- prologue (consumers): entry scalars, guards, stop test ------------
  if (!producer) {
    const Step stp = prologue<NT>(C, P.hist, P.rin, it, tid - 32, red, 1,
                                  blockIdx.x == 0 && tid == 32);
    if (tid == 32) {
      sc[0] = stp.alpha;
      sc[1] = stp.beta;
      *decision = stp.go;
    }
  }
  __syncthreads();
  const int go = *decision;
  if (!go) {
    // drain the copies already in flight before the CTA retires
    if (tid == 0)
      for (long long j = 0; j < my_tiles && j < S; ++j) mbar_wait(&full[j], 0);
    return;
  }
  const double alpha = sc[0], beta = sc[1];

  if (producer) {
    if (tid == 0) {
      for (long long j = S; j < my_tiles; ++j) {
        const int s = (int)(j % S);
        mbar_wait(&empty[s], (uint32_t)((j / S - 1) & 1));
        issue(j);
      }
    }
    return;
  }

  // ---- consumers ----------------------------------------------------------
  const int lt = tid - 32;
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long j = 0; j < my_tiles; ++j) {
    const int s = (int)(j % S);
    const long long t = t_lo + j * t_step;
    const long long t0 = t * TR;
    const long long rows = min((long long)TR, P.n - t0);
    unsigned char* sb = stage0 + (size_t)s * SB;
    const RP* rp_s = reinterpret_cast<const RP*>(sb);
    const double* v_s = reinterpret_cast<const double*>(sb + L::kRpBytes);
    const double* val_s = reinterpret_cast<const double*>(sb + L::kRpBytes + 7 * L::kVecBytes);
    const int* col_s = reinterpret_cast<const int*>(val_s + P.cap_val);
    const long long i = t0 + lt;
    // own w / dinv: issue before waiting on the stage
    double wi = 0.0, di = 0.0;
    if (lt < rows) {
      wi = ldg_nc(w_old + i);
      di = ldg_nc(P.dinv + i);
    }
    mbar_wait(&full[s], (uint32_t)((j / S) & 1));
    if (lt < rows) {
      const long long e0 = rp_s[0];
      const long long cb = e0 & ~3LL, vb = e0 & ~1LL;
      const long long lo = rp_s[lt], hi = rp_s[lt + 1];
      // n_i = sum_k a_ik * m_ck with m = M^-1 w_old, in CSR order.  A batch
      // of 8 entries: first all column indices and values from shared
      // memory, then all gathers back to back, then the ordered accumulation
      // (explicit phases: left to the compiler, the schedule -- and the time
      // -- changed with unrelated edits, measured 0.58-0.74 ms at 256^3).
      double nacc = 0.0;
      for (long long k0 = lo; k0 < hi; k0 += 8) {
        double av[8], mv[8];
        int cc[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const long long k = k0 + t;
          cc[t] = k < hi ? col_s[k - cb] : 0;
          av[t] = k < hi ? val_s[k - vb] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (k0 + t < hi) {
            const int c = cc[t];
            mv[t] = MG ? ldg_nc(P.m[it & 1] + c)                      // stored m
                       : mul(ldg_nc(P.dinv + c), ldg_nc(w_old + c));  // m = M^-1 w
          }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (k0 + t < hi) nacc = add(nacc, mul(av[t], mv[t]));  // n = A m
      }
      const double mi = mul(di, wi);
      const double zi = add(nacc, mul(beta, v_s[0 * TR + lt]));
      const double qi = add(mi, mul(beta, v_s[1 * TR + lt]));
      const double si = add(wi, mul(beta, v_s[2 * TR + lt]));
      const double ui = v_s[6 * TR + lt];
      const double pi = add(ui, mul(beta, v_s[3 * TR + lt]));
      const double xi = add(v_s[4 * TR + lt], mul(alpha, pi));
      const double ri = sub(v_s[5 * TR + lt], mul(alpha, si));
      const double un = sub(ui, mul(alpha, qi));
      const double wn = sub(wi, mul(alpha, zi));
      st_stream(P.vec[0] + i, zi);
      st_stream(P.vec[1] + i, qi);
      st_stream(P.vec[2] + i, si);
      st_stream(P.vec[3] + i, pi);
      st_stream(P.vec[4] + i, xi);
      st_stream(P.vec[5] + i, ri);
      st_stream(P.vec[6] + i, un);
      st_stream(w_new + i, wn);
      if (MG) P.m[(it + 1) & 1][i] = mul(di, wn);  // solvers.py:358 (gathered next iteration)
      acc[0] = add(acc[0], mul(ri, un));
      acc[1] = add(acc[1], mul(wn, un));
      acc[2] = add(acc[2], mul(un, un));
    }
    __syncwarp();
    if ((lt & 31) == 0) mbar_arrive(&empty[s]);
    if (XG)  // the tile's halo rows of the vector the peers gather next
      tile_exchange<NT>(P.X, t, lt, MG ? P.m[(it + 1) & 1] : w_new,
                        MG ? (((it + 1) & 1) ? 12 : 9) : 7 + (int)((it + 1) & 1), 1);
  }
  publish_partials<NT>(acc, lt, red, 1, P.pout, P.fin, P.counter, it, XG ? &P.X : nullptr);
}

// ---------------------------------------------------------------------------
// Variants E / F: the matrix read through its row-pattern dictionary
// (patterns.cu).  Same CTA shape as A / C (producer warp + one consumer
// thread per tile row), but instead of the tile's CSR a stage carries one
// code byte per row: row i's nonzeros are (i + off[k], val[k]) for the
// dictionary slice of its code, held in shared memory for the whole kernel.
// Every sum runs over the same entries in the same order as the CSR row, so
// the roundings are the reference's (kernels.py:64-70).
//
// WIN (the dictionary's offsets form at most kMaxWin runs): the neighbour
// values come from "windows" instead of per-nonzero gathers.  The distinct
// offsets cluster into a few runs (3D 7-pt: -n^2 | -n | -1..1 | n | n^2);
// for a tile [t0, t0 + TR) the values a run needs are one contiguous range
// [t0 + lo, t0 + TR + hi), which the producer bulk-copies (TMA engine) into
// the stage like the streamed vectors -- mostly L2 hits, since the other
// tiles of the sweep read the same lines, so HBM sees each vector once.
// Consumers then read everything from shared memory.
//   F (MG = true):  the stored m_old = dinv * w_old (as C): windows of m,
//                   plus w_old / dinv of the tile rows -> 19 vector streams
//                   (18 when dinv is a function of the row's code);
//   E (MG = false): m_c = dinv[c] * w_old[c] formed on the fly (as A) --
//                   only with WIN when dinv is a function of the row's code
//                   (Jacobi of a constant-coefficient stencil): windows of
//                   w_old and of the codes, dinv[c] = pdinv[code[c]] from
//                   shared memory -> 16 vector streams, the minimum (the 8
//                   recurrence vectors read and written once).  Otherwise E
//                   gathers dinv[c] and w_old[c] per nonzero (17 streams).
// ---------------------------------------------------------------------------
constexpr int kMaxWin = 16;  // windows per tile (more: per-nonzero gathers)

struct WinTable {
  int n;                // runs (0: per-nonzero gathers)
  int elems;            // value-window elements per stage (sum of len)
  int own;              // E: row lt's own w_old is at own + lt (the run holding offset 0)
  int celems;           // E: code-window bytes per stage (sum of clen)
  int cown;             // E: row lt's own code is at cown + lt
  int w0;               // the run holding offset 0
  int dinv_by_code;     // dinv[i] == pdinv[code[i]] for every row (checked)
  int dinv_uniform;     // ... and every pdinv[k] is the same number: E needs no code windows
  double dinv0;         // that number
  long long ld;         // valid length of the windowed vectors (clamp)
  long long code_ld;    // valid length of the code array (clamp)
  int lo[kMaxWin];      // value windows: first offset, rounded down to even
  int len[kMaxWin];     //   elements (even)
  int base[kMaxWin];    //   first element in the stage's window area
  int clo[kMaxWin];     // code windows (E): first offset, rounded down to 16
  int clen[kMaxWin];    //   bytes (multiple of 16)
  int cbase[kMaxWin];   //   first byte in the stage's code-window area
};

template <int TR>
struct FusedLayoutS {
  static constexpr int kVecBytes = TR * 8;
  static constexpr int kHeader = 1024;
  // F+WIN: w_old | dinv | codes | m windows (the 7 streamed vectors are
  //        loaded by the consumers themselves: a smaller stage -> more
  //        stages -> more window bytes in flight)
  // E+WIN: [7 vectors |] w_old windows | code windows (dv: the streamed
  //        vectors loaded by the consumers, as F -- the autotuner times both)
  // gathers: 7 vectors | codes
  __host__ __device__ static int stage_bytes(bool mg, bool win, int elems, int celems, bool dv) {
    if (win && mg) return 2 * kVecBytes + TR + elems * 8;
    if (win) return (dv ? 0 : 7 * kVecBytes) + elems * 8 + celems;
    return 7 * kVecBytes + TR;
  }
};

__device__ __forceinline__ void l2_prefetch_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ unsigned tile_mask(const unsigned short* runs, long long t) {
  unsigned short v;
  asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(runs + t));
  return v;
}

// shared-memory bytes of a dictionary: start | value index | code index |
// val | per-code dinv (16-byte aligned parts)
__host__ __device__ __forceinline__ int pat_smem_bytes(int n_pat, int n_e) {
  return (int)(round_up(4LL * (n_pat + 1), 16) + 2 * round_up(4LL * n_e, 16) + 8LL * n_e +
               round_up(8LL * n_pat, 16));
}

// XG: distributed (row-block shard, [owned | halo] columns): the tile's halo
// rows of w (E) / m (F) are pushed to the peers after each tile, and the
// windows of the first stages are requested only after the prologue has
// seen every peer's previous iteration (they may cover halo rows).
template <int TR, bool MG, bool WIN, bool XG = false, bool DVT = false>
__global__ void __launch_bounds__(TR + 32, TR == 256 ? (MG ? 2 : 3) : (TR == 128 ? 6 : 8))
    pipecg_fused_kernel_s(FusedParams<int> P, WinTable W, int step) {
  using L = FusedLayoutS<TR>;
  constexpr int NT = TR;
  constexpr int VB = L::kVecBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  double* red = reinterpret_cast<double*>(smem + 256);
  volatile int* decision = reinterpret_cast<volatile int*>(smem + 512);
  double* sc = reinterpret_cast<double*>(smem + 768);
  long long* s_it = reinterpret_cast<long long*>(smem + 896);
  unsigned* s_msk = reinterpret_cast<unsigned*>(smem + 128);  // run masks of the first stages
  int* pst = reinterpret_cast<int*>(smem + L::kHeader);
  const int n_start = (int)round_up(P.n_pat + 1, 4), n_e4 = (int)round_up(P.n_pat_e, 4);
  int* pix = pst + n_start;  // WIN: value-window index of the entry for row 0; else the offset
  int* pcx = pix + n_e4;     // E+WIN: code-window index of the entry for row 0
  double* pva = reinterpret_cast<double*>(pcx + n_e4);
  double* pdv = pva + P.n_pat_e;  // per-code dinv
  unsigned char* stage0 = smem + L::kHeader + round_up(pat_smem_bytes(P.n_pat, P.n_pat_e), 128);
  // DV: the consumers load the 7 streamed vectors (F with windows always;
  // E with windows when the plan says so)
  constexpr bool DV = MG ? WIN : (WIN && DVT);
  const int SB = L::stage_bytes(MG, WIN, W.elems, W.celems, DV);
  const int S = P.stages;
  const bool dbc = W.dinv_by_code != 0;
  // F: the stage holds w_old | dinv | codes | m windows
  constexpr int OFF_W = DV ? 0 : 7 * VB, OFF_D = DV ? VB : 8 * VB, OFF_C = DV ? 2 * VB : 9 * VB;
  constexpr int OFF_E = DV ? 0 : 7 * VB;  // E: start of the w_old windows

  Ctrl* C = P.C;
  const int tid = threadIdx.x;
  const bool producer = tid < 32;
  const long long t_lo = blockIdx.x, t_step = gridDim.x;
  const long long my_tiles = P.n_tiles > t_lo ? (P.n_tiles - t_lo + t_step - 1) / t_step : 0;
  // XG: every CTA starts in the middle of its tile list (the sweep order
  // rotated; the tile -> CTA map, hence the partials, unchanged): a
  // z-slab's first tiles are the ones next to the lower halo, and the first
  // tile's SpMV runs before the prologue's wait for the peers (see below)
  const long long rot = XG && my_tiles > 1 ? my_tiles / 2 : 0;
  auto tile_of = [&](long long j) {
    long long jj = j + rot;
    if (jj >= my_tiles) jj -= my_tiles;
    return t_lo + jj * t_step;
  };

  pdl_trigger();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    fence_barrier_init();
  }
  // the dictionary is constant: load it before waiting on the previous grid
  for (int k = tid; k <= P.n_pat; k += blockDim.x) pst[k] = P.pstart[k];
  for (int k = tid; k < P.n_pat; k += blockDim.x) pdv[k] = dbc ? P.pdinv[k] : 0.0;
  // F with windows: entries as one 16-byte record {value, window
  // index} in the space of pix | pcx | pva -- one shared load per nonzero
  // instead of two
  struct PEnt {
    double v;
    int ix, pad;
  };
  PEnt* pent = reinterpret_cast<PEnt*>(pix);
  constexpr bool PE = MG && WIN;  // F reads PEnt records, E pix / pcx / pva
  if (PE) {
    for (int k = tid; k < P.n_pat_e; k += blockDim.x) {
      const int w = P.pwin[k];
      pent[k] = PEnt{P.pval[k], W.base[w] + P.poff[k] - W.lo[w], 0};
    }
  }
  for (int k = tid; k < P.n_pat_e && !PE; k += blockDim.x) {
    if (WIN) {
      const int w = P.pwin[k];
      pix[k] = W.base[w] + P.poff[k] - W.lo[w];
      pcx[k] = W.cbase[w] + P.poff[k] - W.clo[w];
    } else {
      pix[k] = P.poff[k];
    }
    pva[k] = P.pval[k];
  }
  pdl_wait();

  // ---- producer (warp 0: the copies of a tile are spread over its lanes) --
  // One thread issuing a tile's ~12-20 bulk copies (address math, clamps,
  // masks) was the kernel's critical path; each lane now describes and
  // issues at most two of them.  Copy c of tile j:
  //   0-6  the streamed vectors (not with DV)     static
  //   7    F's dinv rows (dinv not by code)       static
  //   8    the tile's codes (F with windows, or no windows)  static
  //   9    F's w_old rows                         written this iteration
  //   10.. value windows (w_old for E, m_old for F): this iteration's own
  //        rows, or -- distributed -- rows reaching into the halo (the peers')
  //   10 + kMaxWin.. E's code windows            static
  // category bits: 1 static, 2 own rows of this iteration, 4 halo rows.
  // msk: the runs the tile's rows use -- distributed only (a shard's halo
  // runs are used by its boundary tiles alone); on one GPU every run is
  // copied.  skip_x: x is neither read nor written this iteration.
  constexpr int kCopies = 10 + 2 * kMaxWin;
  const int lane = tid & 31;
  uint64_t pol = 0;
  struct Cp {
    unsigned char* dst;
    const unsigned char* src;
    uint32_t bytes;
    int cat;
    bool hint;
  };
  auto copy_desc = [&](int c, long long j, unsigned msk, bool skip_x, const double* w_src,
                       const double* m_src) -> Cp {
    Cp d{nullptr, nullptr, 0u, 0, false};
    if (c >= kCopies) return d;
    const int s = (int)(j % S);
    const long long t0 = tile_of(j) * TR;
    const long long rows = min((long long)TR, P.n - t0);
    const uint32_t b_vec = (uint32_t)((rows * 8 + 15) / 16 * 16);
    const uint32_t b_code = (uint32_t)((rows + 15) / 16 * 16);
    unsigned char* sb = stage0 + (size_t)s * SB;
    // range [a, a + len) of an array of `esz`-byte elements, clamped to [0, lim)
    auto range = [&](unsigned char* dst, const void* src, long long a, int len, long long lim,
                     int esz, int cat) {
      const long long e = a + len;
      const long long ca = a < 0 ? 0 : a, ce = e > lim ? lim : e;
      if (ce > ca) {
        d.dst = dst + (ca - a) * esz;
        d.src = static_cast<const unsigned char*>(src) + ca * esz;
        d.bytes = (uint32_t)((ce - ca) * esz);
        d.cat = cat;
      }
    };
    if (c < 7) {
      if (!DV && (c != 4 || !skip_x)) {
        d = Cp{sb + c * VB, reinterpret_cast<const unsigned char*>(P.vec[c] + t0), b_vec, 1, true};
      }
    } else if (c == 7) {
      if (WIN && MG && !dbc)
        d = Cp{sb + OFF_D, reinterpret_cast<const unsigned char*>(P.dinv + t0), b_vec, 1, false};
    } else if (c == 8) {
      if (!WIN || MG) d = Cp{sb + (WIN ? OFF_C : 7 * VB), P.pcode + t0, b_code, 1, false};
    } else if (c == 9) {
      if (WIN && MG)
        d = Cp{sb + OFF_W, reinterpret_cast<const unsigned char*>(w_src + t0), b_vec, 2, false};
    } else if (c < 10 + kMaxWin) {
      const int w = c - 10;
      if (WIN && w < W.n && ((msk >> w) & 1)) {
        const bool halo = XG && t0 + W.lo[w] + W.len[w] > P.n;
        range(sb + (MG ? OFF_C + TR : OFF_E) + (size_t)W.base[w] * 8, MG ? m_src : w_src,
              t0 + W.lo[w], W.len[w], W.ld, 8, halo ? 4 : 2);
      }
    } else {
      const int w = c - 10 - kMaxWin;
      if (WIN && !MG && w < W.n && (!W.dinv_uniform || w == W.w0))
        range(sb + OFF_E + (size_t)W.elems * 8 + W.cbase[w], P.pcode, t0 + W.clo[w], W.clen[w],
              W.code_ld, 1, 1);
    }
    return d;
  };
  // warp 0 issues tile j's copies of categories `cats`; with `expect`, lane 0
  // first arms the stage's barrier with ALL of the tile's bytes
  auto produce = [&](long long j, unsigned msk, bool skip_x, const double* w_src,
                     const double* m_src, int cats, bool expect) {
    const int s = (int)(j % S);
    Cp cp[2] = {copy_desc(lane, j, msk, skip_x, w_src, m_src),
                copy_desc(lane + 32, j, msk, skip_x, w_src, m_src)};
    if (expect) {
      const uint32_t tx = __reduce_add_sync(0xffffffffu, cp[0].bytes + cp[1].bytes);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], tx);
      __syncwarp();
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (cp[q].bytes && (cp[q].cat & cats)) {
        if (cp[q].hint) bulk_g2s(cp[q].dst, cp[q].src, cp[q].bytes, &full[s], pol);
        else bulk_g2s_nohint(cp[q].dst, cp[q].src, cp[q].bytes, &full[s]);
      }
    }
  };
  // Deferred x (defer_x): x_{it+1} = x_it + alpha_it p_it only feeds the
  // result, so even iterations skip it and odd iterations apply both
  // updates in order, x = (x + alpha_{it-1} p_{it-1}) + alpha_it p_it (p_{it-1}
  // is the staged p_old) -- the reference's roundings, one x read + write
  // saved every other iteration.  The producer reads the iteration itself so
  // the first stages know whether to copy x.
  if (producer) {
    pol = policy_evict_first();
    const long long it0 = read_status(C) == PCG_RUNNING ? C->base_it + step : -1;
    const bool skip0 = P.defer_x && it0 >= 0 && (it0 & 1) == 0;
    for (long long j = 0; j < my_tiles && j < S; ++j) {  // the masks first: one latency
      const unsigned m = XG && WIN ? tile_mask(P.tile_runs, tile_of(j)) : ~0u;
      if (lane == 0) s_msk[j] = m;
    }
    __syncwarp();
    for (long long j = 0; j < my_tiles && j < S; ++j)
      produce(j, s_msk[j], skip0, nullptr, nullptr, 1, true);
  }
  if (tid == 32) *s_it = read_status(C) == PCG_RUNNING ? C->base_it + step : -1;
  __syncthreads();
  const long long it = *reinterpret_cast<volatile long long*>(s_it);
  const bool skip_x = P.defer_x && it >= 0 && (it & 1) == 0;
  const long long par = it < 0 ? 0 : it;
  const double* w_old = P.w[par & 1];
  const double* m_old = P.m[par & 1];
  // completes the first stages (before the prologue on one GPU; the halo
  // part after it -- the peers' halo rows have arrived -- when distributed)
  auto produce_first = [&](int cats) {
    if (producer)
      for (long long j = 0; j < my_tiles && j < S; ++j)
        produce(j, s_msk[j], skip_x, w_old, m_old, cats, false);
  };
  produce_first(XG ? 2 : 6);
  if (it < 0) {
    if (XG) produce_first(4);  // (stale data, never read: lets the stages complete)
    if (tid == 0)
      for (long long j = 0; j < my_tiles && j < S; ++j) mbar_wait(&full[j], 0);
    return;
  }
  double* w_new = P.w[(it + 1) & 1];
  const int lt = tid - 32;
  // n_i = sum_k a_ik m_k (CSR order) of row lt of a landed stage, and the
  // row's w_old / dinv
  auto row_spmv = [&](const unsigned char* sb, long long i, double& wi, double& di) -> double {
    const double* v_s = reinterpret_cast<const double*>(sb);
    double nacc = 0.0;
    if (WIN && MG) {
      const double* win = reinterpret_cast<const double*>(sb + OFF_C + TR);
      const int code = sb[OFF_C + lt];
      wi = v_s[OFF_W / 8 + lt];
      di = dbc ? pdv[code] : v_s[OFF_D / 8 + lt];
      const int lo = pst[code], hi = pst[code + 1];
      for (int k = lo; k < hi; ++k) {
        const PEnt e = pent[k];
        nacc = add(nacc, mul(e.v, win[e.ix + lt]));
      }
    } else if (WIN) {
      const double* win = reinterpret_cast<const double*>(sb + OFF_E);
      const unsigned char* cwin = sb + OFF_E + (size_t)W.elems * 8;
      wi = win[W.own + lt];
      const int code = cwin[W.cown + lt];
      if (W.dinv_uniform) {  // one dinv for every row: only the own-row code window
        di = W.dinv0;
        const int lo = pst[code], hi = pst[code + 1];
        // a plain loop: batching the loads 8 at a time measured 8% slower
        // at 256^3 (0.369 vs 0.339 ms, same box) and 15% at 27-pt
        for (int k = lo; k < hi; ++k)
          nacc = add(nacc, mul(pva[k], mul(di, win[pix[k] + lt])));  // m = M^-1 w
      } else {
        di = pdv[code];
        const int lo = pst[code], hi = pst[code + 1];
        for (int k = lo; k < hi; ++k) {
          const double mc = mul(pdv[cwin[pcx[k] + lt]], win[pix[k] + lt]);  // m = M^-1 w
          nacc = add(nacc, mul(pva[k], mc));
        }
      }
    } else {
      // per-nonzero gathers, three explicit phases per batch as in A (wi, di
      // were loaded by the caller before the stage wait)
      const int code = sb[7 * VB + lt];
      const int lo = pst[code], hi = pst[code + 1];
      const int ii = (int)i;
      for (int k0 = lo; k0 < hi; k0 += 8) {
        double av[8], mv[8];
        int cc[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int k = k0 + t < hi ? k0 + t : lo;
          cc[t] = ii + pix[k];
          av[t] = pva[k];
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (k0 + t < hi) {
            const int c = cc[t];
            mv[t] = MG ? ldg_nc(m_old + c) : mul(ldg_nc(P.dinv + c), ldg_nc(w_old + c));
          }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (k0 + t < hi) nacc = add(nacc, mul(av[t], mv[t]));
      }
    }
    return nacc;
  };
  // PIPECG's overlap (Ghysels-Vanroose): n = A m_old needs no
  // alpha, so when this CTA's first tile reads no halo rows its SpMV runs
  // BEFORE the prologue waits for the peers' arrivals -- the rendezvous
  // overlaps it.  (Distributed only; on one GPU the wait is trivial.)
  bool pre = false;
  double pre_n = 0.0, pre_w = 0.0, pre_d = 0.0;
  double pre_dv[7];
  if (XG && WIN && !producer && my_tiles > 0) {
    const long long t0 = tile_of(0) * TR;
    const unsigned m0 = s_msk[0];
    bool halo = false;
    for (int w = 0; w < W.n; ++w)
      halo = halo || (((m0 >> w) & 1) && t0 + W.lo[w] + W.len[w] > P.n);
    if (!halo) {
      pre = true;
      const long long rows = min((long long)TR, P.n - t0);
      const long long i = t0 + lt;
      if (DV && lt < rows) {
#pragma unroll
        for (int k = 0; k < 7; ++k) pre_dv[k] = (k == 4 && skip_x) ? 0.0 : ld_stream(P.vec[k] + i);
      }
      mbar_wait(&full[0], 0u);
      if (lt < rows) pre_n = row_spmv(stage0, i, pre_w, pre_d);
    }
  }
  if (!producer) {
    const Step stp = prologue<NT>(C, P.hist, P.rin, it, tid - 32, red, 1,
                                  blockIdx.x == 0 && tid == 32);
    if (tid == 32) {
      sc[0] = stp.alpha;
      sc[1] = stp.beta;
      sc[2] = stp.alpha_prev;
      *decision = stp.go;
    }
  }
  __syncthreads();
  if (XG && WIN && producer)  // peers' halo stores (acquired in the prologue) before TMA reads
    asm volatile("fence.proxy.async.global;" ::: "memory");
  if (XG) produce_first(4);
  if (!*decision) {
    if (tid == 0)
      for (long long j = 0; j < my_tiles && j < S; ++j) mbar_wait(&full[j], 0);
    // the solve stops here.  A pending deferred x update (it odd) is NOT
    // applied by this kernel: block 0's prologue has already published the
    // stop, so a CTA that starts after that reads it = -1 and could not tell
    // it had rows to finish.  finalize_x_kernel, enqueued by the host after
    // the run, applies it from the control block instead.
    return;
  }
  const double alpha = sc[0], beta = sc[1], alpha_prev = sc[2];
  if (producer) {
    unsigned nmsk = XG && WIN && S < my_tiles ? tile_mask(P.tile_runs, tile_of(S)) : ~0u;
    for (long long j = S; j < my_tiles; ++j) {
      const unsigned msk = nmsk;
      if (XG && WIN && j + 1 < my_tiles)  // in flight while the stage drains
        nmsk = tile_mask(P.tile_runs, tile_of(j + 1));
      if (P.l2_prefetch && lane == 0 && j + P.l2_prefetch < my_tiles) {
        // HBM -> L2 for a tile that is loaded l2_prefetch stages from now:
        // more bytes in flight than the shared-memory ring holds
        const long long tp = tile_of(j + P.l2_prefetch) * TR;
        const uint32_t bp = (uint32_t)((min((long long)TR, P.n - tp) * 8 + 15) / 16 * 16);
#pragma unroll
        for (int k = 0; k < 7; ++k) l2_prefetch_bulk(P.vec[k] + tp, bp);
        if (MG) l2_prefetch_bulk(w_old + tp, bp);
        if (WIN) {  // the leading run: the only window not yet in L2
          const int w = W.n - 1;
          const long long a = tp + W.lo[w], e = min(a + W.len[w], W.ld);
          if (e > a && a >= 0)
            l2_prefetch_bulk((MG ? m_old : w_old) + a, (uint32_t)((e - a) * 8));
        }
      }
      mbar_wait(&empty[j % S], (uint32_t)((j / S - 1) & 1));
      produce(j, msk, skip_x, w_old, m_old, 7, true);
    }
    return;
  }

  // ---- consumers -----------------------------------------------------------
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long j = 0; j < my_tiles; ++j) {
    const int s = (int)(j % S);
    const long long t0 = tile_of(j) * TR;
    const long long rows = min((long long)TR, P.n - t0);
    const unsigned char* sb = stage0 + (size_t)s * SB;
    const double* v_s = reinterpret_cast<const double*>(sb);
    const long long i = t0 + lt;
    const bool done = pre && j == 0;  // SpMV already run before the prologue
    double wi = 0.0, di = 0.0;
    if (!WIN && lt < rows) {
      wi = ldg_nc(w_old + i);
      di = ldg_nc(P.dinv + i);
    }
    // DV: this row's streamed vectors, in flight while the stage lands (a
    // one-tile register look-ahead measured 3% slower at 27-pt)
    double dv[7];
    if (DV && lt < rows) {
#pragma unroll
      for (int k = 0; k < 7; ++k)
        dv[k] = done ? pre_dv[k] : (k == 4 && skip_x) ? 0.0 : ld_stream(P.vec[k] + i);
    }
    // the tile's send range, loaded now so its latency hides under the tile
    // (loaded after the tile it stalled every tile: +0.085 ms per iteration
    // for 2 virtual ranks at 256^3)
    int xe0 = 0, xe1 = 0;
    if (XG) {
      xe0 = ldg_nc(P.X.ptr + t0 / TR);
      xe1 = ldg_nc(P.X.ptr + t0 / TR + 1);
    }
    if (!done) mbar_wait(&full[s], (uint32_t)((j / S) & 1));
    if (lt < rows) {
      double nacc;
      if (done) {
        nacc = pre_n;
        wi = pre_w;
        di = pre_d;
      } else {
        nacc = row_spmv(sb, i, wi, di);
      }
      auto vec = [&](int k) { return DV ? dv[k] : v_s[k * TR + lt]; };
      const double mi = mul(di, wi);
      const double zi = add(nacc, mul(beta, vec(0)));
      const double qi = add(mi, mul(beta, vec(1)));
      const double si = add(wi, mul(beta, vec(2)));
      const double ui = vec(6);
      const double p_old = vec(3);
      const double pi = add(ui, mul(beta, p_old));
      // (deferred x: odd iterations first apply iteration it-1's update)
      const double xi = skip_x ? 0.0
                        : add(P.defer_x ? add(vec(4), mul(alpha_prev, p_old)) : vec(4),
                              mul(alpha, pi));
      const double ri = sub(vec(5), mul(alpha, si));
      const double un = sub(ui, mul(alpha, qi));
      const double wn = sub(wi, mul(alpha, zi));
      st_stream(P.vec[0] + i, zi);
      st_stream(P.vec[1] + i, qi);
      st_stream(P.vec[2] + i, si);
      st_stream(P.vec[3] + i, pi);
      if (!skip_x) st_stream(P.vec[4] + i, xi);
      st_stream(P.vec[5] + i, ri);
      st_stream(P.vec[6] + i, un);
      st_stream(w_new + i, wn);
      if (MG) P.m[(it + 1) & 1][i] = mul(di, wn);  // solvers.py:358
      acc[0] = add(acc[0], mul(ri, un));
      acc[1] = add(acc[1], mul(wn, un));
      acc[2] = add(acc[2], mul(un, un));
    }
    __syncwarp();
    if ((lt & 31) == 0) mbar_arrive(&empty[s]);
    if (XG)  // the tile's halo rows of the vector the peers read next
      tile_exchange_range<NT>(P.X, xe0, xe1, lt, MG ? P.m[(it + 1) & 1] : w_new,
                              MG ? (((it + 1) & 1) ? 12 : 9) : 7 + (int)((it + 1) & 1), 1);
  }
  publish_partials<NT>(acc, lt, red, 1, P.pout, P.fin, P.counter, it, XG ? &P.X : nullptr);
}

// ---------------------------------------------------------------------------
// Variant D: nnz-balanced tiles for irregular rows (power-law graphs,
// SuiteSparse-like matrices).  Tiles are row ranges [tile_row[t],
// tile_row[t+1]) of at most TR rows and at most `cap` staged nonzeros,
// built once per matrix (tile_build_kernel); a row longer than `hub_len`
// is a tile of its own ("hub") whose nonzeros are not staged.
//   normal tile: the 9 own-row vectors (z q s p x r u w_old dinv) and the
//     tile's CSR are bulk-copied to shared memory; the consumers then form
//     every product a_k * m_old[c_k] cooperatively (thread k mod TR: the
//     scattered gathers are spread evenly over the CTA whatever the row
//     lengths), in place over the staged values, and after one named
//     barrier each thread sums its own row's products strictly in CSR
//     order -- the same roundings as kernels.py:64-70, so every non-hub row
//     is bitwise the reference's;
//   hub tile: all TR consumers stride the row's nonzeros straight from
//     global memory and combine with a fixed tree (deterministic; not the
//     reference's order -- tolerance-graded like any parallel dot).
// Everything after n_i is variant C: stored m_new = dinv * w_new is the
// next iteration's gather source (one gather per nonzero).
template <typename RP, int TR>
struct FusedLayoutD {
  static constexpr int kRpBytes = (int)(((TR + 1 + 4) * sizeof(RP) + 15) / 16 * 16);
  static constexpr int kVecStride = TR + 2;  // doubles per staged vector (start aligned down)
  static constexpr int kVecs = 9;
  __host__ __device__ static int stage_bytes(int cap_val, int cap_col) {
    return kRpBytes + kVecs * kVecStride * 8 + cap_val * 8 + (cap_col * 4 + 15) / 16 * 16;
  }
  static constexpr int kHeader = 2048;  // barriers, reduction scratch, per-stage tile meta
};

struct TileMeta {
  long long t0, e0;
  int rows, hub;
  long long pad;
};

// Consumer threads per CTA (all TR tile heights): the gather phase of a
// tile is spread over every consumer, the row phase uses the first `rows`.
constexpr int kDThreads = 256;
constexpr int kDBatch = 8;  // gathers in flight per consumer thread

template <typename RP, int TR, bool XG = false>
__global__ void __launch_bounds__(kDThreads + 32) pipecg_fused_kernel_d(FusedParams<RP> P, int step) {
  using L = FusedLayoutD<RP, TR>;
  constexpr int NT = kDThreads;  // consumer threads
  constexpr int RPA = 16 / (int)sizeof(RP);
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);       // [stages]
  uint64_t* empty = full + 8;                                // [stages]
  double* red = reinterpret_cast<double*>(smem + 256);       // 3*NT/32 doubles
  volatile int* decision = reinterpret_cast<volatile int*>(smem + 640);
  double* sc = reinterpret_cast<double*>(smem + 704);        // alpha, beta
  TileMeta* meta = reinterpret_cast<TileMeta*>(smem + 768);  // [stages]
  unsigned char* stage0 = smem + L::kHeader;
  const int SB = L::stage_bytes(P.cap_val, P.cap_col);
  const int S = P.stages;

  Ctrl* C = P.C;
  pdl_trigger();
  pdl_wait();  // everything below reads what the previous kernel wrote
  const long long it = cta_iteration(C, step, reinterpret_cast<long long*>(smem + 1024));
  if (it < 0) return;
  const double* w_old = P.w[it & 1];
  double* w_new = P.w[(it + 1) & 1];
  const double* m_old = P.m[it & 1];
  double* m_new = P.m[(it + 1) & 1];

  const int tid = threadIdx.x;
  const bool producer = tid < 32;
  const long long my_tiles =
      P.n_tiles > (long long)blockIdx.x ? (P.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();

  uint64_t pol = 0;
  auto issue = [&](long long j) {
    const int s = (int)(j % S);
    const long long t = blockIdx.x + j * (long long)gridDim.x;
    const long long t0 = P.tile_row[t], t1 = P.tile_row[t + 1];
    const long long e0 = P.tile_e[t], e1 = P.tile_e[t + 1];
    const int rows = (int)(t1 - t0);
    const int hub = rows == 1 && e1 - e0 > P.hub_len;
    meta[s] = TileMeta{t0, e0, rows, hub, 0};
    const long long ra = t0 & ~(long long)(RPA - 1), va = t0 & ~1LL;
    const uint32_t b_rp = (uint32_t)(((t1 + 1 - ra) * (long long)sizeof(RP) + 15) / 16 * 16);
    const uint32_t b_vec = (uint32_t)(((t1 - va) * 8 + 15) / 16 * 16);
    const long long cb = e0 & ~3LL, ce = (e1 + 3) & ~3LL;
    const long long vb = e0 & ~1LL, ve = (e1 + 1) & ~1LL;
    const uint32_t b_val = hub ? 0u : (uint32_t)((ve - vb) * 8);
    const uint32_t b_col = hub ? 0u : (uint32_t)((ce - cb) * 4);
    unsigned char* sb = stage0 + (size_t)s * SB;
    mbar_arrive_expect_tx(&full[s], b_rp + L::kVecs * b_vec + b_val + b_col);
    bulk_g2s(sb, P.rp + ra, b_rp, &full[s], pol);
    double* vs = reinterpret_cast<double*>(sb + L::kRpBytes);
#pragma unroll
    for (int k = 0; k < 7; ++k) bulk_g2s(vs + k * L::kVecStride, P.vec[k] + va, b_vec, &full[s], pol);
    bulk_g2s(vs + 7 * L::kVecStride, w_old + va, b_vec, &full[s], pol);
    bulk_g2s(vs + 8 * L::kVecStride, P.dinv + va, b_vec, &full[s], pol);
    unsigned char* sval = sb + L::kRpBytes + L::kVecs * L::kVecStride * 8;
    if (b_val) bulk_g2s(sval, P.val + vb, b_val, &full[s], pol);
    if (b_col) bulk_g2s(sval + (size_t)P.cap_val * 8, P.col + cb, b_col, &full[s], pol);
  };

  if (producer && tid == 0) {
    pol = policy_evict_first();
    for (long long j = 0; j < my_tiles && j < S; ++j) issue(j);
  }

  if (!producer) {
    const Step stp = prologue<NT>(C, P.hist, P.rin, it, tid - 32, red, 1,
                                  blockIdx.x == 0 && tid == 32);
    if (tid == 32) {
      sc[0] = stp.alpha;
      sc[1] = stp.beta;
      *decision = stp.go;
    }
  }
  __syncthreads();
  const int go = *decision;
  if (!go) {
    if (tid == 0)
      for (long long j = 0; j < my_tiles && j < S; ++j) mbar_wait(&full[j], 0);
    return;
  }
  const double alpha = sc[0], beta = sc[1];

  if (producer) {
    if (tid == 0) {
      for (long long j = S; j < my_tiles; ++j) {
        const int s = (int)(j % S);
        mbar_wait(&empty[s], (uint32_t)((j / S - 1) & 1));
        issue(j);
      }
    }
    return;
  }

  // ---- consumers ----------------------------------------------------------
  const int lt = tid - 32;
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long j = 0; j < my_tiles; ++j) {
    const int s = (int)(j % S);
    mbar_wait(&full[s], (uint32_t)((j / S) & 1));
    const TileMeta tm = meta[s];
    unsigned char* sb = stage0 + (size_t)s * SB;
    const long long ra = tm.t0 & ~(long long)(RPA - 1), va = tm.t0 & ~1LL;
    const RP* rp_s = reinterpret_cast<const RP*>(sb) + (tm.t0 - ra);
    const double* v_s = reinterpret_cast<const double*>(sb + L::kRpBytes) + (tm.t0 - va);
    double* val_s = reinterpret_cast<double*>(sb + L::kRpBytes + L::kVecs * L::kVecStride * 8);
    const int* col_s = reinterpret_cast<const int*>(val_s + P.cap_val);
    double nacc = 0.0;
    if (tm.hub) {
      // one long row, all consumers, straight from global memory
      const long long lo = rp_s[0], hi = rp_s[1];
      double part[1] = {0.0};
      for (long long k0 = lo + lt; k0 < hi; k0 += (long long)kDBatch * NT) {
        double a[kDBatch], mv[kDBatch];
#pragma unroll
        for (int u = 0; u < kDBatch; ++u) {
          const long long k = k0 + (long long)u * NT;
          a[u] = 0.0;
          mv[u] = 0.0;
          if (k < hi) {
            a[u] = ldg_nc(P.val + k);
            mv[u] = ldg_nc(m_old + ldg_nc(P.col + k));
          }
        }
#pragma unroll
        for (int u = 0; u < kDBatch; ++u)
          if (k0 + (long long)u * NT < hi) part[0] = add(part[0], mul(a[u], mv[u]));
      }
      group_sum<1, NT>(part, lt, red, 1);
      nacc = part[0];
    } else {
      // products a_k * m_old[c_k] for every staged nonzero, in place
      const int vo = (int)(tm.e0 & 1LL), co = (int)(tm.e0 & 3LL);
      const int span = (int)(rp_s[tm.rows] - tm.e0);
      for (int k0 = lt; k0 < span; k0 += kDBatch * NT) {
        double mv[kDBatch];
#pragma unroll
        for (int u = 0; u < kDBatch; ++u) {
          const int k = k0 + u * NT;
          mv[u] = k < span ? ldg_nc(m_old + col_s[co + k]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kDBatch; ++u) {
          const int k = k0 + u * NT;
          if (k < span) val_s[vo + k] = mul(val_s[vo + k], mv[u]);
        }
      }
      bar_sync(1, NT);
      if (lt < tm.rows) {
        const int lo = (int)(rp_s[lt] - tm.e0), hi = (int)(rp_s[lt + 1] - tm.e0);
        for (int k = lo; k < hi; ++k) nacc = add(nacc, val_s[vo + k]);  // n = A m, CSR order
      }
    }
    const int row_thread = tm.hub ? 0 : lt;
    if (lt == row_thread && lt < tm.rows) {
      const long long i = tm.t0 + lt;
      const double wi = v_s[7 * L::kVecStride + lt];
      const double di = v_s[8 * L::kVecStride + lt];
      const double mi = mul(di, wi);
      const double zi = add(nacc, mul(beta, v_s[0 * L::kVecStride + lt]));
      const double qi = add(mi, mul(beta, v_s[1 * L::kVecStride + lt]));
      const double si = add(wi, mul(beta, v_s[2 * L::kVecStride + lt]));
      const double ui = v_s[6 * L::kVecStride + lt];
      const double pi = add(ui, mul(beta, v_s[3 * L::kVecStride + lt]));
      const double xi = add(v_s[4 * L::kVecStride + lt], mul(alpha, pi));
      const double ri = sub(v_s[5 * L::kVecStride + lt], mul(alpha, si));
      const double un = sub(ui, mul(alpha, qi));
      const double wn = sub(wi, mul(alpha, zi));
      st_stream(P.vec[0] + i, zi);
      st_stream(P.vec[1] + i, qi);
      st_stream(P.vec[2] + i, si);
      st_stream(P.vec[3] + i, pi);
      st_stream(P.vec[4] + i, xi);
      st_stream(P.vec[5] + i, ri);
      st_stream(P.vec[6] + i, un);
      st_stream(w_new + i, wn);
      m_new[i] = mul(di, wn);  // solvers.py:358 (gathered next iteration)
      acc[0] = add(acc[0], mul(ri, un));
      acc[1] = add(acc[1], mul(wn, un));
      acc[2] = add(acc[2], mul(un, un));
    }
    __syncwarp();
    if ((lt & 31) == 0) mbar_arrive(&empty[s]);
    if (XG)  // the tile's halo rows of the stored m (gathered next iteration)
      tile_exchange<NT>(P.X, blockIdx.x + j * (long long)gridDim.x, lt, m_new,
                        ((it + 1) & 1) ? 12 : 9, 1);
  }
  publish_partials<NT>(acc, lt, red, 1, P.pout, P.fin, P.counter, it, XG ? &P.X : nullptr);
}


// ---------------------------------------------------------------------------
// Persistent variant of A/C for latency-bound (small) problems: ONE launch
// runs a whole chunk of K iterations, CTAs meeting at a grid-wide barrier
// (monotonic counter, reset by the chunk graph) between iterations instead
// of a kernel boundary.  The producer keeps streaming: the first tiles of
// iteration it+1 are bulk-copied while the grid is still finishing it (they
// only read this CTA's own rows, ordered by a proxy fence + the stage's
// empty barrier); only the gathers of neighbour rows and the dot partials
// wait for the grid barrier.  Cross-CTA data written inside the launch is
// read with L2-coherent loads.  Same arithmetic as A/C (bitwise).
template <typename RP, int TR, bool MG>
__global__ void __launch_bounds__(TR + 32) pipecg_fused_kernel_p(FusedParams<RP> P, int K,
                                                                  unsigned long long* gbar) {
  using L = FusedLayoutA<RP, TR>;
  constexpr int NT = TR;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  double* red = reinterpret_cast<double*>(smem + 256);
  volatile int* stop = reinterpret_cast<volatile int*>(smem + 512);           // consumers stopped
  volatile int* producer_done = reinterpret_cast<volatile int*>(smem + 516);
  volatile long long* issued = reinterpret_cast<volatile long long*>(smem + 768);
  long long* s_base = reinterpret_cast<long long*>(smem + 896);
  unsigned char* stage0 = smem + L::kHeader;
  const int SB = L::stage_bytes(P.cap_val, P.cap_col);
  Ctrl* C = P.C;
  const int tid = threadIdx.x;
  const bool producer = tid < 32;
  const long long my_tiles =
      P.n_tiles > (long long)blockIdx.x ? (P.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  // never more stages than own tiles: a stage is then only refilled after
  // the consumers finished the SAME tile of the previous iteration
  const int S = (int)max(1LL, min((long long)P.stages, my_tiles));
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    fence_barrier_init();
    *s_base = read_status(C) == PCG_RUNNING ? *reinterpret_cast<volatile long long*>(&C->base_it) : -1;
    *stop = 0;
    *producer_done = 0;
    *issued = 0;
  }
  __syncthreads();
  const long long base = *reinterpret_cast<volatile long long*>(s_base);
  if (base < 0) return;

  uint64_t pol = 0;
  auto issue = [&](long long g) {  // g = running tile counter over the launch
    const int s = (int)(g % S);
    const long long t = blockIdx.x + (g % my_tiles) * (long long)gridDim.x;
    const long long t0 = t * TR;
    const long long rows = min((long long)TR, P.n - t0);
    const long long e0 = P.rp[t0], e1 = P.rp[t0 + rows];
    const long long cb = e0 & ~3LL, ce = (e1 + 3) & ~3LL;
    const long long vb = e0 & ~1LL, ve = (e1 + 1) & ~1LL;
    const uint32_t b_rp = (uint32_t)((((rows + 1) * sizeof(RP)) + 15) / 16 * 16);
    const uint32_t b_vec = (uint32_t)((rows * 8 + 15) / 16 * 16);
    const uint32_t b_val = (uint32_t)((ve - vb) * 8);
    const uint32_t b_col = (uint32_t)((ce - cb) * 4);
    unsigned char* sb = stage0 + (size_t)s * SB;
    mbar_arrive_expect_tx(&full[s], b_rp + 7 * b_vec + b_val + b_col);
    bulk_g2s(sb, P.rp + t0, b_rp, &full[s], pol);
#pragma unroll
    for (int k = 0; k < 7; ++k)
      bulk_g2s(sb + L::kRpBytes + k * L::kVecBytes, P.vec[k] + t0, b_vec, &full[s], pol);
    unsigned char* sval = sb + L::kRpBytes + 7 * L::kVecBytes;
    if (b_val) bulk_g2s(sval, P.val + vb, b_val, &full[s], pol);
    if (b_col) bulk_g2s(sval + (size_t)P.cap_val * 8, P.col + cb, b_col, &full[s], pol);
  };
  const long long total = (long long)K * my_tiles;

  if (producer) {
    // streams every tile of every iteration of the chunk, up to S ahead of
    // the consumers; after a stop (breakdown / convergence / max_iterations
    // mid-chunk) it issues nothing new, and the consumers drain what it did
    // issue before the CTA retires
    if (tid == 0) {
      pol = policy_evict_first();
      for (long long g = 0; g < total; ++g) {
        const int s = (int)(g % S);
        if (g >= S) mbar_wait(&empty[s], (uint32_t)((g / S - 1) & 1));
        if (*stop) break;
        issue(g);
        *issued = g + 1;
      }
      __threadfence_block();
      *producer_done = 1;
    }
    return;
  }
  const int lt = tid - 32;
  long long g = 0;
  bool stopped = false;
  for (int step = 0; step < K; ++step) {
    const long long it = base + step;
    if (step > 0) {  // grid barrier: every CTA finished iteration it - 1
      if (lt == 0) {
        const unsigned long long target = (unsigned long long)step * gridDim.x;
        // GPU-scope acquire spin (P is single-GPU only): 2D 512^2 11.2 -> 11.0 us/it
        while (ld_acquire_gpu(gbar) < target) {
        }
      }
      bar_sync(1, NT);
    }
    const Step stp = prologue<NT>(C, P.hist, P.rin, it, lt, red, 1, blockIdx.x == 0 && lt == 0);
    if (!stp.go) {  // identical decision in every CTA: nobody waits at a later barrier
      if (lt == 0) *stop = 1;
      stopped = true;
      break;
    }
    const double alpha = stp.alpha, beta = stp.beta;
    const double* w_old = P.w[it & 1];
    double* w_new = P.w[(it + 1) & 1];
    double acc[3] = {0.0, 0.0, 0.0};
    for (long long j = 0; j < my_tiles; ++j, ++g) {
      const int s = (int)(g % S);
      const long long t = blockIdx.x + j * (long long)gridDim.x;
      const long long t0 = t * TR;
      const long long rows = min((long long)TR, P.n - t0);
      unsigned char* sb = stage0 + (size_t)s * SB;
      const RP* rp_s = reinterpret_cast<const RP*>(sb);
      const double* v_s = reinterpret_cast<const double*>(sb + L::kRpBytes);
      const double* val_s = reinterpret_cast<const double*>(sb + L::kRpBytes + 7 * L::kVecBytes);
      const int* col_s = reinterpret_cast<const int*>(val_s + P.cap_val);
      const long long i = t0 + lt;
      double wi = 0.0, di = 0.0;
      if (lt < rows) {
        wi = __ldcg(w_old + i);
        di = ldg_nc(P.dinv + i);
      }
      mbar_wait(&full[s], (uint32_t)((g / S) & 1));
      if (lt < rows) {
        const long long e0 = rp_s[0];
        const long long cb = e0 & ~3LL, vb = e0 & ~1LL;
        const long long lo = rp_s[lt], hi = rp_s[lt + 1];
        double nacc = 0.0;
        for (long long k0 = lo; k0 < hi; k0 += 8) {
          double av[8], mv[8];
          int cc[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const long long k = k0 + u;
            cc[u] = k < hi ? col_s[k - cb] : 0;
            av[u] = k < hi ? val_s[k - vb] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (k0 + u < hi) {
              const int c = cc[u];
              mv[u] = MG ? __ldcg(P.m[it & 1] + c) : mul(ldg_nc(P.dinv + c), __ldcg(w_old + c));
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (k0 + u < hi) nacc = add(nacc, mul(av[u], mv[u]));
        }
        const double mi = mul(di, wi);
        const double zi = add(nacc, mul(beta, v_s[0 * TR + lt]));
        const double qi = add(mi, mul(beta, v_s[1 * TR + lt]));
        const double si = add(wi, mul(beta, v_s[2 * TR + lt]));
        const double ui = v_s[6 * TR + lt];
        const double pi = add(ui, mul(beta, v_s[3 * TR + lt]));
        const double xi = add(v_s[4 * TR + lt], mul(alpha, pi));
        const double ri = sub(v_s[5 * TR + lt], mul(alpha, si));
        const double un = sub(ui, mul(alpha, qi));
        const double wn = sub(wi, mul(alpha, zi));
        P.vec[0][i] = zi;
        P.vec[1][i] = qi;
        P.vec[2][i] = si;
        P.vec[3][i] = pi;
        P.vec[4][i] = xi;
        P.vec[5][i] = ri;
        P.vec[6][i] = un;
        w_new[i] = wn;
        if (MG) P.m[(it + 1) & 1][i] = mul(di, wn);
        acc[0] = add(acc[0], mul(ri, un));
        acc[1] = add(acc[1], mul(wn, un));
        acc[2] = add(acc[2], mul(un, un));
      }
      // the producer re-reads these rows with the bulk-copy (async) proxy
      // next iteration: order the generic-proxy stores before the release
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncwarp();
      if ((lt & 31) == 0) mbar_arrive(&empty[s]);
    }
    publish_partials<NT>(acc, lt, red, 1, P.pout, P.fin, nullptr, it);
    // arrive at the grid barrier (all of this CTA's stores before the count)
    bar_sync(1, NT);
    if (lt == 0) {
      __threadfence();
      atomicAdd(gbar, 1ull);
    }
  }
  // stopped mid-chunk: consume (without computing) every tile the producer
  // still issued, releasing its stages, until it has quit -- no bulk copy may
  // be in flight when the CTA retires, and the producer never blocks
  if (stopped) {
    for (;;) {
      if (g < *issued) {
        const int s = (int)(g % S);
        mbar_wait(&full[s], (uint32_t)((g / S) & 1));
        __syncwarp();
        if ((lt & 31) == 0) mbar_arrive(&empty[s]);
        ++g;
        continue;
      }
      if (*producer_done && g >= *issued) break;
      __nanosleep(64);
    }
  }
}

// ===========================================================================
// Engine 2: K1 (update + Jacobi + dot partials) and K2 (gated SpMV)
// ===========================================================================
struct TwoParams {
  long long n;
  double *z, *q, *s, *p, *x, *r, *u, *w, *m, *nv;
  const double* dinv;
  Ctrl* C;
  double* hist;
  ReduceIn rin;
  double* pout;
  double* fin;
  unsigned* counter;
};

// POL: L2 hints -- the streams evict-first, m (gathered by the SpMV next)
// stored evict-last
template <bool POL>
__global__ void __launch_bounds__(256) pipecg_k1_kernel(TwoParams P, int step) {
  __shared__ double red[3 * 8 + 1];
  Ctrl* C = P.C;
  pdl_trigger();
  pdl_wait();  // n from the SpMV kernels of the previous iteration
  const long long it = cta_iteration(C, step);
  if (it < 0) return;
  const Step stp = prologue<256>(C, P.hist, P.rin, it, threadIdx.x, red, 1,
                                 blockIdx.x == 0 && threadIdx.x == 0);
  if (!stp.go) return;
  const double alpha = stp.alpha, beta = stp.beta;
  double acc[3] = {0.0, 0.0, 0.0};
  const uint64_t pf = POL ? policy_l2(1) : 0, pl = POL ? policy_l2(2) : 0;
  auto ld = [&](const double* a) { return POL ? ld_hint(a, pf) : *a; };
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < P.n; i += (long long)gridDim.x * 256) {
    const double zi = add(ld(P.nv + i), mul(beta, ld(P.z + i)));
    const double qi = add(ld(P.m + i), mul(beta, ld(P.q + i)));
    const double wi = ld(P.w + i), ui = ld(P.u + i);
    const double si = add(wi, mul(beta, ld(P.s + i)));
    const double pi = add(ui, mul(beta, ld(P.p + i)));
    const double xi = add(ld(P.x + i), mul(alpha, pi));
    const double ri = sub(ld(P.r + i), mul(alpha, si));
    const double un = sub(ui, mul(alpha, qi));
    const double wn = sub(wi, mul(alpha, zi));
    P.z[i] = zi;
    P.q[i] = qi;
    P.s[i] = si;
    P.p[i] = pi;
    P.x[i] = xi;
    P.r[i] = ri;
    P.u[i] = un;
    P.w[i] = wn;
    if (POL) st_hint(P.m + i, mul(ld(P.dinv + i), wn), pl);  // solvers.py:358
    else P.m[i] = mul(P.dinv[i], wn);
    acc[0] = add(acc[0], mul(ri, un));
    acc[1] = add(acc[1], mul(wn, un));
    acc[2] = add(acc[2], mul(un, un));
  }
  publish_partials<256>(acc, threadIdx.x, red, 1, P.pout, P.fin, P.counter, it);
}

template <typename RP>
__global__ void __launch_bounds__(256) gated_spmv_rows(const Ctrl* C, long long n, const RP* __restrict__ rp,
                                                        const int* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y, long long thr) {
  if (read_status(C) != PCG_RUNNING) return;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const long long lo = rp[i], hi = rp[i + 1];
    if (hi - lo > thr) continue;
    double acc = 0.0;
    for (long long k = lo; k < hi; ++k) acc = add(acc, mul(ldg_nc(val + k), ldg_nc(x + ldg_nc(col + k))));
    y[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// Engine 2's K2 in SELL-C-sigma layout (irregular rows): rows sorted by
// length inside windows of kSellSigma rows, packed in slices of 32 rows
// whose k-th nonzeros are contiguous (column-major inside the slice).  One
// warp per slice, one lane per row: a warp's load of "entry k" is one
// coalesced 256-byte segment instead of 32 scattered ones, the rows of a
// warp have similar lengths (little divergence), and every lane still sums
// its own row strictly in CSR order -- bitwise the reference's _spmv.
// Rows longer than kLongRow keep the block-per-row kernel (slen = -1 here).
// 256 = engine 3's window (one CTA); engine 2 reads the same copy (1024
// measured within noise for engine 2's SELL kernel alone)
constexpr int kSellSigma = 1024;

template <int SB, bool POL>
__global__ void __launch_bounds__(256) sell_spmv_kernel(const Ctrl* C, long long n, long long n_slices,
                                                         const long long* __restrict__ sptr,
                                                         const int* __restrict__ perm,
                                                         const int* __restrict__ slen,
                                                         const int* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x,
                                                         double* __restrict__ y, int gld) {
  pdl_wait();     // m from K1
  pdl_trigger();  // ... then the hub-row chunks may start beside this kernel
  if (C && read_status(C) != PCG_RUNNING) return;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const uint64_t pf = POL ? policy_l2(1) : 0, pl = POL ? policy_l2(2) : 0;
  for (long long sl = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); sl < n_slices;
       sl += warps) {
    const long long p = sl * 32 + lane;
    const bool valid = p < n;
    const int r = valid ? perm[p] : 0;
    const int len = valid ? slen[p] : -1;
    int L = max(len, 0);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) L = max(L, __shfl_xor_sync(0xffffffffu, L, o));
    const long long base = sptr[sl] + lane;
    double acc = 0.0;
    for (int k0 = 0; k0 < L; k0 += SB) {  // batches: indices + values, gathers, ordered adds
      int c[SB];
      double a[SB], xv[SB];
#pragma unroll
      for (int u = 0; u < SB; ++u) {
        const bool on = k0 + u < len;
        c[u] = on ? (POL ? ld_hint(col + base + 32LL * (k0 + u), pf) : ldg_nc(col + base + 32LL * (k0 + u))) : 0;
        a[u] = on ? (POL ? ld_hint(val + base + 32LL * (k0 + u), pf) : ldg_nc(val + base + 32LL * (k0 + u))) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < SB; ++u)
        xv[u] = k0 + u < len ? (POL ? (gld == 1 ? __ldca(x + c[u]) : gld == 2 ? __ldcg(x + c[u])
                                                     : ld_gather(x + c[u], pl))
                                    : ldg_nc(x + c[u]))
                             : 0.0;
#pragma unroll
      for (int u = 0; u < SB; ++u)
        if (k0 + u < len) acc = add(acc, mul(a[u], xv[u]));
    }
    if (valid && len >= 0) y[r] = acc;
  }
}

// SELL build (setup): sort keys, slice widths, packing
template <typename RP>
__global__ void sell_keys_kernel(long long n, const RP* rp, long long thr, int* key, int* idx) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long len = (long long)rp[i + 1] - rp[i];
    key[i] = len > thr ? (int)thr + 1 : (int)(thr - len);  // ascending key = descending length, long last
    idx[i] = (int)i;
  }
}

template <typename RP>
__global__ void sell_len_kernel(long long n, const RP* rp, long long thr, const int* perm, int* slen,
                                long long n_slices, long long* width) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int r = perm[p];
    const long long len = (long long)rp[r + 1] - rp[r];
    slen[p] = len > thr ? -1 : (int)len;
    if ((p & 31) == 0) width[p >> 5] = 32LL * (len > thr ? 0 : len);  // first = longest of the slice
  }
}

template <typename RP>
__global__ void sell_fill_kernel(long long n, const RP* rp, const int* col, const double* val,
                                 const int* perm, const int* slen, const long long* sptr,
                                 int* col_s, double* val_s) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int len = slen[p];
    if (len <= 0) continue;
    const long long src = rp[perm[p]], dst = sptr[p >> 5] + (p & 31);
    for (int k = 0; k < len; ++k) {
      col_s[dst + 32LL * k] = col[src + k];
      val_s[dst + 32LL * k] = val[src + k];
    }
  }
}

// Long rows split into chunks of at most kChunkNnz nonzeros, one CTA per
// chunk (hub rows of 49k nonzeros no longer serialise one CTA): each CTA
// reduces its chunk with a fixed tree; a row's last chunk to finish (atomic
// ticket) sums the chunk partials in chunk order.  Deterministic.
constexpr long long kChunkNnz = 2048;

struct LongChunk {
  long long lo, hi;  // nonzero range
  int row;           // matrix row
  int first;         // index of the row's first chunk
  int n;             // chunks of this row
  int slot;          // ticket counter of the row (multi-chunk rows)
  int hub;           // index of the row in the long-row list (engine 3: its dot slot)
  int pad_;
};

__global__ void __launch_bounds__(256) gated_spmv_chunks(const Ctrl* C, const LongChunk* __restrict__ ch,
                                                          const int* __restrict__ col,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y, double* part,
                                                          unsigned* ticket) {
  __shared__ double red[9];
  __shared__ int last;
  // Launched (programmatically) while the SELL kernel still runs: the hub
  // rows only need K1's m, which SELL waited for before letting this kernel
  // start.  Every thread waits for SELL to complete before it exits, so the
  // next K1 -- ordered after this grid -- sees all of n.
  struct WaitOnExit {
    __device__ ~WaitOnExit() { pdl_wait(); }
  } wait_on_exit;
  if (cta_iteration(C, 0) < 0) return;
  const LongChunk c = ch[blockIdx.x];
  double v[1] = {0.0};
  for (long long k0 = c.lo + threadIdx.x; k0 < c.hi; k0 += 4 * 256) {
    double a[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long k = k0 + 256LL * u;
      a[u] = 0.0;
      xv[u] = 0.0;
      if (k < c.hi) {
        a[u] = ldg_nc(val + k);
        xv[u] = ldg_nc(x + ldg_nc(col + k));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (k0 + 256LL * u < c.hi) v[0] = add(v[0], mul(a[u], xv[u]));
  }
  group_sum<1, 256>(v, threadIdx.x, red, 1);
  if (c.n == 1) {
    if (threadIdx.x == 0) y[c.row] = v[0];
    return;
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = v[0];
    __threadfence();
    last = atomicAdd(ticket + c.slot, 1u) == (unsigned)(c.n - 1);
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (int j = 0; j < c.n; ++j) s = add(s, __ldcg(part + c.first + j));
    y[c.row] = s;
    ticket[c.slot] = 0u;  // next iteration (stream-ordered)
  }
}

template <typename RP>
__global__ void __launch_bounds__(256) gated_spmv_long(const Ctrl* C, const int* __restrict__ rows,
                                                        const RP* __restrict__ rp,
                                                        const int* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y) {
  __shared__ double red[8];
  if (cta_iteration(C, 0) < 0) return;
  const long long i = rows[blockIdx.x];
  const long long lo = rp[i], hi = rp[i + 1];
  double v[1] = {0.0};
  for (long long k = lo + threadIdx.x; k < hi; k += 256)
    v[0] = add(v[0], mul(ldg_nc(val + k), ldg_nc(x + ldg_nc(col + k))));
  group_sum<1, 256>(v, threadIdx.x, red, 1);
  if (threadIdx.x == 0) y[i] = v[0];
}

// ===========================================================================
// Engine 3 ("fused-g"): irregular matrices, ONE kernel per iteration
// ===========================================================================
// Engine 2 runs an irregular matrix as K1 (20 vector streams) + a SELL SpMV
// (n written, then re-read by the next K1) + hub-row chunks.  Engine 3 makes
// the SpMV of iteration it+1 and the update of iteration it one pass, as the
// fused engine does, keeping engine 2's irregular-row machinery:
//
//   * the solver state lives in SELL order: position p holds row perm[p]
//     (rows sorted by length inside 256-row windows), so the lane that sums
//     row perm[p] -- one lane per row, 32-row slices whose k-th nonzeros
//     are contiguous (coalesced column / value loads) -- also updates
//     position p of every vector with coalesced loads and stores.  Warps
//     are independent: no shared memory, no CTA barrier per slice.  The
//     SELL copy's columns are renumbered into positions (iperm[col]); the
//     permutation stays inside each window, so the gathers keep the matrix's
//     locality.  b and the caller-facing x are natural order (init permutes
//     the state in, solver_x / solver_state permute out).
//   * the eight recurrences (kernels.py:100-111), with m_p = dinv_p * w_p
//     formed from the w the lane reads anyway (bit for bit the stored m),
//     m_new = dinv * w_new stored for the next iteration's gathers
//     (ping-pong m), dot partials;
//   * rows longer than kLongRow ("hubs", SELL length -1) are packed
//     (positions, values) at setup and cut into chunks of <= kGChunkNnz
//     nonzeros, one WARP each; the row's last chunk to finish (atomic
//     ticket) sums the chunk partials in chunk order and applies the row's
//     update, its three dot terms going into the row's slot; the grid's
//     last CTA sums the block partials and then the hub slots in a fixed
//     order (deterministic).
//
// Bytes per iteration: z q s p x r u w read + written, dinv read, m_new
// written (18 streams) + the SELL copy (12 B per nonzero) + the m gathers,
// which L2 serves when the streams are marked evict-first.
// Every row sums its nonzeros in CSR order (bitwise the reference's _spmv,
// kernels.py:64-70); only the order of the dot partials is a tree.
constexpr int kGRows = 256;              // SELL sigma (window) and CTA size
constexpr long long kGChunkNnz = 512;    // hub chunk = one warp
// rows longer than this leave the lane-per-row SELL path for warp chunks: a
// lane's row is a chain of dependent (index -> gather) loads, and a slice
// of 256-nonzero rows would be the kernel's critical path
constexpr long long kGLaneRow = 64;

struct GParams {
  long long n;
  long long n_slices;       // ceil(n / 32)
  long long n_chunks;       // hub-row chunks (0: no hub rows)
  const long long* sptr;    // SELL slice starts (elements)
  const int* slen;          // SELL position -> row length (-1: hub row)
  const int* scol;          // SELL columns as positions
  const double* sval;
  const LongChunk* chunks;  // hub chunks: ranges of hcol / hval, row = position
  const int* hcol;          // hub rows packed: columns as positions
  const double* hval;
  double* chunk_part;
  unsigned* chunk_ticket;
  double* hubdot;           // [n_hub][4]: dot terms of each multi-chunk row
  int n_hub;
  const double* dinv;       // inv_diag in SELL order
  double *z, *q, *s, *p, *x, *r, *u, *w;
  double* m[2];             // ping-pong: gather m[it&1], write m[(it+1)&1]
  Ctrl* C;
  double* hist;
  ReduceIn rin;
  double* pout;             // block partials [2][grid][4]
  double* fin;              // [2][4]
  unsigned* counter;        // [2]
};

struct GRow {
  double z, q, s, p, x, r, u, w, d;
};

__device__ __forceinline__ GRow g_load(const GParams& P, long long i, uint64_t pol) {
  GRow v;
  v.z = ld_hint(P.z + i, pol);
  v.q = ld_hint(P.q + i, pol);
  v.s = ld_hint(P.s + i, pol);
  v.p = ld_hint(P.p + i, pol);
  v.x = ld_hint(P.x + i, pol);
  v.r = ld_hint(P.r + i, pol);
  v.u = ld_hint(P.u + i, pol);
  v.w = ld_hint(P.w + i, pol);
  v.d = ld_hint(P.dinv + i, pol);
  return v;
}

// kernels.py:100-111 (order and roundings of _fused_update), m = M^-1 w
// (solvers.py:358) and the three dot terms of position i
__device__ __forceinline__ void g_update(const GParams& P, long long i, const GRow& v, double nval,
                                         double alpha, double beta, double* m_new, uint64_t pst,
                                         uint64_t pm, double (&acc)[3]) {
  const double mi = mul(v.d, v.w);  // = the stored m_old bit for bit
  const double zi = add(nval, mul(beta, v.z));
  const double qi = add(mi, mul(beta, v.q));
  const double si = add(v.w, mul(beta, v.s));
  const double pi = add(v.u, mul(beta, v.p));
  const double xi = add(v.x, mul(alpha, pi));
  const double ri = sub(v.r, mul(alpha, si));
  const double un = sub(v.u, mul(alpha, qi));
  const double wn = sub(v.w, mul(alpha, zi));
  st_hint(P.z + i, zi, pst);
  st_hint(P.q + i, qi, pst);
  st_hint(P.s + i, si, pst);
  st_hint(P.p + i, pi, pst);
  st_hint(P.x + i, xi, pst);
  st_hint(P.r + i, ri, pst);
  st_hint(P.u + i, un, pst);
  st_hint(P.w + i, wn, pst);
  st_hint(m_new + i, mul(v.d, wn), pm);
  acc[0] = add(acc[0], mul(ri, un));
  acc[1] = add(acc[1], mul(wn, un));
  acc[2] = add(acc[2], mul(un, un));
}

// SB: SELL nonzeros per lane per load batch; MB: CTAs per SM compiled for;
// PF: the lane's update operands are loaded before its SpMV (in flight during
// the gathers, 18 more live registers) or after it
template <int SB, int MB, bool PF>
__global__ void __launch_bounds__(kGRows, MB) pipecg_fused_kernel_g(GParams P, int step) {
  __shared__ double red[3 * (kGRows / 32) + 1];
  __shared__ int s_last;
  __shared__ long long s_it;
  Ctrl* C = P.C;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  pdl_trigger();
  pdl_wait();  // m_old, the vectors and the partials of the previous iteration
  const long long it = cta_iteration(C, step, &s_it);
  if (it < 0) return;
  const Step stp = prologue<kGRows>(C, P.hist, P.rin, it, tid, red, 1, blockIdx.x == 0 && tid == 0);
  if (!stp.go) return;
  const double alpha = stp.alpha, beta = stp.beta;
  const double* m_old = P.m[it & 1];
  double* m_new = P.m[(it + 1) & 1];
  // L2: everything streamed once per iteration (SELL copy, the state
  // vectors) evict-first; m (stored now, gathered next iteration) and its
  // gathers evict-last, so the randomly gathered vector stays L2-resident
  const uint64_t p_sell = policy_l2(1), p_str = p_sell;
  const uint64_t p_m = policy_l2(2), p_g = p_m;
  const long long gwarp = (long long)blockIdx.x * (kGRows / 32) + warp;
  const long long n_warps = (long long)gridDim.x * (kGRows / 32);
  double acc[3] = {0.0, 0.0, 0.0};

  // ---- hub rows: chunks of <= kGChunkNnz nonzeros, one warp each -------
  for (long long c = gwarp; c < P.n_chunks; c += n_warps) {
    const LongChunk ch = P.chunks[c];
    // products 32 at a time (lane l: entry 32 r + l), summed IN ORDER by
    // every lane through shuffles: the chunk's sum is a left-to-right sum
    // of its entries, so a one-chunk row is the reference's _spmv row
    double v = 0.0;
    for (long long k0 = ch.lo + lane; k0 < ch.hi + lane; k0 += 32LL * 4) {
      double pr[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const long long k = k0 + 32LL * t;
        pr[t] = 0.0;
        if (k < ch.hi) pr[t] = mul(ld_hint(P.hval + k, p_sell), ld_gather(m_old + ld_hint(P.hcol + k, p_sell), p_g));
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const long long r0 = k0 - lane + 32LL * t;  // entry of lane 0 in this round
        const int cnt = (int)max(0LL, min(32LL, ch.hi - r0));
        for (int l = 0; l < cnt; ++l) v = add(v, __shfl_sync(0xffffffffu, pr[t], l));
      }
    }
    if (lane == 0) {
      double nrow = v;
      bool mine = true;
      if (ch.n > 1) {  // the row's last chunk to finish sums the chunk partials in order
        P.chunk_part[c] = v;
        __threadfence();
        mine = atomicAdd(P.chunk_ticket + ch.slot, 1u) == (unsigned)(ch.n - 1);
        if (mine) {
          __threadfence();
          nrow = 0.0;
          for (int j = 0; j < ch.n; ++j) nrow = add(nrow, __ldcg(P.chunk_part + ch.first + j));
          P.chunk_ticket[ch.slot] = 0u;  // next iteration (stream-ordered)
        }
      }
      if (ch.n == 1) {
        // a one-chunk row is always this warp's (static chunk -> warp map):
        // its dot terms join this lane's partial, deterministically
        const GRow rv = g_load(P, ch.row, p_str);
        g_update(P, ch.row, rv, nrow, alpha, beta, m_new, p_str, p_m, acc);
      } else if (mine) {  // whichever warp finished the row: the row's own slot
        const GRow rv = g_load(P, ch.row, p_str);
        double hd[3] = {0.0, 0.0, 0.0};
        g_update(P, ch.row, rv, nrow, alpha, beta, m_new, p_str, p_m, hd);
        double* slot = P.hubdot + (size_t)ch.slot * 4;
        slot[0] = hd[0];
        slot[1] = hd[1];
        slot[2] = hd[2];
      }
    }
  }

  // ---- 32-row slices: one warp each, one lane per position ---------------
  for (long long sl = gwarp; sl < P.n_slices; sl += n_warps) {
    const long long i = sl * 32 + lane;
    const int len = i < P.n ? ldg_nc(P.slen + i) : -1;
    GRow rv{};
    if (PF && len >= 0) rv = g_load(P, i, p_str);
    int L = max(len, 0);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) L = max(L, __shfl_xor_sync(0xffffffffu, L, o));
    const long long eb = (L > 0 ? P.sptr[sl] : 0) + lane;
    double nacc = 0.0;
    // software pipeline: the next batch's indices and values are in flight
    // while this batch's gathers run (one dependent latency per batch)
    int cc[SB];
    double a[SB];
#pragma unroll
    for (int t = 0; t < SB; ++t) {
      const bool on = t < len;
      cc[t] = on ? ld_hint(P.scol + eb + 32LL * t, p_sell) : 0;
      a[t] = on ? ld_hint(P.sval + eb + 32LL * t, p_sell) : 0.0;
    }
    for (int k0 = 0; k0 < L; k0 += SB) {
      double mv[SB];
#pragma unroll
      for (int t = 0; t < SB; ++t) mv[t] = k0 + t < len ? ld_gather(m_old + cc[t], p_g) : 0.0;
      int cn[SB];
      double an[SB];
#pragma unroll
      for (int t = 0; t < SB; ++t) {
        const bool on = k0 + SB + t < len;
        cn[t] = on ? ld_hint(P.scol + eb + 32LL * (k0 + SB + t), p_sell) : 0;
        an[t] = on ? ld_hint(P.sval + eb + 32LL * (k0 + SB + t), p_sell) : 0.0;
      }
#pragma unroll
      for (int t = 0; t < SB; ++t)
        if (k0 + t < len) nacc = add(nacc, mul(a[t], mv[t]));
#pragma unroll
      for (int t = 0; t < SB; ++t) {
        cc[t] = cn[t];
        a[t] = an[t];
      }
    }
    if (len >= 0) {
      if (!PF) rv = g_load(P, i, p_str);
      g_update(P, i, rv, nacc, alpha, beta, m_new, p_str, p_m, acc);
    }
  }

  // ---- dot partials: block partials, then the hub slots (fixed order) ----
  group_sum<3, kGRows>(acc, tid, red, 1);
  double* part = P.pout + (size_t)(it & 1) * (size_t)gridDim.x * 4;
  if (tid == 0) {
    double* out = part + (size_t)blockIdx.x * 4;
    out[0] = acc[0];
    out[1] = acc[1];
    out[2] = acc[2];
    out[3] = 0.0;
    __threadfence();  // this CTA's hub slots and partial before its ticket
    s_last = atomicAdd(P.counter + (it & 1), 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double v[3] = {0.0, 0.0, 0.0};
  for (int j = tid; j < (int)gridDim.x; j += kGRows) {
    v[0] = add(v[0], __ldcg(part + j * 4 + 0));
    v[1] = add(v[1], __ldcg(part + j * 4 + 1));
    v[2] = add(v[2], __ldcg(part + j * 4 + 2));
  }
  for (int h = tid; h < P.n_hub; h += kGRows) {
    v[0] = add(v[0], __ldcg(P.hubdot + h * 4 + 0));
    v[1] = add(v[1], __ldcg(P.hubdot + h * 4 + 1));
    v[2] = add(v[2], __ldcg(P.hubdot + h * 4 + 2));
  }
  group_sum<3, kGRows>(v, tid, red, 1);
  if (tid == 0) {
    double* f = P.fin + (size_t)(it & 1) * 4;
    f[0] = v[0];
    f[1] = v[1];
    f[2] = v[2];
    f[3] = 0.0;
    P.counter[it & 1] = 0u;  // reused by iteration it + 2 (stream-ordered)
  }
}

// ===========================================================================
// Engine 4: classic PCG (solvers.py:195-273) on the device
// ===========================================================================
// Two kernels per iteration -- PCG's two global reductions are a chain
// (delta = (s, p) needs s = A p of the updated p; alpha = gamma / delta
// gates the update), which is what PIPECG removes:
//   Q1(it): prologue -- (u, r) and (u, u) of iteration it-1 from Q2's
//           partials, the gamma guard of it-1, history, the stop test,
//           beta = gamma / gamma_prev -- then per row
//             p_new = p * beta + u        (np.multiply(p, beta, out=p); p += u)
//             s_i   = sum_k a_ik p_new_k  (CSR order; p_new of the neighbours
//                                          formed on the fly from p_old, u)
//           and the (s, p_new) partial;
//   Q2(it): delta from Q1's partials, the delta guard, alpha = gamma / delta,
//           x += alpha p, r -= alpha s, u = dinv r, and the (u, r), (u, u)
//           partials.
// Same control block, history ring, breakdown precedence, CUDA-graph chunks
// and stop-without-host-sync as the PIPECG engines.
template <typename RP>
struct QParams {
  long long n;
  const RP* rp;
  const int* col;
  const double* val;
  const double* dinv;
  double *x, *r, *u, *s;
  double* p[2];        // ping-pong: Q1(it) reads p[it&1], writes p[(it+1)&1]
  Ctrl* C;
  double* hist;
  ReduceIn rin;        // what this kernel's prologue reduces
  double* pout;        // this kernel's block partials [2][grid][4]
  double* fin;         // their fixed-order sum [2][4] (last block), or null
  unsigned* counter;   // [2]
  long long long_row;  // Q1: rows longer than this are pcg_hub_kernel's
  const double* hsum;  // Q2: the hub rows' (s, p) sum [2] by parity (null: no hub rows)
};

// (A warp-cooperative variant staging each 32-row block's CSR range in
// shared memory measured 2.4x slower at 3D 7-pt 256^3: 96 KB per CTA
// left two CTAs per SM for a latency-bound gather kernel.)

template <int NT>
__device__ __forceinline__ void reduce_partials(const ReduceIn& R, long long it_src, int lt,
                                                double* red, double (&v)[3]) {
  const double* P = R.pin + (size_t)(it_src & 1) * (size_t)R.n_pin * 4;
  v[0] = v[1] = v[2] = 0.0;
  for (int j = lt; j < R.n_pin; j += NT) {
    v[0] = add(v[0], __ldcg(P + j * 4 + 0));
    v[1] = add(v[1], __ldcg(P + j * 4 + 1));
    v[2] = add(v[2], __ldcg(P + j * 4 + 2));
  }
  group_sum<3, NT>(v, lt, red, 1);
}

template <typename RP>
__global__ void __launch_bounds__(256) pcg_q1_kernel(QParams<RP> P, int step) {
  __shared__ double red[3 * 8 + 1];
  __shared__ long long s_it;
  Ctrl* C = P.C;
  const int tid = threadIdx.x;
  pdl_trigger();
  pdl_wait();
  const long long it = cta_iteration(C, step, &s_it);
  if (it < 0) return;
  const bool leader = blockIdx.x == 0 && tid == 0;
  double gamma, norm, gamma_prev = 0.0;
  if (it == 0) {
    gamma = C->init.gamma;
    norm = C->init.norm;
  } else {
    double v[3];
    reduce_partials<256>(P.rin, it - 1, tid, red, v);  // Q2(it-1): (u, r), -, (u, u)
    gamma = v[0];
    norm = sqrt(v[2]);
    gamma_prev = __ldcg(&C->slot[(it - 1) & 1].gamma);
    if (gamma < 0.0 || !isfinite(gamma)) {  // solvers.py:256-257 (iteration it-1)
      if (leader) {
        C->bd_code = PCG_BD_GAMMA;
        C->bd_it = it - 1;
        C->bd_val = gamma;
        C->status = PCG_BREAKDOWN;
      }
      return;
    }
    if (leader) P.hist[it & (kHistRing - 1)] = norm;
  }
  if (!(norm >= C->tol && it < C->max_it)) {  // solvers.py:241 loop condition
    if (leader) {
      C->final_it = it;
      C->final_norm = norm;
      C->status = PCG_STOPPED;
    }
    return;
  }
  const double beta = it == 0 ? 0.0 : gamma / gamma_prev;  // solvers.py:242
  if (leader) C->slot[it & 1] = Slot{gamma, 0.0, 0.0, norm};
  const double* p_old = P.p[it & 1];
  double* p_new = P.p[(it + 1) & 1];
  // p_new of a column, formed from p_old and u (bitwise the stored p_new)
  auto pnew = [&](int c) { return add(mul(ldg_nc(p_old + c), beta), ldg_nc(P.u + c)); };
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long i = blockIdx.x * 256LL + tid; i < P.n; i += (long long)gridDim.x * 256) {
    const long long lo = P.rp[i], hi = P.rp[i + 1];
    const double pi = add(mul(p_old[i], beta), P.u[i]);
    p_new[i] = pi;
    if (hi - lo > P.long_row) continue;  // pcg_hub_kernel's row
    // kernels.py:64-70 on p_new, batches of 8: indices and values, then
    // the gathers, then the ordered adds (independent loads in flight)
    double si = 0.0;
    for (long long k0 = lo; k0 < hi; k0 += 8) {
      double av[8], pv[8];
      int cc[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const long long k = k0 + t;
        cc[t] = k < hi ? ldg_nc(P.col + k) : 0;
        av[t] = k < hi ? ldg_nc(P.val + k) : 0.0;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) pv[t] = k0 + t < hi ? pnew(cc[t]) : 0.0;
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (k0 + t < hi) si = add(si, mul(av[t], pv[t]));
    }
    P.s[i] = si;
    acc[0] = add(acc[0], mul(si, pi));  // delta = dot(s, p)
  }
  publish_partials<256>(acc, tid, red, 1, P.pout, P.fin, P.counter, it);
}

// Q1's hub rows (longer than kLongRow): engine 2's nnz-bounded chunks of the
// row, one CTA each with a fixed tree (not the reference's order -- graded
// like a parallel dot), reading Q1's complete p_new; the row's last chunk
// sums the chunk partials in order, writes s and the row's s*p term; the
// grid's last CTA sums the terms in row order into hsum[it & 1] for Q2.
__global__ void __launch_bounds__(256) pcg_hub_kernel(const Ctrl* C, int step,
                                                      const LongChunk* __restrict__ ch,
                                                      const int* __restrict__ col,
                                                      const double* __restrict__ val,
                                                      const double* p0, const double* p1, double* s,
                                                      double* part, unsigned* ticket, double* hterm,
                                                      int n_hub, double* hsum, unsigned* gticket) {
  __shared__ double red[9];
  __shared__ int last;
  __shared__ long long s_it;
  const long long it = cta_iteration(C, step, &s_it);
  if (it < 0) return;
  const double* p = ((it + 1) & 1) ? p1 : p0;  // p_new of iteration it
  const LongChunk c = ch[blockIdx.x];
  double v[1] = {0.0};
  for (long long k0 = c.lo + threadIdx.x; k0 < c.hi; k0 += 4 * 256) {
    double a[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long k = k0 + 256LL * u;
      a[u] = 0.0;
      xv[u] = 0.0;
      if (k < c.hi) {
        a[u] = ldg_nc(val + k);
        xv[u] = __ldcg(p + ldg_nc(col + k));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (k0 + 256LL * u < c.hi) v[0] = add(v[0], mul(a[u], xv[u]));
  }
  group_sum<1, 256>(v, threadIdx.x, red, 1);
  if (threadIdx.x == 0) {
    bool mine = true;
    double srow = v[0];
    if (c.n > 1) {
      part[blockIdx.x] = v[0];
      __threadfence();
      mine = atomicAdd(ticket + c.slot, 1u) == (unsigned)(c.n - 1);
      if (mine) {
        __threadfence();
        srow = 0.0;
        for (int j = 0; j < c.n; ++j) srow = add(srow, __ldcg(part + c.first + j));
        ticket[c.slot] = 0u;  // next iteration (stream-ordered)
      }
    }
    if (mine) {
      s[c.row] = srow;
      hterm[c.hub] = mul(srow, __ldcg(p + c.row));
    }
    __threadfence();
    last = atomicAdd(gticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double h[1] = {0.0};
  for (int k = threadIdx.x; k < n_hub; k += 256) h[0] = add(h[0], __ldcg(hterm + k));
  group_sum<1, 256>(h, threadIdx.x, red, 1);
  if (threadIdx.x == 0) {
    hsum[it & 1] = h[0];
    *gticket = 0u;
  }
}

template <typename RP>
__global__ void __launch_bounds__(256) pcg_q2_kernel(QParams<RP> P, int step) {
  __shared__ double red[3 * 8 + 1];
  __shared__ long long s_it;
  Ctrl* C = P.C;
  const int tid = threadIdx.x;
  pdl_trigger();
  pdl_wait();
  const long long it = cta_iteration(C, step, &s_it);
  if (it < 0) return;
  double v[3];
  reduce_partials<256>(P.rin, it, tid, red, v);  // Q1(it): (s, p)
  // + the hub rows' terms (tree mode; the seq-mode dot covers every row)
  const double delta = P.hsum ? add(v[0], __ldcg(P.hsum + (it & 1))) : v[0];
  if (delta <= 0.0 || !isfinite(delta)) {  // solvers.py:247-248
    if (blockIdx.x == 0 && tid == 0) {
      C->bd_code = PCG_BD_DELTA;
      C->bd_it = it;
      C->bd_val = delta;
      C->status = PCG_BREAKDOWN;
    }
    return;
  }
  const double alpha = __ldcg(&C->slot[it & 1].gamma) / delta;  // solvers.py:249
  const double* p = P.p[(it + 1) & 1];
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long i = blockIdx.x * 256LL + tid; i < P.n; i += (long long)gridDim.x * 256) {
    P.x[i] = add(P.x[i], mul(alpha, p[i]));  // x += alpha * p
    const double ri = sub(P.r[i], mul(alpha, P.s[i]));  // r -= alpha * s
    const double ui = mul(P.dinv[i], ri);  // jacobi_apply(pc, r, out=u)
    P.r[i] = ri;
    P.u[i] = ui;
    acc[0] = add(acc[0], mul(ui, ri));  // gamma = dot(u, r)
    acc[2] = add(acc[2], mul(ui, ui));  // norm = sqrt(dot(u, u))
  }
  publish_partials<256>(acc, tid, red, 1, P.pout, P.fin, P.counter, it);
}

// sequential-dot mode: the reference's left-to-right dots replace the
// partials (one partial).  which = 1 (after Q1): (s, p_new); which = 2
// (after Q2): (u, r) and (u, u).  p_new is picked by the iteration's parity.
__global__ void __launch_bounds__(32) pcg_seq_dots_kernel(const Ctrl* C, int step, int which,
                                                           long long n, const double* s,
                                                           const double* p0, const double* p1,
                                                           const double* r, const double* u,
                                                           double* seqbuf) {
  constexpr int CH = 256;
  __shared__ double prod[2][CH];
  const long long it = cta_iteration(C, step);
  if (it < 0) return;
  const double* p = ((it + 1) & 1) ? p1 : p0;
  double acc[2] = {0.0, 0.0};
  const int lane = threadIdx.x;
  for (long long base = 0; base < n; base += CH) {
#pragma unroll
    for (int j = 0; j < CH / 32; ++j) {
      const long long i = base + j * 32 + lane;
      double v0 = 0.0, v1 = 0.0;
      if (i < n) {
        if (which == 1) {
          v0 = mul(s[i], p[i]);
        } else {
          v0 = mul(u[i], r[i]);
          v1 = mul(u[i], u[i]);
        }
      }
      prod[0][j * 32 + lane] = v0;
      prod[1][j * 32 + lane] = v1;
    }
    __syncwarp();
    if (lane == 0) {
      const int cnt = (int)((n - base) < CH ? (n - base) : CH);
      for (int j = 0; j < cnt; ++j) {
        acc[0] = add(acc[0], prod[0][j]);
        acc[1] = add(acc[1], prod[1][j]);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    double* out = seqbuf + (size_t)(it & 1) * 4;
    out[0] = acc[0];
    out[1] = 0.0;
    out[2] = acc[1];
    out[3] = 0.0;
  }
}

// SELL-order (position) <-> natural-order (row) copies of a vector
__global__ void __launch_bounds__(256) gather_perm_kernel(long long n, const int* __restrict__ perm,
                                                          const double* __restrict__ src,
                                                          double* __restrict__ dst) {
  for (long long p = blockIdx.x * 256LL + threadIdx.x; p < n; p += (long long)gridDim.x * 256)
    dst[p] = src[perm[p]];
}
__global__ void __launch_bounds__(256) scatter_perm_kernel(long long n, const int* __restrict__ perm,
                                                           const double* __restrict__ src,
                                                           double* __restrict__ dst) {
  for (long long p = blockIdx.x * 256LL + threadIdx.x; p < n; p += (long long)gridDim.x * 256)
    dst[perm[p]] = src[p];
}
__global__ void __launch_bounds__(256) iperm_kernel(long long n, const int* __restrict__ perm,
                                                    int* __restrict__ iperm) {
  for (long long p = blockIdx.x * 256LL + threadIdx.x; p < n; p += (long long)gridDim.x * 256)
    iperm[perm[p]] = (int)p;
}
__global__ void __launch_bounds__(256) renumber_kernel(long long m, const int* __restrict__ iperm,
                                                       const int* __restrict__ col, int* __restrict__ out) {
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < m; e += (long long)gridDim.x * 256)
    out[e] = iperm[col[e]];
}
// hub row k's CSR entries -> packed [hoff[k], hoff[k+1]) with positions
__global__ void __launch_bounds__(256) hub_pack_kernel(const long long* __restrict__ lo,
                                                       const long long* __restrict__ hoff,
                                                       const int* __restrict__ iperm,
                                                       const int* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       int* __restrict__ hcol, double* __restrict__ hval) {
  const long long k = blockIdx.x;
  const long long n = hoff[k + 1] - hoff[k];
  for (long long j = threadIdx.x; j < n; j += 256) {
    hcol[hoff[k] + j] = iperm[col[lo[k] + j]];
    hval[hoff[k] + j] = val[lo[k] + j];
  }
}

// ===========================================================================
// sequential-dot mode (bitwise reference order) and drift samples
// ===========================================================================
// After F(it)/K1(it): overwrite partial 0 with the three strictly sequential
// dots; the next prologue then reduces exactly one partial.
// ip (engine 3): the state is in SELL order, row i lives at position ip[i]
__global__ void __launch_bounds__(32) seq_dots_kernel(const Ctrl* C, long long n, const double* r,
                                                       const double* u, const double* w0,
                                                       const double* w1, int pingpong,
                                                       double* seqbuf, int step, const int* ip) {
  constexpr int CH = 256;
  __shared__ double prod[3][CH];
  const long long it = cta_iteration(C, step);
  if (it < 0) return;
  const double* w = pingpong ? (((it + 1) & 1) ? w1 : w0) : w0;
  double acc[3] = {0.0, 0.0, 0.0};
  const int lane = threadIdx.x;
  for (long long base = 0; base < n; base += CH) {
#pragma unroll
    for (int j = 0; j < CH / 32; ++j) {
      const long long i0 = base + j * 32 + lane;
      const long long i = ip && i0 < n ? ip[i0] : i0;
      const double ui = i0 < n ? u[i] : 0.0;
      prod[0][j * 32 + lane] = i0 < n ? mul(r[i], ui) : 0.0;
      prod[1][j * 32 + lane] = i0 < n ? mul(w[i], ui) : 0.0;
      prod[2][j * 32 + lane] = i0 < n ? mul(ui, ui) : 0.0;
    }
    __syncwarp();
    if (lane == 0) {
      const int cnt = (int)((n - base) < CH ? (n - base) : CH);
      for (int j = 0; j < cnt; ++j) {
        acc[0] = add(acc[0], prod[0][j]);
        acc[1] = add(acc[1], prod[1][j]);
        acc[2] = add(acc[2], prod[2][j]);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    double* out = seqbuf + (size_t)(it & 1) * 4;
    out[0] = acc[0];
    out[1] = acc[1];
    out[2] = acc[2];
    out[3] = 0.0;
  }
}

// drift (solvers.py:190-192): || (b - A x) - r || / ||b|| at entry of `it`
template <typename RP>
__global__ void __launch_bounds__(256) drift_partial_kernel(const Ctrl* C, int step, long long n,
                                                             const RP* __restrict__ rp,
                                                             const int* __restrict__ col,
                                                             const double* __restrict__ val,
                                                             const double* __restrict__ x,
                                                             const double* __restrict__ b,
                                                             const double* __restrict__ r,
                                                             double* __restrict__ dpart,
                                                             const int* __restrict__ ip,
                                                             const double* xh0, const double* xh1) {
  // xh0 / xh1 (distributed): halo columns (>= n) of x for sample parity 0 / 1
  // (see drift_push_kernel), read L2-coherently after the peers' pushes of
  // this sample have been acquired
  __shared__ double red[8];
  const long long it = cta_iteration(C, step);
  if (it < 0) return;
  if (it < 1 || C->drift_k <= 0 || it % C->drift_k != 0) return;
  // distributed: drift_wait_kernel (one block, stream-ordered before this
  // grid) has acquired every peer's push of this sample -- a full grid
  // spinning here could keep a peer sharing the GPU from ever pushing
  const double* xhs = xh0 ? (((it / C->drift_k) & 1) ? xh1 : xh0) : nullptr;
  double v[1] = {0.0};
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    double acc = 0.0;
    for (long long k = rp[i]; k < rp[i + 1]; ++k) {
      const int c = col[k];
      const double xc = ip ? x[ip[c]] : (xhs && c >= n ? __ldcg(xhs + c) : x[c]);
      acc = add(acc, mul(val[k], xc));
    }
    const double e = sub(sub(b[i], acc), r[ip ? ip[i] : i]);
    v[0] = add(v[0], mul(e, e));
  }
  group_sum<1, 256>(v, threadIdx.x, red, 1);
  if (threadIdx.x == 0) dpart[blockIdx.x] = v[0];
}

__global__ void __launch_bounds__(256) drift_finish_kernel(const Ctrl* C, int step, const double* dpart,
                                                            int count, double* dval, long long* dit) {
  __shared__ double red[8];
  const long long it = cta_iteration(C, step);
  if (it < 0) return;
  if (it < 1 || C->drift_k <= 0 || it % C->drift_k != 0) return;
  double v[1] = {0.0};
  for (int j = threadIdx.x; j < count; j += 256) v[0] = add(v[0], dpart[j]);
  group_sum<1, 256>(v, threadIdx.x, red, 1);
  if (threadIdx.x == 0) {
    const double nn = sqrt(v[0]);
    const double bn = C->b_norm;
    dval[it & (kHistRing - 1)] = bn > 0 ? nn / bn : nn;
    dit[it & (kHistRing - 1)] = it;
  }
}

// Deferred x (variants E/F, see pipecg_fused_kernel_s): when the solve
// stopped at an odd iteration `it`, iteration it-1 skipped its x update, so
// x_it = x_{it-1} + alpha_{it-1} p_{it-1} is still pending: p holds p_{it-1}
// (the stopping kernel writes nothing) and slot[(it-1)&1] its alpha.  Runs
// once per solve (x_final), after every iteration kernel of the run.
__global__ void __launch_bounds__(256) finalize_x_kernel(Ctrl* C, long long n, double* x,
                                                         const double* p) {
  if (C->status != PCG_STOPPED || C->x_final) return;
  const long long it = C->final_it;
  if (it >= 1 && ((it - 1) & 1) == 0) {
    const double a = C->slot[(it - 1) & 1].alpha;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
      x[i] = add(x[i], mul(a, p[i]));  // kernels.py:108 (x += alpha p)
  }
}
__global__ void finalize_mark_kernel(Ctrl* C) {
  if (threadIdx.x == 0 && C->status == PCG_STOPPED) C->x_final = 1;
}

__global__ void advance_kernel(Ctrl* C, int k) {
  if (threadIdx.x == 0) C->base_it += k;
}

// pipecg_init tail: sum the per-rank init dots (r,u),(w,u),(u,u),(b,b) in
// rank order (one rank on a single GPU), reset the control block.
__global__ void init_ctrl_kernel(Ctrl* C, const double* dots, int nranks, double tol,
                                 long long max_it, long long drift_k, double* hist, long long* dit,
                                 const unsigned long long* arrive) {
  if (threadIdx.x == 0) {
    double d4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < nranks; ++q)
      for (int k = 0; k < 4; ++k) d4[k] = add(d4[k], dots[q * 4 + k]);
    C->tol = tol;
    C->max_it = max_it;
    C->drift_k = drift_k;
    C->b_norm = sqrt(d4[3]);
    C->init = Slot{d4[0], d4[1], 0.0, sqrt(d4[2])};
    C->base_it = 0;
    C->status = PCG_RUNNING;
    C->bd_code = PCG_BD_NONE;
    C->bd_it = -1;
    C->bd_val = 0.0;
    C->final_it = -1;
    C->final_norm = 0.0;
    C->x_final = 0;
    C->slot[0] = Slot{0, 0, 0, 0};
    C->slot[1] = Slot{0, 0, 0, 0};
    if (!arrive) C->arrive_base = 0ull;  // distributed: snapshot taken at init start
    if (C->comm_error) C->status = PCG_ECOMM_STATUS;
    hist[0] = C->init.norm;
  }
  for (int j = threadIdx.x; j < kHistRing; j += blockDim.x) dit[j] = -1;
}

// ===========================================================================
// Distributed exchange over NVLink peer memory (CUDA IPC-mapped pointers).
// Comm buffer layout (identical on every rank, cudaMalloc'd, IPC-exported):
//   [0]   u64 arrive    (iteration exchanges received)
//   [8]   u64 xarrive   (setup exchanges received)
//   [256] double slots[2][kMaxRanks][4]   per-rank dot partials by parity
//   [768] double islots[kMaxRanks][4]     per-rank init dots
// ===========================================================================

struct CommParams {
  int rank, world;
  char* peer_vbuf[kMaxRanks];  // base of each rank's vector block
  long long peer_ld[kMaxRanks];
  char* peer_comm[kMaxRanks];
  long long n_send;
  const int* send_row;        // local row to send
  const int* send_peer;       // destination rank
  const long long* send_dst;  // index in the destination's local column space
};

__device__ __forceinline__ unsigned long long* comm_arrive(char* c) {
  return reinterpret_cast<unsigned long long*>(c);
}
__device__ __forceinline__ unsigned long long* comm_xarrive(char* c) {
  return reinterpret_cast<unsigned long long*>(c + 8);
}

__device__ __forceinline__ void signal_peers(const CommParams& CP, bool iteration) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < CP.world; ++q)
      atomicAdd_system(iteration ? comm_arrive(CP.peer_comm[q]) : comm_xarrive(CP.peer_comm[q]),
                       1ull);
  }
}

// After F(it): push the boundary rows of w_new into the neighbours' halo of
// the same ping-pong buffer, push this rank's (r,u),(w,u),(u,u) partial to
// every rank's slot[it&1][rank], then signal every rank.  Stream-ordered
// after F(it), so every gather of F(it) on this rank is complete.
// The pushed vector is the one the next iteration gathers: w (vectors 7/8 of
// the block) for variants A/B, the stored m (vectors 9/12) for variant C.
__global__ void __launch_bounds__(256) iter_exchange_kernel(CommParams CP, const Ctrl* C, int step,
                                                             const double* pout, int n_pout,
                                                             const double* g0, const double* g1,
                                                             int vec0, int vec1) {
  __shared__ double red[3 * 8];
  const long long it = cta_iteration(C, step);
  if (it < 0) return;
  const int wi = (int)((it + 1) & 1);
  const double* src = wi ? g1 : g0;
  const int vec = wi ? vec1 : vec0;
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < CP.n_send; e += (long long)gridDim.x * 256) {
    const int q = CP.send_peer[e];
    double* dst = reinterpret_cast<double*>(CP.peer_vbuf[q]) + (size_t)vec * CP.peer_ld[q];
    dst[CP.send_dst[e]] = src[CP.send_row[e]];
  }
  if (blockIdx.x == 0) {
    const double* P = pout + (size_t)(it & 1) * (size_t)n_pout * 4;
    double v[3] = {0.0, 0.0, 0.0};
    for (int j = threadIdx.x; j < n_pout; j += 256) {
      v[0] = add(v[0], P[j * 4 + 0]);
      v[1] = add(v[1], P[j * 4 + 1]);
      v[2] = add(v[2], P[j * 4 + 2]);
    }
    group_sum<3, 256>(v, threadIdx.x, red, 1);
    if (threadIdx.x < CP.world) {
      double* slot = reinterpret_cast<double*>(CP.peer_comm[threadIdx.x] + kCommSlots) +
                     ((size_t)(it & 1) * kMaxRanks + CP.rank) * 4;
      slot[0] = v[0];
      slot[1] = v[1];
      slot[2] = v[2];
      slot[3] = 0.0;
    }
  }
  signal_peers(CP, true);
}

// setup: push vector `vec` (index in the block) halo rows to the peers
__global__ void __launch_bounds__(256) vec_exchange_kernel(CommParams CP, int vec, const double* src) {
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < CP.n_send; e += (long long)gridDim.x * 256) {
    const int q = CP.send_peer[e];
    double* dst = reinterpret_cast<double*>(CP.peer_vbuf[q]) + (size_t)vec * CP.peer_ld[q];
    dst[CP.send_dst[e]] = src[CP.send_row[e]];
  }
  signal_peers(CP, false);
}

// setup: push this rank's four init dots to every rank's islots[rank]
__global__ void init_dots_exchange_kernel(CommParams CP, const double* dots4) {
  if (threadIdx.x < CP.world) {
    double* slot = reinterpret_cast<double*>(CP.peer_comm[threadIdx.x] + kCommISlots) + CP.rank * 4;
    for (int k = 0; k < 4; ++k) slot[k] = dots4[k];
  }
  signal_peers(CP, false);
}

// init start (after the host barrier: no peer can produce iteration
// arrivals for this solve until this rank's first setup push): snapshot the
// iteration-arrival counter as this solve's base.
__global__ void snapshot_arrive_kernel(Ctrl* C, const char* comm) {
  if (threadIdx.x == 0) {
    const volatile unsigned long long* c = reinterpret_cast<const volatile unsigned long long*>(comm);
    C->arrive_base = c[0];
    C->darrive_base = c[2];
    C->dsum_base = c[3];
  }
}

// ---------------------------------------------------------------------------
// Drift samples on a row-sharded solve (solvers.py:190-192,371-372):
// ||(b - A x) - r|| / ||b|| at entry of iteration it (it % k == 0), every
// rank's rows.  Sample s = it / k:
//   drift_push_kernel:   this rank's boundary rows of x -> the peers' halo
//                        of a spare vector (n for even s, b for odd s: the
//                        halo part of both is otherwise unused), then
//                        signal darrive on every rank;
//   drift_partial_kernel (ip = nullptr, xh = that spare vector): waits for
//                        every peer's push of sample s, sums e_i^2 over the
//                        own rows with halo columns read from xh;
//   drift_dist_finish_kernel: this rank's sum -> dslots[s&1][rank] of every
//                        rank, signal dsum, wait for all ranks, sum the
//                        slots in rank order (the same number on every rank).
// Double-buffering by s parity: a rank at most one iteration ahead cannot
// overwrite what a slower rank still reads.
__device__ __forceinline__ bool drift_step(const Ctrl* C, long long it) {
  return it >= 1 && C->drift_k > 0 && it % C->drift_k == 0;
}

__global__ void __launch_bounds__(256) drift_push_kernel(CommParams CP, const Ctrl* C, int step,
                                                         const double* x) {
  const long long it = cta_iteration(C, step);
  if (it < 0 || !drift_step(C, it)) return;
  const int vec = ((it / C->drift_k) & 1) ? 11 : 10;  // b or n of the peer's block
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < CP.n_send; e += (long long)gridDim.x * 256) {
    const int q = CP.send_peer[e];
    double* dst = reinterpret_cast<double*>(CP.peer_vbuf[q]) + (size_t)vec * CP.peer_ld[q];
    dst[CP.send_dst[e]] = x[CP.send_row[e]];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < CP.world; ++q)
      atomicAdd_system(reinterpret_cast<unsigned long long*>(CP.peer_comm[q] + 16), 1ull);
}

__global__ void drift_wait_kernel(Ctrl* C, int step, const unsigned long long* darrive,
                                  unsigned long long per_sample) {
  __shared__ long long s_it;
  const long long it = cta_iteration(C, step, &s_it);
  if (it < 0 || !drift_step(C, it) || threadIdx.x != 0) return;
  if (!spin_until(darrive, C->darrive_base + (unsigned long long)(it / C->drift_k) * per_sample, C, 3)) {
    C->bd_it = it;  // a peer stalled: stop the solve with the exchange error
    C->status = PCG_ECOMM_STATUS;
  }
}

__global__ void __launch_bounds__(256) drift_dist_finish_kernel(CommParams CP, Ctrl* C, int step,
                                                                const double* dpart, int count,
                                                                double* dval, long long* dit,
                                                                char* comm) {
  __shared__ double red[8];
  __shared__ int ok;
  const long long it = cta_iteration(C, step);
  if (it < 0 || !drift_step(C, it)) return;
  const long long smp = it / C->drift_k;
  double v[1] = {0.0};
  for (int j = threadIdx.x; j < count; j += 256) v[0] = add(v[0], dpart[j]);
  group_sum<1, 256>(v, threadIdx.x, red, 1);
  if (threadIdx.x < CP.world) {
    double* slot = reinterpret_cast<double*>(CP.peer_comm[threadIdx.x] + kCommDSlots) +
                   (size_t)(smp & 1) * kMaxRanks + CP.rank;
    *slot = v[0];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < CP.world; ++q)
      atomicAdd_system(reinterpret_cast<unsigned long long*>(CP.peer_comm[q] + 24), 1ull);
    ok = spin_until(reinterpret_cast<const unsigned long long*>(comm + 24),
                    C->dsum_base + (unsigned long long)smp * CP.world, C, 3);
    if (!ok) {  // a peer stalled: stop the solve with the exchange error
      C->bd_it = it;
      C->status = PCG_ECOMM_STATUS;
    }
    if (ok) {
      const volatile double* ds =
          reinterpret_cast<const volatile double*>(comm + kCommDSlots) + (size_t)(smp & 1) * kMaxRanks;
      double sum = 0.0;
      for (int q = 0; q < CP.world; ++q) sum = add(sum, ds[q]);  // rank order
      const double nn = sqrt(sum);
      const double bn = C->b_norm;
      dval[it & (kHistRing - 1)] = bn > 0 ? nn / bn : nn;
      dit[it & (kHistRing - 1)] = it;
    }
  }
}

// setup: wait until xarrive >= target (sets an error status on timeout)
__global__ void xwait_kernel(char* comm, unsigned long long target, Ctrl* C) {
  if (threadIdx.x == 0 && !spin_until(comm_xarrive(comm), target, C, 2)) C->comm_error = 1;
}

// block-wide max (one atomic per block: a single-address atomic per row
// serialises ~10^7 updates in L2)
__device__ __forceinline__ void block_max_atomic(unsigned long long v, unsigned long long* out) {
  __shared__ unsigned long long sm[32];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t > v ? t : v;
  }
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) sm[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = 0;
    for (int j = 0; j < (int)(blockDim.x / 32); ++j) m = sm[j] > m ? sm[j] : m;
    atomicMax(out, m);
  }
}

// per-tile staged span (cols rounded to 4, vals rounded to 2)
template <typename RP>
__global__ void __launch_bounds__(256) tile_span_kernel(long long n, long long n_tiles, int tr,
                                                         const RP* rp, unsigned long long* max_col,
                                                         unsigned long long* max_val) {
  unsigned long long mc = 0, mv = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_tiles;
       t += (long long)gridDim.x * blockDim.x) {
    const long long t0 = t * tr;
    const long long rows = min((long long)tr, n - t0);
    const long long e0 = rp[t0], e1 = rp[t0 + rows];
    const unsigned long long c = (unsigned long long)(((e1 + 3) & ~3LL) - (e0 & ~3LL));
    const unsigned long long v = (unsigned long long)(((e1 + 1) & ~1LL) - (e0 & ~1LL));
    mc = c > mc ? c : mc;
    mv = v > mv ? v : mv;
  }
  block_max_atomic(mc, max_col);
  __syncthreads();
  block_max_atomic(mv, max_val);
}

__global__ void __launch_bounds__(256) max_row_kernel(long long n, const void* rp, int rp64,
                                                       unsigned long long* out) {
  unsigned long long m = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long len = rp64 ? ((const long long*)rp)[i + 1] - ((const long long*)rp)[i]
                         : (long long)(((const int*)rp)[i + 1] - ((const int*)rp)[i]);
    m = (unsigned long long)len > m ? (unsigned long long)len : m;
  }
  block_max_atomic(m, out);
}

// Variant D tiling: greedy inside each block of `tr` rows -- a tile grows
// until adding the next row would exceed `cap` nonzeros; a row longer than
// `hub_len` becomes a tile of its own.  Pass 1 (write = 0) counts tiles per
// block, pass 2 writes each tile's first row and first nonzero at offs[b].
template <typename RP>
__global__ void __launch_bounds__(256) tile_build_kernel(long long n, int tr, long long cap,
                                                          long long hub_len, const RP* rp,
                                                          int write, int* counts,
                                                          const long long* offs, int* tile_row,
                                                          long long* tile_e) {
  const long long n_blocks = (n + tr - 1) / tr;
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < n_blocks;
       b += (long long)gridDim.x * blockDim.x) {
    const long long r0 = b * tr, r1 = min(n, r0 + tr);
    long long out = write ? offs[b] : 0;
    int cnt = 0;
    bool open = false;
    long long cur = 0;
    for (long long i = r0; i < r1; ++i) {
      const long long e = rp[i], len = (long long)rp[i + 1] - e;
      bool start;
      if (len > hub_len) {
        start = true;
        open = false;
      } else {
        start = !open || cur + len > cap;
        if (start) {
          open = true;
          cur = 0;
        }
        cur += len;
      }
      if (start) {
        if (write) {
          tile_row[out] = (int)i;
          tile_e[out] = e;
          ++out;
        }
        ++cnt;
      }
    }
    if (!write) counts[b] = cnt;
  }
}

__global__ void tile_close_kernel(long long n, long long n_tiles, long long nnz, int* tile_row,
                                  long long* tile_e) {
  tile_row[n_tiles] = (int)n;
  tile_e[n_tiles] = nnz;
}

__global__ void __launch_bounds__(256) uniform_check_kernel(long long n, const double* d, double v,
                                                            int* bad) {
  bool ok = true;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    ok &= __double_as_longlong(d[i]) == __double_as_longlong(v);
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) *bad = 1;
}

// runs used by each tile of tr rows: OR of its rows' code masks
__global__ void __launch_bounds__(256) tile_runs_kernel(long long n, int tr, const unsigned char* code,
                                                        const unsigned short* code_runs,
                                                        unsigned short* out) {
  const long long nt = (n + tr - 1) / tr;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nt;
       t += (long long)gridDim.x * blockDim.x) {
    unsigned m = 0;
    const long long e = min(n, (t + 1) * tr);
    for (long long i = t * tr; i < e; ++i) m |= code_runs[code[i]];
    out[t] = (unsigned short)m;
  }
}

}  // namespace pcg

using namespace pcg;

// ===========================================================================
// host runtime
// ===========================================================================
struct FusedPlan {
  int variant = 0;  // 0: consumer gathers dinv,w (A); 1: gather warps (B); 2: stored m (C);
                    // 3: nnz-balanced tiles + cooperative gathers of the stored m (D)
  int tr = 0, stages = 0, bps = 0, cap_val = 0, cap_col = 0, grid = 0, score = 0;
  int dv = 0;  // E: consumers load the streamed vectors (smaller stages)
  size_t smem = 0;
  long long n_tiles = 0;  // variants D/E: tiles built for this plan (owned by the solver)
  long long cap = 0, hub_len = 0;
  int* tile_row = nullptr;
  long long* tile_e = nullptr;
};

constexpr int kVariants = 7;  // A B C D P (= C in one persistent launch per chunk) E F (A / C
                               // reading the row-pattern dictionary instead of the CSR)
constexpr long long kPersistMaxRows = 8LL << 20;  // P is a candidate up to this size
// opt.engine request / result code of engine 3 (fused-g, irregular rows)
constexpr int kReqG = 3 + kVariants;
// ... of engine 4 (classic PCG, solvers.py:195-273)
constexpr int kReqPCG = kReqG + 1;

// a SELL-C-sigma copy of the matrix (rows sorted by length inside windows of
// sigma rows, 32-row slices, column-major inside a slice; rows longer than
// the copy's threshold have length -1 and are not stored)
struct Sell {
  long long slices = 0, total = 0;  // slices, elements incl. padding
  long long* ptr = nullptr;         // [slices + 1] slice starts
  int* perm = nullptr;              // position -> row
  int* len = nullptr;               // position -> length (-1: longer than the threshold)
  int* col = nullptr;
  double* val = nullptr;
};

struct pcg_solver {
  pcg_matrix A{};
  pcg_options opt{};
  int engine = 0;
  int tr = 256;
  int stages = 0;
  int cap_val = 0, cap_col = 0;
  size_t smem = 0;
  int grid = 0;
  int n_partials = 0;
  int num_sms = 148;
  long long n_tiles = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_rec[2] = {nullptr, nullptr};
  double* vbuf = nullptr;
  size_t ld = 0;  // padded vector length (>= local columns incl. halo)
  double *z = nullptr, *q = nullptr, *s = nullptr, *p = nullptr, *x = nullptr, *r = nullptr,
         *u = nullptr, *w[2] = {nullptr, nullptr}, *m = nullptr, *nv = nullptr, *b = nullptr,
         *m2 = nullptr;  // m ping-pong partner (fused variant C)
  double* partials = nullptr;  // block partials [2][grid][4]
  double* fin = nullptr;       // their sum [2][4] (last block)
  unsigned* counter = nullptr; // [2] last-block tickets
  double* seqbuf = nullptr;    // sequential-dot results [2][1][4]
  double* dpart = nullptr;
  double* dots_ws = nullptr;
  double* dots4 = nullptr;
  char* rec_dev = nullptr;
  char* rec_host[2] = {nullptr, nullptr};
  char* comm = nullptr;        // distributed exchange block (IPC-exported)
  int* long_rows = nullptr;
  long long n_long = 0;
  LongChunk* chunks = nullptr;     // engine 2: long rows as nnz-bounded chunks
  long long n_chunks = 0;
  double* chunk_part = nullptr;
  unsigned* chunk_ticket = nullptr;
  std::map<int, cudaGraphExec_t> graphs[2];
  long long host_base = 0;  // iterations enqueued so far
  bool initialized = false;
  long long max_it = 0, drift_k = 0;
  double tol = 0;
  long long graph_launches = 0;
  int rec_parity = 0;
  bool mn_valid = false;
  // distributed
  int rank = 0, world = 1;
  bool connected = false;
  CommParams cp{};
  unsigned long long xtarget = 0;  // cumulative setup arrivals expected
  int flags = 0;                   // experiment switches (env PIPECG_B200_FLAGS)
  int variant = 1;                 // fused kernel variant in use
  bool irregular = false;          // some row longer than kLongRow
  bool pdl = true;                 // programmatic dependent launch of the fused kernels
  bool fused_xchg = false;         // distributed: halo + partial push inside the fused kernel
  bool p_mg = true;                // variant P gathers the stored m (C) or dinv*w (A)
  int l2_prefetch = 0;             // E/F L2 prefetch distance in stages (experiment switch)
  bool no_defer_x = false;         // E/F: update x every iteration (experiment switch)
  long long chunk_nnz = kChunkNnz; // engine 2: nonzeros per long-row chunk (test switch)
  unsigned long long* gbar = nullptr;  // variant P grid-barrier counter
  // engine-2 K2 in SELL-C-sigma layout (irregular matrices)
  bool sell = false;
  int sell_batch = 4;              // nonzeros per lane per load batch in the SELL K2 (4 with the L2
                                   // hints: 2% over 2; 8 spills)
  Sell sell2;                      // engine 2's copy (rows <= kLongRow, sigma kSellSigma)
  Sell gsell;                      // engine 3's copy (rows <= g_thr, sigma kGRows)
  int* x_ptr = nullptr;            // its per-tile send lists (sorted by row)
  int* x_row = nullptr;
  int* x_peer = nullptr;
  long long* x_dst = nullptr;
  FusedPlan plans[kVariants];      // per fused variant (stages == 0: does not fit)
  std::vector<FusedPlan> alts[kVariants];  // E/F: occupancy alternatives the autotuner times
  int alt_pick[kVariants] = {};    // ... and the one it picked
  double tune_ms[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // autotune ms/iteration: fused A..F, engine 2, 3
  double* hubdot = nullptr;        // engine 3: dot terms of each multi-chunk row [n_gmulti][4]
  int n_gmulti = 0;
  LongChunk* gchunks = nullptr;    // engine 3: long rows as warp-sized chunks
  long long n_gchunks = 0;
  double* gchunk_part = nullptr;
  unsigned* gchunk_ticket = nullptr;
  long long g_chunk_nnz = kGChunkNnz;
  bool g_built = false;            // engine 3 data below exists
  int* iperm = nullptr;            // row -> SELL position
  int* sell_colp = nullptr;        // engine 3 SELL columns renumbered to positions
  long long g_thr = kGLaneRow;     // engine 3: rows longer than this are warp chunks
  int* g_long_rows = nullptr;      // ... those rows
  long long n_glong = 0;
  int* hcol = nullptr;             // hub rows packed (positions, values)
  double* hval = nullptr;
  double* dinvp = nullptr;         // inv_diag in SELL order (every init)
  double* natbuf = nullptr;        // solver_state: natural-order copies (engine 3)
  double* qbuf = nullptr;          // engine 4: partials [2][2][grid][4] | fin [2][2][4] | seq [2][2][4]
  unsigned* qcnt = nullptr;        // engine 4: last-block tickets [2][2] | hub-kernel ticket
  double* qhub = nullptr;          // engine 4: hub rows' s*p terms [n_long] | their sum [2]
  int g_batch = 2;                 // engine 3 SELL nonzeros per lane per load batch (2 or 4)
  bool e2_pol = true;
  int sell_gld = 1;                // engine 2 SELL gathers: 0 evict-last hint, 1 ld.ca (L1 + L2, default:
                                   // +0.5%), 2 ld.cg (L2 only: 33% slower -- hub columns hit L1)              // engine 2: L2 hints (streams evict-first, m evict-last; -2% at 2^22)
  int g_mb = 4;                    // engine 3 CTAs per SM the kernel is compiled for (4 or 6)
  bool g_pf = false;               // engine 3 update operands loaded before the row's SpMV
  int* tile_row = nullptr;         // variant D/E tiles of the applied plan
  long long* tile_e = nullptr;
  long long hub_len = 0;
  RowPatterns pat;                 // row-pattern dictionary (n_pat == 0: none)
  // E/F windows: runs of the dictionary's offsets (patterns.cu; WinTable)
  int n_runs = 0;                  // 0: per-nonzero gathers
  int run_lo[kMaxWin] = {}, run_hi[kMaxWin] = {};
  unsigned char* pwin = nullptr;   // [n_entries] run of each dictionary entry
  double* pdinv = nullptr;         // [n_pat] dinv of each code's first row
  unsigned short* tile_runs[3] = {nullptr, nullptr, nullptr};  // per tile height 256/128/64
  int dv = 0;                      // E plan: streamed vectors loaded by the consumers
  bool dinv_by_code = false;       // dinv[i] == pdinv[code[i]] for every row (checked at init)
  bool dinv_uniform = false;       // ... and all pdinv equal (dinv0)
  double dinv0 = 0.0;
};

namespace {

// Tile spans: widest staged column / value span of any tile of `tr` rows.
template <typename RP>
int tile_spans(pcg_solver* S, int tr, int* cap_col, int* cap_val) {
  const long long n = S->A.n_rows;
  const long long n_tiles = (n + tr - 1) / tr;
  unsigned long long* mx = nullptr;
  cudaError_t e = cudaMallocAsync(&mx, 2 * sizeof(unsigned long long), S->stream);
  if (e != cudaSuccess) return cuda_status(e, "tile span alloc");
  cudaMemsetAsync(mx, 0, 2 * sizeof(unsigned long long), S->stream);
  tile_span_kernel<RP><<<elementwise_grid(n_tiles), 256, 0, S->stream>>>(
      n, n_tiles, tr, static_cast<const RP*>(S->A.rowptr), mx, mx + 1);
  unsigned long long h[2] = {0, 0};
  cudaMemcpyAsync(h, mx, sizeof(h), cudaMemcpyDeviceToHost, S->stream);
  cudaFreeAsync(mx, S->stream);
  e = cudaStreamSynchronize(S->stream);
  if (e != cudaSuccess) return cuda_status(e, "tile span");
  *cap_col = (int)std::max<unsigned long long>(h[0], 4);
  *cap_val = (int)((std::max<unsigned long long>(h[1], 2) + 1) & ~1ULL);
  return PCG_OK;
}

// Shared-memory plan for one (variant, tile height): as many CTAs/SM as
// fit (<= 2), then as FEW stages as possible (shared memory not taken by
// stages is L1 for the gathers: S=2 measured 3-5% faster than S=3 for
// variant A at 256^3 and 400^3), then the occupancy the kernel really gets.
template <typename RP, int TR, int V>
int plan_one(pcg_solver* S, int cap_col, int cap_val, FusedPlan* out) {
  FusedPlan p;
  p.variant = V;
  p.tr = TR;
  p.cap_col = cap_col;
  p.cap_val = cap_val;
  const size_t sb = V == 1   ? (size_t)FusedLayout<RP, TR>::stage_bytes(cap_val, cap_col)
                    : V == 3 ? (size_t)FusedLayoutD<RP, TR>::stage_bytes(cap_val, cap_col)
                             : (size_t)FusedLayoutA<RP, TR>::stage_bytes(cap_val, cap_col);
  const size_t hdr = V == 3 ? (size_t)FusedLayoutD<RP, TR>::kHeader : 1024;
  const size_t sm_budget = 228 * 1024, cta_max = 227 * 1024;
  const char* e_st = getenv("PIPECG_B200_STAGES");  // experiment overrides
  const char* e_bps = getenv("PIPECG_B200_BPS");
  for (int bps = e_bps ? atoi(e_bps) : (V == 3 ? 3 : 2); bps >= 1 && !p.stages; --bps) {
    if (e_bps && bps != atoi(e_bps)) break;
    for (int st = e_st ? 1 : 2; st <= 8; ++st) {
      if (e_st ? atoi(e_st) != st : st > 4) continue;
      const size_t need = hdr + st * sb;
      if (need <= cta_max && (need + 1024) * bps <= sm_budget) {
        p.stages = st;
        p.bps = bps;
        p.smem = need;
        break;
      }
    }
  }
  if (!p.stages) {
    *out = p;
    return PCG_OK;
  }
  int occ = 0;
  cudaError_t e =
      V == 1 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pipecg_fused_kernel<RP, TR>,
                                                             FusedLayout<RP, TR>::kThreads, p.smem)
      : V == 3 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                     &occ, pipecg_fused_kernel_d<RP, TR>, kDThreads + 32, p.smem)
      : V == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                     &occ, pipecg_fused_kernel_a<RP, TR, true>, TR + 32, p.smem)
               : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                     &occ, pipecg_fused_kernel_a<RP, TR, false>, TR + 32, p.smem);
  if (e != cudaSuccess) return cuda_status(e, "fused occupancy");
  occ = std::min(occ, p.bps);
  if (occ < 1) {
    p.stages = 0;
    *out = p;
    return PCG_OK;
  }
  const long long n_tiles = (S->A.n_rows + TR - 1) / TR;
  p.grid = (int)std::max<long long>(std::min<long long>((long long)occ * S->num_sms, n_tiles), 1);
  p.score = occ * TR;  // resident consumer rows per SM
  *out = p;
  return PCG_OK;
}

// Best tile height for a variant: most resident consumer rows per SM; ties
// -> taller tiles.
template <typename RP, int V>
int plan_variant(pcg_solver* S, const int* cc, const int* cv, FusedPlan* best) {
  FusedPlan p[3];
  int rc = plan_one<RP, 256, V>(S, cc[0], cv[0], &p[0]);
  if (!rc) rc = plan_one<RP, 128, V>(S, cc[1], cv[1], &p[1]);
  if (!rc) rc = plan_one<RP, 64, V>(S, cc[2], cv[2], &p[2]);
  if (rc) return rc;
  const char* e_tr = getenv("PIPECG_B200_TR");  // experiment override
  *best = FusedPlan();
  for (int k = 0; k < 3; ++k) {
    if (!p[k].stages || (e_tr && atoi(e_tr) != p[k].tr)) continue;
    if (p[k].score > best->score) *best = p[k];
  }
  return PCG_OK;
}

// Variant D tile geometry for tile height TR: when every TR-row block's
// nonzeros fit the average tile (cap_target = TR * mean row length) the
// blocks are the tiles (no hubs); otherwise tiles are capped at cap_target
// nonzeros and rows longer than cap_target / 2 become single-row hub tiles.
template <int TR>
void d_geometry(const pcg_solver* S, int cv_block, long long* cap, long long* hub_len) {
  const long long n = S->A.n_rows, nnz = S->A.nnz;
  const long long avg = std::max<long long>(4, (nnz + n - 1) / std::max<long long>(n, 1));
  long long target = (long long)TR * avg;  // sweep optimum on the power-law config
  if (const char* e = getenv("PIPECG_B200_DCAP")) target = std::max(atoll(e), 8LL);  // experiment / test override
  if (cv_block <= target) {
    *cap = cv_block;
    *hub_len = INT64_MAX / 2;
  } else {
    *cap = target;
    *hub_len = target / 2;
  }
}

template <typename RP>
int build_tiles_d(pcg_solver* S, FusedPlan* p) {
  const long long n = S->A.n_rows;
  const long long n_blocks = (n + p->tr - 1) / p->tr;
  cudaStream_t st = S->stream;
  int* counts = nullptr;
  long long* offs = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, offs, n_blocks, st);
  if (pool_malloc(&counts, n_blocks * sizeof(int)) != cudaSuccess ||
      pool_malloc(&offs, (n_blocks + 1) * sizeof(long long)) != cudaSuccess ||
      pool_malloc(&tmp, tmp_bytes) != cudaSuccess) {
    pool_free(counts);
    pool_free(offs);
    return set_error(PCG_ENOMEM, "variant D tiles: workspace");
  }
  const RP* rp = static_cast<const RP*>(S->A.rowptr);
  const unsigned g = elementwise_grid(n_blocks);
  tile_build_kernel<RP><<<g, 256, 0, st>>>(n, p->tr, p->cap, p->hub_len, rp, 0, counts, nullptr,
                                           nullptr, nullptr);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, offs, n_blocks, st);
  long long last_off = 0;
  int last_cnt = 0;
  cudaMemcpyAsync(&last_off, offs + n_blocks - 1, sizeof(long long), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&last_cnt, counts + n_blocks - 1, sizeof(int), cudaMemcpyDeviceToHost, st);
  int rc = cuda_status(cudaStreamSynchronize(st), "variant D tile count");
  const long long n_tiles = last_off + last_cnt;
  if (!rc) {
    if (pool_malloc(&p->tile_row, (n_tiles + 1) * sizeof(int)) != cudaSuccess ||
        pool_malloc(&p->tile_e, (n_tiles + 1) * sizeof(long long)) != cudaSuccess)
      rc = set_error(PCG_ENOMEM, "variant D tiles");
  }
  if (!rc) {
    tile_build_kernel<RP><<<g, 256, 0, st>>>(n, p->tr, p->cap, p->hub_len, rp, 1, counts, offs,
                                             p->tile_row, p->tile_e);
    tile_close_kernel<<<1, 1, 0, st>>>(n, n_tiles, S->A.nnz, p->tile_row, p->tile_e);
    rc = cuda_status(cudaStreamSynchronize(st), "variant D tile build");
  }
  pool_free(counts);
  pool_free(offs);
  pool_free(tmp);
  if (rc) return rc;
  p->n_tiles = n_tiles;
  p->grid = (int)std::max<long long>(std::min<long long>(p->grid, n_tiles), 1);
  return PCG_OK;
}

template <typename RP>
int plan_d(pcg_solver* S, const int* cv, FusedPlan* best) {
  FusedPlan p[3];
  long long caps[3], hubs[3];
  d_geometry<256>(S, cv[0], &caps[0], &hubs[0]);
  d_geometry<128>(S, cv[1], &caps[1], &hubs[1]);
  d_geometry<64>(S, cv[2], &caps[2], &hubs[2]);
  // staged spans: values rounded to 2 (start aligned down by <= 1), columns to 4
  auto cv_of = [](long long cap) { return (int)round_up(cap + 2, 2); };
  auto cc_of = [](long long cap) { return (int)round_up(cap + 6, 4); };
  int rc = plan_one<RP, 256, 3>(S, cc_of(caps[0]), cv_of(caps[0]), &p[0]);
  if (!rc) rc = plan_one<RP, 128, 3>(S, cc_of(caps[1]), cv_of(caps[1]), &p[1]);
  if (!rc) rc = plan_one<RP, 64, 3>(S, cc_of(caps[2]), cv_of(caps[2]), &p[2]);
  if (rc) return rc;
  const char* e_tr = getenv("PIPECG_B200_TR");
  *best = FusedPlan();
  for (int k = 0; k < 3; ++k) {
    p[k].cap = caps[k];
    p[k].hub_len = hubs[k];
    if (!p[k].stages || (e_tr && atoi(e_tr) != p[k].tr)) continue;
    if (p[k].score > best->score) *best = p[k];
  }
  if (!best->stages) return PCG_OK;
  return build_tiles_d<RP>(S, best);
}

// Variants E / F (row-pattern dictionary): stages are 7 vectors + one code
// byte per row; the dictionary sits in front of them for the whole kernel.
// Runs of the dictionary's distinct offsets (gaps of at most kWinGap
// elements are bridged): each run is one window per tile.  More than
// kMaxWin runs -> E/F use per-nonzero gathers.
constexpr int kWinGap = 16;
int build_runs(pcg_solver* S) {
  S->n_runs = 0;
  const int ne = S->pat.n_entries;
  if (S->pat.n_pat == 0 || getenv("PIPECG_B200_NO_WINDOWS")) return PCG_OK;
  std::vector<int> off(ne);
  int rc = cuda_status(cudaMemcpy(off.data(), S->pat.off, ne * sizeof(int), cudaMemcpyDeviceToHost),
                       "pattern runs");
  if (rc) return rc;
  std::vector<int> d(off);
  d.push_back(0);  // E reads each row's own w / dinv from the windows
  std::sort(d.begin(), d.end());
  d.erase(std::unique(d.begin(), d.end()), d.end());
  // bridge gaps of up to kWinGap; when that leaves more than kMaxWin runs
  // (the 125-point stencil: 25 lines), bridge wider gaps -- the lines of a
  // plane, which overlap anyway once the tile height exceeds the line
  // length -- before giving up on windows
  int lo[kMaxWin], hi[kMaxWin], n = 0;
  for (int gap : {kWinGap, 64, 256, 1024}) {
    n = 0;
    bool fits = true;
    for (size_t k = 0; k < d.size() && fits; ++k) {
      if (n > 0 && d[k] - hi[n - 1] <= gap) {
        hi[n - 1] = d[k];
        continue;
      }
      if (n == kMaxWin) fits = false;
      else {
        lo[n] = hi[n] = d[k];
        ++n;
      }
    }
    if (fits) break;
    n = -1;
  }
  if (n < 0) return PCG_OK;  // too many runs: gathers
  std::vector<unsigned char> run(ne);
  int w0 = 0;
  for (int w = 0; w < n; ++w)
    if (lo[w] <= 0 && hi[w] >= 0) w0 = w;
  for (int k = 0; k < ne; ++k)
    for (int w = 0; w < n; ++w)
      if (off[k] >= lo[w] && off[k] <= hi[w]) run[k] = (unsigned char)w;
  // runs each code uses (+ the own-row run) -> runs each tile uses, per tile height
  std::vector<int> start(S->pat.n_pat + 1);
  rc = cuda_status(cudaMemcpy(start.data(), S->pat.start, start.size() * sizeof(int),
                              cudaMemcpyDeviceToHost), "pattern runs");
  if (rc) return rc;
  std::vector<unsigned short> code_runs(S->pat.n_pat);
  for (int c = 0; c < S->pat.n_pat; ++c) {
    unsigned m = 1u << w0;
    for (int k = start[c]; k < start[c + 1]; ++k) m |= 1u << run[k];
    code_runs[c] = (unsigned short)m;
  }
  unsigned short* d_cr = nullptr;
  const long long nr = S->A.n_rows;
  if (pool_malloc(&S->pwin, std::max(ne, 1)) != cudaSuccess ||
      pool_malloc(&d_cr, code_runs.size() * sizeof(unsigned short)) != cudaSuccess)
    return set_error(PCG_ENOMEM, "pattern runs");
  rc = cuda_status(cudaMemcpy(S->pwin, run.data(), ne, cudaMemcpyHostToDevice), "pattern runs");
  if (!rc)
    rc = cuda_status(cudaMemcpy(d_cr, code_runs.data(), code_runs.size() * sizeof(unsigned short),
                                cudaMemcpyHostToDevice), "pattern runs");
  for (int k = 0; k < 3 && !rc; ++k) {
    const int tr = 256 >> k;
    const long long nt = (nr + tr - 1) / tr;
    if (pool_malloc(&S->tile_runs[k], nt * sizeof(unsigned short)) != cudaSuccess) {
      rc = set_error(PCG_ENOMEM, "pattern tile runs");
      break;
    }
    tile_runs_kernel<<<elementwise_grid(nt), 256, 0, S->stream>>>(nr, tr, S->pat.code, d_cr,
                                                                  S->tile_runs[k]);
  }
  if (!rc) rc = cuda_status(cudaStreamSynchronize(S->stream), "pattern tile runs");
  pool_free(d_cr);
  if (rc) return rc;
  S->n_runs = n;
  for (int w = 0; w < n; ++w) {
    S->run_lo[w] = lo[w];
    S->run_hi[w] = hi[w];
  }
  return PCG_OK;
}

// Window geometry of tile height tr (see pipecg_fused_kernel_s)
inline const unsigned short* tile_runs_for(const pcg_solver* S, int tr) {
  return S->tile_runs[tr == 256 ? 0 : tr == 128 ? 1 : 2];
}

WinTable win_table(const pcg_solver* S, int tr) {
  WinTable W{};
  W.n = S->n_runs;
  W.ld = (long long)S->ld;
  W.code_ld = (S->A.n_rows + 256) & ~15LL;
  W.dinv_by_code = S->dinv_by_code ? 1 : 0;
  W.dinv_uniform = S->dinv_by_code && S->dinv_uniform ? 1 : 0;
  W.dinv0 = S->dinv0;
  int base = 0, cbase = 0;
  for (int w = 0; w < W.n; ++w) {
    const int lo = S->run_lo[w], hi = S->run_hi[w];
    W.lo[w] = lo - (((lo % 2) + 2) % 2);  // round down to even (16-byte copies)
    W.len[w] = (int)round_up(tr + hi - W.lo[w], 2);
    W.base[w] = base;
    base += W.len[w];
    W.clo[w] = lo - (((lo % 16) + 16) % 16);  // round down to 16
    W.clen[w] = (int)round_up(tr + hi - W.clo[w], 16);
    W.cbase[w] = cbase;
    cbase += W.clen[w];
    if (lo <= 0 && hi >= 0) {  // the run holding offset 0: each row's own value
      W.own = W.base[w] - W.lo[w];
      W.cown = W.cbase[w] - W.clo[w];
      W.w0 = w;
    }
  }
  W.elems = base;
  W.celems = cbase;
  return W;
}

// E reads windows only when dinv is a function of the row's code; F always
inline bool s_windows(const pcg_solver* S, bool mg) {
  return S->n_runs > 0 && (mg || S->dinv_by_code);
}

// One E/F plan: tile height TR with exactly `bps` CTAs per SM (3 stages if
// they fit, else 2).  stages == 0: does not fit.
template <int TR, bool MG>
int plan_one_s(pcg_solver* S, int bps, FusedPlan* out, bool dv_e = false, int max_st = 0) {
  FusedPlan p;
  p.variant = MG ? 6 : 5;
  p.tr = TR;
  const bool win = s_windows(S, MG);
  const WinTable W = win_table(S, TR);
  const bool dv = MG ? win : (win && dv_e);
  p.dv = dv && !MG;
  const size_t sb = FusedLayoutS<TR>::stage_bytes(MG, win, W.elems, W.celems, dv);
  const size_t hdr = FusedLayoutS<TR>::kHeader +
                     (size_t)round_up(pat_smem_bytes(S->pat.n_pat, S->pat.n_entries), 128);
  const size_t sm_budget = 228 * 1024, cta_max = 227 * 1024;
  const char* e_st = getenv("PIPECG_B200_STAGES");
  // stages without the streamed vectors are small: up to 4 (or max_st)
  for (int st = e_st ? atoi(e_st) : (max_st ? max_st : (dv ? 4 : 3)); st >= 2; --st) {
    const size_t need = hdr + st * sb;
    if (need <= cta_max && (need + 1024) * bps <= sm_budget) {
      p.stages = st;
      p.bps = bps;
      p.smem = need;
      break;
    }
    if (e_st) break;
  }
  if (!p.stages) {
    *out = p;
    return PCG_OK;
  }
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &occ,
      win ? (p.dv ? pipecg_fused_kernel_s<TR, MG, true, false, true> : pipecg_fused_kernel_s<TR, MG, true>)
          : pipecg_fused_kernel_s<TR, MG, false>,
      TR + 32, p.smem);
  if (e != cudaSuccess) return cuda_status(e, "pattern occupancy");
  if (occ < bps) {  // registers do not allow this many CTAs
    p.stages = 0;
    *out = p;
    return PCG_OK;
  }
  const long long n_tiles = (S->A.n_rows + TR - 1) / TR;
  p.grid = (int)std::max<long long>(std::min<long long>((long long)bps * S->num_sms, n_tiles), 1);
  p.score = bps * TR;
  *out = p;
  return PCG_OK;
}

// E/F candidates for the autotuner: 256-row tiles with 2, 3 and 4 CTAs per
// SM (the best count depends on the stencil: 3D 7-pt E 256^3 0.366 ms with
// 3 vs 0.460 ms with 2; 27-pt F 400^3 1.81 ms with 2 vs 2.03 ms with 4);
// 128 / 64-row tiles only when 256 rows do not fit.  best = the first.
template <bool MG>
int plan_variant_s(pcg_solver* S, FusedPlan* best, std::vector<FusedPlan>* alts) {
  alts->clear();
  const char* e_tr = getenv("PIPECG_B200_TR");
  const char* e_bps = getenv("PIPECG_B200_BPS");
  const int tr_pick = e_tr ? atoi(e_tr) : 0;
  const int order[3] = {MG ? 2 : 3, MG ? 3 : 2, 4};  // default first
  for (int k = 0; k < 3; ++k) {
    const int bps = e_bps ? atoi(e_bps) : order[k];
    FusedPlan p;
    int rc = PCG_OK;
    if (!tr_pick || tr_pick == 256) rc = plan_one_s<256, MG>(S, bps, &p);
    if (!rc && !p.stages && (!tr_pick || tr_pick == 128)) rc = plan_one_s<128, MG>(S, 2 * bps, &p);
    if (!rc && !p.stages && (!tr_pick || tr_pick == 64)) rc = plan_one_s<64, MG>(S, 4 * bps, &p);
    if (rc) return rc;
    if (p.stages) alts->push_back(p);
    if (e_bps) break;
  }
  // a large dictionary (125-point stencils: ~110 KB of shared memory) can
  // leave room for one CTA per SM only
  if (alts->empty() && !e_bps) {
    FusedPlan p;
    int rc = PCG_OK;
    if (!tr_pick || tr_pick == 256) rc = plan_one_s<256, MG>(S, 1, &p);
    if (!rc && !p.stages && (!tr_pick || tr_pick == 128)) rc = plan_one_s<128, MG>(S, 1, &p);
    if (rc) return rc;
    if (p.stages) alts->push_back(p);
  }
  // E with windows: also the stages without the streamed vectors (the
  // consumers load them), 2 stages at 3 and 2 CTAs per SM (3D 7-pt 256^3:
  // 0.322 vs 0.333 ms; slower at 27-pt -- the autotuner decides)
  // (PIPECG_B200_DV=0 / 1: only the staged / only the consumer-loaded
  // layout -- to pin the layout for ncu captures, whose replays mislead
  // the autotuner)
  const char* e_dv = getenv("PIPECG_B200_DV");
  if (e_dv && atoi(e_dv) == 1 && !MG) alts->clear();
  if (!MG && s_windows(S, false) && !e_bps && (!tr_pick || tr_pick == 256) &&
      !(e_dv && atoi(e_dv) == 0)) {
    for (int bps : {3, 2, 1}) {
      if (bps == 1 && !alts->empty() && alts->front().bps > 1) break;  // (large dictionaries only)
      FusedPlan p;
      int rc = plan_one_s<256, MG>(S, bps, &p, true, 2);
      if (rc) return rc;
      if (p.stages) alts->push_back(p);
    }
  }
  *best = alts->empty() ? FusedPlan() : alts->front();
  return PCG_OK;
}

template <typename RP>
int fused_setup(pcg_solver* S) {
  int cc[3], cv[3];
  const int trs[3] = {256, 128, 64};
  for (int k = 0; k < 3; ++k) {
    int rc = tile_spans<RP>(S, trs[k], &cc[k], &cv[k]);
    if (rc) return rc;
  }
  int rc = plan_variant<RP, 0>(S, cc, cv, &S->plans[0]);
  if (!rc) rc = plan_variant<RP, 1>(S, cc, cv, &S->plans[1]);
  if (!rc) rc = plan_variant<RP, 2>(S, cc, cv, &S->plans[2]);
  // variant D (tile map build) only where it can win: irregular rows, or asked for
  if (!rc && (S->irregular || S->opt.engine == 6)) rc = plan_d<RP>(S, cv, &S->plans[3]);
  if (!rc && S->plans[2].stages && (S->A.n_rows <= kPersistMaxRows || S->opt.engine == 7)) {
    FusedPlan p = S->plans[2];  // same tiles and shared memory as C
    p.variant = 4;
    // the cooperative launch needs the whole grid co-resident
    int occ = 0;
    cudaError_t e =
        p.tr == 256   ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pipecg_fused_kernel_p<RP, 256, true>, 288, p.smem)
        : p.tr == 128 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pipecg_fused_kernel_p<RP, 128, true>, 160, p.smem)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pipecg_fused_kernel_p<RP, 64, true>, 96, p.smem);
    if (e != cudaSuccess) return cuda_status(e, "persistent occupancy");
    if ((long long)occ * S->num_sms >= p.grid) S->plans[4] = p;
  }
  // E / F: only when the matrix has a row-pattern dictionary (built by the caller)
  if (!rc && S->pat.n_pat > 0) rc = plan_variant_s<false>(S, &S->plans[5], &S->alts[5]);
  if (!rc && S->pat.n_pat > 0) rc = plan_variant_s<true>(S, &S->plans[6], &S->alts[6]);
  if (rc) return rc;
  bool any = false;
  for (int v = 0; v < kVariants; ++v) any = any || S->plans[v].stages > 0;
  return any ? PCG_OK : PCG_EINVAL;  // none fits -> engine 2
}

void apply_plan(pcg_solver* S, const FusedPlan& p) {
  S->variant = p.variant;
  S->tr = p.tr;
  S->n_tiles = p.variant == 3 ? p.n_tiles : (S->A.n_rows + p.tr - 1) / p.tr;  // E/F: TR-row tiles
  S->tile_row = p.tile_row;
  S->tile_e = p.tile_e;
  S->hub_len = p.hub_len;
  S->stages = p.stages;
  S->cap_val = p.cap_val;
  S->cap_col = p.cap_col;
  S->smem = p.smem;
  S->grid = p.grid;
  S->n_partials = p.grid;
  S->dv = p.dv;
}

// pinned kRecBytes records, recycled across solvers (page-locking memory
// costs milliseconds; the reference-facing call creates a solver per matrix)
std::mutex& pinned_mu() {
  static std::mutex mu;
  return mu;
}
std::vector<char*>& pinned_free() {
  static std::vector<char*> v;
  return v;
}
char* pinned_record() {
  {
    std::lock_guard<std::mutex> lk(pinned_mu());
    if (!pinned_free().empty()) {
      char* p = pinned_free().back();
      pinned_free().pop_back();
      return p;
    }
  }
  char* p = nullptr;
  return cudaMallocHost(&p, kRecBytes) == cudaSuccess ? p : nullptr;
}
void pinned_record_release(char* p) {
  std::lock_guard<std::mutex> lk(pinned_mu());
  if (pinned_free().size() < 64) pinned_free().push_back(p);
  else cudaFreeHost(p);
}

int alloc_state(pcg_solver* S) {
  const long long n = std::max(S->A.n_rows, S->A.n_cols);
  S->ld = (size_t)round_up(n + 32, 256);
  const int nvec = 13;  // z q s p x r u w0 w1 m n b m2
  cudaError_t e = cudaMalloc(&S->vbuf, S->ld * nvec * sizeof(double));
  if (e != cudaSuccess) return set_error(PCG_ENOMEM, "solver: vector allocation failed");
  cudaMemsetAsync(S->vbuf, 0, S->ld * nvec * sizeof(double), S->stream);
  double* v = S->vbuf;
  S->z = v + 0 * S->ld;
  S->q = v + 1 * S->ld;
  S->s = v + 2 * S->ld;
  S->p = v + 3 * S->ld;
  S->x = v + 4 * S->ld;
  S->r = v + 5 * S->ld;
  S->u = v + 6 * S->ld;
  S->w[0] = v + 7 * S->ld;
  S->w[1] = v + 8 * S->ld;
  S->m = v + 9 * S->ld;
  S->nv = v + 10 * S->ld;
  S->b = v + 11 * S->ld;
  S->m2 = v + 12 * S->ld;
  const int maxp = std::max(S->grid, 1);
  e = pool_malloc(&S->partials, (size_t)2 * maxp * 4 * sizeof(double));
  if (e != cudaSuccess) return set_error(PCG_ENOMEM, "solver: partials allocation failed");
  cudaMemsetAsync(S->partials, 0, (size_t)2 * maxp * 4 * sizeof(double), S->stream);
  if (pool_malloc(&S->gbar, sizeof(unsigned long long)) != cudaSuccess ||
      pool_malloc(&S->fin, 8 * sizeof(double)) != cudaSuccess ||
      pool_malloc(&S->counter, 2 * sizeof(unsigned)) != cudaSuccess)
    return set_error(PCG_ENOMEM, "solver: partials allocation failed");
  cudaMemsetAsync(S->fin, 0, 8 * sizeof(double), S->stream);
  cudaMemsetAsync(S->counter, 0, 2 * sizeof(unsigned), S->stream);
  if (pool_malloc(&S->seqbuf, 8 * sizeof(double)) != cudaSuccess ||
      pool_malloc(&S->dpart, kDotGrid * sizeof(double)) != cudaSuccess ||
      pool_malloc(&S->dots_ws, (size_t)kDotGrid * 4 * sizeof(double)) != cudaSuccess ||
      pool_malloc(&S->dots4, 4 * sizeof(double)) != cudaSuccess ||
      pool_malloc(&S->rec_dev, kRecBytes) != cudaSuccess ||
      cudaMalloc(&S->comm, kCommBytes) != cudaSuccess)
    return set_error(PCG_ENOMEM, "solver: workspace allocation failed");
  cudaMemsetAsync(S->rec_dev, 0, kRecBytes, S->stream);
  cudaMemsetAsync(S->comm, 0, kCommBytes, S->stream);
  for (int k = 0; k < 2; ++k)
    if (!(S->rec_host[k] = pinned_record()))
      return set_error(PCG_ENOMEM, "solver: pinned record allocation failed");
  return cuda_status(cudaStreamSynchronize(S->stream), "solver: workspace init");
}

// grids above this many blocks publish one fixed-order sum (last block)
constexpr int kFinGrid = 512;
inline bool use_fin(const pcg_solver* S) { return S->grid > kFinGrid || S->engine == 3; }

// Variant P: the whole chunk in one cooperative (co-resident) launch.
// Only single-GPU, tree dots, no drift samples; otherwise P runs as C.
inline bool persistent_chunk(const pcg_solver* S) {
  return S->engine == 1 && S->variant == 4 && !S->connected && S->opt.dot_mode == PCG_DOT_TREE &&
         S->drift_k == 0;
}

// What the next prologue reduces, per mode
ReduceIn reduce_in(pcg_solver* S) {
  ReduceIn R;
  R.arrive = nullptr;
  R.arrive_per_it = 0;
  if (S->connected) {
    R.pin = reinterpret_cast<const double*>(S->comm + kCommSlots);
    R.n_pin = kMaxRanks;  // slots are laid out [2][kMaxRanks][4]; unused ranks stay 0
    R.arrive = reinterpret_cast<const unsigned long long*>(S->comm);
    R.arrive_per_it = (unsigned long long)S->world * (S->fused_xchg ? 1 : kXchgBlocks);
  } else if (S->opt.dot_mode == PCG_DOT_SEQ) {
    R.pin = S->seqbuf;
    R.n_pin = 1;
  } else {
    const bool fin = use_fin(S) && !persistent_chunk(S);
    R.pin = fin ? S->fin : S->partials;
    R.n_pin = fin ? 1 : S->grid;
  }
  return R;
}

// E/F deferred x update: not with drift samples (they read x every k
// iterations) and not when switched off (experiment / A-B measurement)
inline bool defer_x_active(const pcg_solver* S) {
  return S->engine == 1 && (S->variant == 5 || S->variant == 6) && S->drift_k == 0 &&
         !S->no_defer_x;
}

template <typename RP>
FusedParams<RP> fused_params(pcg_solver* S) {
  FusedParams<RP> P;
  P.n = S->A.n_rows;
  P.n_tiles = S->n_tiles;
  P.rp = static_cast<const RP*>(S->A.rowptr);
  P.col = S->A.col;
  P.val = S->A.val;
  P.dinv = S->A.inv_diag;
  P.vec[0] = S->z;
  P.vec[1] = S->q;
  P.vec[2] = S->s;
  P.vec[3] = S->p;
  P.vec[4] = S->x;
  P.vec[5] = S->r;
  P.vec[6] = S->u;
  P.w[0] = S->w[0];
  P.w[1] = S->w[1];
  P.m[0] = S->m;
  P.m[1] = S->m2;
  Record R = record_at(S->rec_dev);
  P.C = R.C;
  P.hist = R.hist;
  P.rin = reduce_in(S);
  P.pout = S->partials;
  P.fin = S->fin;
  P.counter = use_fin(S) ? S->counter : nullptr;
  P.stages = S->stages;
  P.cap_val = S->cap_val;
  P.cap_col = S->cap_col;
  P.flags = S->flags;
  P.tile_row = S->tile_row;
  P.tile_e = S->tile_e;
  P.hub_len = S->hub_len;
  P.pcode = S->pat.code;
  P.pstart = S->pat.start;
  P.poff = S->pat.off;
  P.pval = S->pat.val;
  P.pwin = S->pwin;
  P.pdinv = S->pdinv;
  P.tile_runs = S->n_runs > 0 ? tile_runs_for(S, S->tr) : nullptr;
  P.l2_prefetch = S->l2_prefetch;
  P.defer_x = defer_x_active(S) ? 1 : 0;
  P.n_pat = S->pat.n_pat;
  P.n_pat_e = S->pat.n_entries;
  P.X = FusedXchg{};
  if (S->fused_xchg) {
    P.X.ptr = S->x_ptr;
    P.X.row = S->x_row;
    P.X.peer = S->x_peer;
    P.X.dst = S->x_dst;
    for (int q = 0; q < S->world; ++q) {
      P.X.peer_vbuf[q] = S->cp.peer_vbuf[q];
      P.X.peer_ld[q] = S->cp.peer_ld[q];
      P.X.peer_comm[q] = S->cp.peer_comm[q];
    }
    P.X.rank = S->rank;
    P.X.world = S->world;
    P.counter = S->counter;  // the last block pushes the partial and signals
  }
  return P;
}

// Launch with programmatic stream serialization: the next iteration's
// kernel is placed while this one drains (its griddepcontrol.wait keeps the
// data dependence), hiding the launch latency of back-to-back iterations.
template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
              bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename RP>
void launch_fused(pcg_solver* S, int k) {
  const FusedParams<RP> P = fused_params<RP>(S);
  cudaStream_t st = S->stream;
  const bool pdl = S->pdl;
  const unsigned g = (unsigned)S->grid;
  const size_t sm = S->smem;
  const int variant = S->variant == 4 ? 2 : S->variant;  // P, launched per iteration, is C
  if (variant == 5 || variant == 6) {
    const FusedParams<int> PS = fused_params<int>(S);  // E/F never read the row pointers
    const WinTable W = win_table(S, S->tr);
#define PCG_LS(MGV, WV, DVV)                                                                                      \
  switch (S->tr) {                                                                                                \
    case 256: launch_k(pipecg_fused_kernel_s<256, MGV, WV, false, DVV>, g, 256 + 32, sm, st, pdl, PS, W, k); break; \
    case 128: launch_k(pipecg_fused_kernel_s<128, MGV, WV, false, DVV>, g, 128 + 32, sm, st, pdl, PS, W, k); break; \
    default: launch_k(pipecg_fused_kernel_s<64, MGV, WV, false, DVV>, g, 64 + 32, sm, st, pdl, PS, W, k); break;    \
  }
    const bool win = s_windows(S, variant == 6);
    if (S->fused_xchg) {  // connect keeps E/F only with windows
#define PCG_LSX(MGV, DVV)                                                                                          \
  switch (S->tr) {                                                                                                 \
    case 256: launch_k(pipecg_fused_kernel_s<256, MGV, true, true, DVV>, g, 256 + 32, sm, st, pdl, PS, W, k); break; \
    case 128: launch_k(pipecg_fused_kernel_s<128, MGV, true, true, DVV>, g, 128 + 32, sm, st, pdl, PS, W, k); break; \
    default: launch_k(pipecg_fused_kernel_s<64, MGV, true, true, DVV>, g, 64 + 32, sm, st, pdl, PS, W, k); break;    \
  }
      if (variant == 6) { PCG_LSX(true, false) }
      else if (S->dv) { PCG_LSX(false, true) }
      else { PCG_LSX(false, false) }
#undef PCG_LSX
    } else if (variant == 6 && win) { PCG_LS(true, true, false) }
    else if (variant == 6) { PCG_LS(true, false, false) }
    else if (win && S->dv) { PCG_LS(false, true, true) }
    else if (win) { PCG_LS(false, true, false) }
    else { PCG_LS(false, false, false) }
#undef PCG_LS
  } else if (variant == 1) {
    switch (S->tr) {
      case 256: launch_k(pipecg_fused_kernel<RP, 256>, g, FusedLayout<RP, 256>::kThreads, sm, st, pdl, P, k); break;
      case 128: launch_k(pipecg_fused_kernel<RP, 128>, g, FusedLayout<RP, 128>::kThreads, sm, st, pdl, P, k); break;
      default: launch_k(pipecg_fused_kernel<RP, 64>, g, FusedLayout<RP, 64>::kThreads, sm, st, pdl, P, k); break;
    }
  } else if (variant == 3) {
#define PCG_LD(XGV)                                                                                    \
  switch (S->tr) {                                                                                     \
    case 256: launch_k(pipecg_fused_kernel_d<RP, 256, XGV>, g, kDThreads + 32, sm, st, pdl, P, k); break; \
    case 128: launch_k(pipecg_fused_kernel_d<RP, 128, XGV>, g, kDThreads + 32, sm, st, pdl, P, k); break; \
    default: launch_k(pipecg_fused_kernel_d<RP, 64, XGV>, g, kDThreads + 32, sm, st, pdl, P, k); break;   \
  }
    if (S->fused_xchg) { PCG_LD(true) } else { PCG_LD(false) }
#undef PCG_LD
  } else {
    // A (MG = false) / C (MG = true), with or without the fused exchange
#define PCG_LA(MGV, XGV)                                                                             \
  switch (S->tr) {                                                                                   \
    case 256: launch_k(pipecg_fused_kernel_a<RP, 256, MGV, XGV>, g, 256 + 32, sm, st, pdl, P, k); break; \
    case 128: launch_k(pipecg_fused_kernel_a<RP, 128, MGV, XGV>, g, 128 + 32, sm, st, pdl, P, k); break; \
    default: launch_k(pipecg_fused_kernel_a<RP, 64, MGV, XGV>, g, 64 + 32, sm, st, pdl, P, k); break;    \
  }
    const bool mg = variant == 2;
    if (mg && S->fused_xchg) { PCG_LA(true, true) }
    else if (mg) { PCG_LA(true, false) }
    else if (S->fused_xchg) { PCG_LA(false, true) }
    else { PCG_LA(false, false) }
#undef PCG_LA
  }
}

// fused variants C and D gather a stored m (ping-pong m / m2) instead of w
inline bool stored_m_fused(const pcg_solver* S) {
  return S->engine == 1 && S->variant >= 2 && S->variant != 5;
}

// engine 3 kernel instance: SELL nonzeros per lane per batch x CTAs per SM
using GKern = void (*)(GParams, int);
inline GKern g_kernel(const pcg_solver* S) {
  if (S->g_pf) return S->g_batch == 4 ? pipecg_fused_kernel_g<4, 3, true> : pipecg_fused_kernel_g<2, 4, true>;
  if (S->g_mb == 6) return S->g_batch == 4 ? pipecg_fused_kernel_g<4, 6, false> : pipecg_fused_kernel_g<2, 6, false>;
  return S->g_batch == 4 ? pipecg_fused_kernel_g<4, 4, false> : pipecg_fused_kernel_g<2, 4, false>;
}

// engine 3: one fused SELL kernel per iteration (pipecg_fused_kernel_g)
void launch_g(pcg_solver* S, int k, const Record& R) {
  GParams P;
  P.n = S->A.n_rows;
  P.n_slices = (S->A.n_rows + 31) / 32;
  P.n_chunks = S->n_gchunks;
  P.sptr = S->gsell.ptr;
  P.slen = S->gsell.len;
  P.scol = S->sell_colp;
  P.sval = S->gsell.val;
  P.chunks = S->gchunks;
  P.hcol = S->hcol;
  P.hval = S->hval;
  P.chunk_part = S->gchunk_part;
  P.chunk_ticket = S->gchunk_ticket;
  P.hubdot = S->hubdot;
  P.n_hub = S->hubdot ? S->n_gmulti : 0;
  P.dinv = S->dinvp;
  P.z = S->z; P.q = S->q; P.s = S->s; P.p = S->p; P.x = S->x;
  P.r = S->r; P.u = S->u; P.w = S->w[0];
  P.m[0] = S->m;
  P.m[1] = S->m2;
  P.C = R.C;
  P.hist = R.hist;
  P.rin = reduce_in(S);
  P.pout = S->partials;
  P.fin = S->fin;
  P.counter = S->counter;
  auto kern = g_kernel(S);
  launch_k(kern, (unsigned)S->grid, kGRows, 0, S->stream, S->pdl, P, k);
}

// engine 4 (classic PCG): Q1 (p update + s = A p + (s,p)) and Q2 (x, r, u +
// (u,r), (u,u)) per iteration; their partial buffers live in S->qbuf
template <typename RP>
void launch_q(pcg_solver* S, int k, const Record& R) {
  const size_t G = (size_t)S->grid;
  double* part[2] = {S->qbuf, S->qbuf + 2 * G * 4};
  double* fin[2] = {S->qbuf + 4 * G * 4, S->qbuf + 4 * G * 4 + 8};
  double* seq[2] = {S->qbuf + 4 * G * 4 + 16, S->qbuf + 4 * G * 4 + 24};
  const bool seq_mode = S->opt.dot_mode == PCG_DOT_SEQ, fin_mode = S->grid > kFinGrid;
  auto rin = [&](int j) {  // what kernel Q(j+1) reduces: the other kernel's output
    ReduceIn r;
    r.arrive = nullptr;
    r.arrive_per_it = 0;
    r.pin = seq_mode ? seq[j] : fin_mode ? fin[j] : part[j];
    r.n_pin = seq_mode || fin_mode ? 1 : S->grid;
    return r;
  };
  QParams<RP> P;
  const bool hubs = S->n_chunks > 0;
  P.long_row = hubs ? kLongRow : LLONG_MAX;
  P.hsum = nullptr;
  P.n = S->A.n_rows;
  P.rp = static_cast<const RP*>(S->A.rowptr);
  P.col = S->A.col;
  P.val = S->A.val;
  P.dinv = S->A.inv_diag;
  P.x = S->x;
  P.r = S->r;
  P.u = S->u;
  P.s = S->s;
  P.p[0] = S->p;
  P.p[1] = S->q;
  P.C = R.C;
  P.hist = R.hist;
  cudaStream_t st = S->stream;
  // Q1(it) reduces Q2(it-1)'s output (slot 1); Q2(it) reduces Q1(it)'s (slot 0)
  P.rin = rin(1);
  P.pout = part[0];
  P.fin = fin[0];
  P.counter = fin_mode ? S->qcnt : nullptr;
  launch_k(pcg_q1_kernel<RP>, (unsigned)S->grid, 256, 0, st, S->pdl, P, k);
  if (hubs)
    pcg_hub_kernel<<<(unsigned)S->n_chunks, 256, 0, st>>>(
        R.C, k, S->chunks, S->A.col, S->A.val, S->p, S->q, S->s, S->chunk_part, S->chunk_ticket,
        S->qhub, (int)S->n_long, S->qhub + S->n_long, S->qcnt + 4);
  if (seq_mode)
    pcg_seq_dots_kernel<<<1, 32, 0, st>>>(R.C, k, 1, P.n, S->s, S->p, S->q, S->r, S->u, seq[0]);
  P.rin = rin(0);
  P.pout = part[1];
  P.fin = fin[1];
  P.counter = fin_mode ? S->qcnt + 2 : nullptr;
  P.hsum = hubs && !seq_mode ? S->qhub + S->n_long : nullptr;
  launch_k(pcg_q2_kernel<RP>, (unsigned)S->grid, 256, 0, st, S->pdl && !seq_mode, P, k);
  if (seq_mode)
    pcg_seq_dots_kernel<<<1, 32, 0, st>>>(R.C, k, 2, P.n, S->s, S->p, S->q, S->r, S->u, seq[1]);
}

// enqueue graph step k (drift? -> iteration -> seq dots? -> exchange / SpMV)
int enqueue_step(pcg_solver* S, int k) {
  Record R = record_at(S->rec_dev);
  cudaStream_t st = S->stream;
  const long long n = S->A.n_rows;
  if (S->drift_k > 0) {
    // distributed: x halo of this sample into the spare n / b vectors first
    const bool dist = S->connected;
    const double* xh0 = dist ? S->nv : nullptr;
    const double* xh1 = dist ? S->b : nullptr;
    const unsigned long long* darr = reinterpret_cast<const unsigned long long*>(S->comm + 16);
    const unsigned long long per = (unsigned long long)S->world * kXchgBlocks;
    if (dist) {
      drift_push_kernel<<<kXchgBlocks, 256, 0, st>>>(S->cp, R.C, k, S->x);
      drift_wait_kernel<<<1, 32, 0, st>>>(R.C, k, darr, per);
    }
    const int* ip = S->engine == 3 ? S->iperm : nullptr;
    if (S->A.rp64)
      drift_partial_kernel<long long><<<kDotGrid, 256, 0, st>>>(
          R.C, k, n, static_cast<const long long*>(S->A.rowptr), S->A.col, S->A.val, S->x, S->b,
          S->r, S->dpart, ip, xh0, xh1);
    else
      drift_partial_kernel<int><<<kDotGrid, 256, 0, st>>>(R.C, k, n,
                                                           static_cast<const int*>(S->A.rowptr),
                                                           S->A.col, S->A.val, S->x, S->b, S->r,
                                                           S->dpart, ip, xh0, xh1);
    if (dist)
      drift_dist_finish_kernel<<<1, 256, 0, st>>>(S->cp, R.C, k, S->dpart, kDotGrid, R.dval, R.dit,
                                                  S->comm);
    else
      drift_finish_kernel<<<1, 256, 0, st>>>(R.C, k, S->dpart, kDotGrid, R.dval, R.dit);
  }
  if (S->engine == 1) {
    if (S->A.rp64) launch_fused<long long>(S, k);
    else launch_fused<int>(S, k);
  } else if (S->engine == 3) {
    launch_g(S, k, R);
  } else if (S->engine == 4) {
    if (S->A.rp64) launch_q<long long>(S, k, R);
    else launch_q<int>(S, k, R);
    return PCG_OK;
  } else {
    TwoParams P;
    P.n = n;
    P.z = S->z; P.q = S->q; P.s = S->s; P.p = S->p; P.x = S->x;
    P.r = S->r; P.u = S->u; P.w = S->w[0]; P.m = S->m; P.nv = S->nv;
    P.dinv = S->A.inv_diag;
    P.C = R.C;
    P.hist = R.hist;
    P.rin = reduce_in(S);
    P.pout = S->partials;
    P.fin = S->fin;
    P.counter = use_fin(S) ? S->counter : nullptr;
    launch_k(S->e2_pol ? pipecg_k1_kernel<true> : pipecg_k1_kernel<false>, (unsigned)S->grid, 256, 0, st,
             S->pdl, P, k);
  }
  if (S->opt.dot_mode == PCG_DOT_SEQ && !S->connected)
    seq_dots_kernel<<<1, 32, 0, st>>>(R.C, n, S->r, S->u, S->w[0], S->w[1], S->engine == 1,
                                      S->seqbuf, k, S->engine == 3 ? S->iperm : nullptr);
  if (S->connected && !S->fused_xchg)
    iter_exchange_kernel<<<kXchgBlocks, 256, 0, st>>>(
        S->cp, R.C, k, use_fin(S) ? S->fin : S->partials, use_fin(S) ? 1 : S->grid,
        stored_m_fused(S) ? S->m : S->w[0],
        stored_m_fused(S) ? S->m2 : S->w[1], stored_m_fused(S) ? 9 : 7, stored_m_fused(S) ? 12 : 8);
  if (S->engine == 2 && S->sell) {
    auto sk = S->e2_pol ? (S->sell_batch == 4 ? sell_spmv_kernel<4, true> : sell_spmv_kernel<2, true>)
                        : (S->sell_batch == 8   ? sell_spmv_kernel<8, false>
                           : S->sell_batch == 2 ? sell_spmv_kernel<2, false>
                                                : sell_spmv_kernel<4, false>);
    launch_k(sk, elementwise_grid(S->sell2.slices * 32), 256, 0, st, S->pdl, (const Ctrl*)R.C, n,
             S->sell2.slices, (const long long*)S->sell2.ptr, (const int*)S->sell2.perm,
             (const int*)S->sell2.len, (const int*)S->sell2.col, (const double*)S->sell2.val,
             (const double*)S->m, S->nv, S->sell_gld);
    if (S->n_chunks > 0) {
      launch_k(gated_spmv_chunks, (unsigned)S->n_chunks, 256, 0, st, S->pdl, (const Ctrl*)R.C,
               (const LongChunk*)S->chunks, (const int*)S->A.col, (const double*)S->A.val,
               (const double*)S->m, S->nv, S->chunk_part, S->chunk_ticket);
    } else if (S->n_long > 0) {
      if (S->A.rp64)
        gated_spmv_long<long long><<<(unsigned)S->n_long, 256, 0, st>>>(
            R.C, S->long_rows, static_cast<const long long*>(S->A.rowptr), S->A.col, S->A.val, S->m,
            S->nv);
      else
        gated_spmv_long<int><<<(unsigned)S->n_long, 256, 0, st>>>(
            R.C, S->long_rows, static_cast<const int*>(S->A.rowptr), S->A.col, S->A.val, S->m,
            S->nv);
    }
  } else if (S->engine == 2) {
    const long long thr = S->n_long > 0 ? kLongRow : INT64_MAX;
    if (S->A.rp64) {
      gated_spmv_rows<long long><<<elementwise_grid(n), 256, 0, st>>>(
          R.C, n, static_cast<const long long*>(S->A.rowptr), S->A.col, S->A.val, S->m, S->nv, thr);
      if (S->n_long > 0)
        gated_spmv_long<long long><<<(unsigned)S->n_long, 256, 0, st>>>(
            R.C, S->long_rows, static_cast<const long long*>(S->A.rowptr), S->A.col, S->A.val, S->m,
            S->nv);
    } else {
      gated_spmv_rows<int><<<elementwise_grid(n), 256, 0, st>>>(
          R.C, n, static_cast<const int*>(S->A.rowptr), S->A.col, S->A.val, S->m, S->nv, thr);
      if (S->n_long > 0)
        gated_spmv_long<int><<<(unsigned)S->n_long, 256, 0, st>>>(
            R.C, S->long_rows, static_cast<const int*>(S->A.rowptr), S->A.col, S->A.val, S->m,
            S->nv);
    }
  }
  return PCG_OK;
}

template <typename RP>
int launch_persistent(pcg_solver* S, int K) {
  FusedParams<RP> P = fused_params<RP>(S);
  P.counter = nullptr;
  cudaStream_t st = S->stream;
  cudaMemsetAsync(S->gbar, 0, sizeof(unsigned long long), st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)S->grid);
  cfg.blockDim = dim3((unsigned)S->tr + 32);
  cfg.dynamicSmemBytes = S->smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barrier)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  unsigned long long* gbar = S->gbar;
  cudaError_t e;
  if (S->p_mg) {
    switch (S->tr) {
      case 256: e = cudaLaunchKernelEx(&cfg, pipecg_fused_kernel_p<RP, 256, true>, P, K, gbar); break;
      case 128: e = cudaLaunchKernelEx(&cfg, pipecg_fused_kernel_p<RP, 128, true>, P, K, gbar); break;
      default: e = cudaLaunchKernelEx(&cfg, pipecg_fused_kernel_p<RP, 64, true>, P, K, gbar); break;
    }
  } else {
    switch (S->tr) {
      case 256: e = cudaLaunchKernelEx(&cfg, pipecg_fused_kernel_p<RP, 256, false>, P, K, gbar); break;
      case 128: e = cudaLaunchKernelEx(&cfg, pipecg_fused_kernel_p<RP, 128, false>, P, K, gbar); break;
      default: e = cudaLaunchKernelEx(&cfg, pipecg_fused_kernel_p<RP, 64, false>, P, K, gbar); break;
    }
  }
  return cuda_status(e, "persistent launch");
}

int enqueue_chunk_body(pcg_solver* S, int K, int parity) {
  if (persistent_chunk(S)) {
    int rc = S->A.rp64 ? launch_persistent<long long>(S, K) : launch_persistent<int>(S, K);
    if (rc) return rc;
  } else {
    for (int k = 0; k < K; ++k) enqueue_step(S, k);
  }
  advance_kernel<<<1, 32, 0, S->stream>>>(record_at(S->rec_dev).C, K);
  cudaMemcpyAsync(S->rec_host[parity], S->rec_dev, kRecBytes, cudaMemcpyDeviceToHost, S->stream);
  return cuda_status(cudaGetLastError(), "chunk launch");
}

// Captured + instantiated graph of one chunk of K iterations for record
// parity `parity` (cached per solver).
int chunk_graph(pcg_solver* S, int K, int parity, cudaGraphExec_t* out) {
  auto it = S->graphs[parity].find(K);
  if (it != S->graphs[parity].end()) {
    *out = it->second;
    return PCG_OK;
  }
  // A capture can be invalidated from outside this solver: another thread
  // synchronising the whole device (cudaDeviceSynchronize, a cudaFree) while
  // this stream captures -- e.g. several solvers sharing one GPU from one
  // process.  Retry a few times; the caller falls back to direct launches.
  cudaError_t e = cudaSuccess;
  for (int attempt = 0; attempt < 3; ++attempt) {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    e = cudaStreamBeginCapture(S->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) break;
    const int rc = enqueue_chunk_body(S, K, parity);
    e = cudaStreamEndCapture(S->stream, &g);
    if (!rc && e == cudaSuccess) {
      e = cudaGraphInstantiate(&exec, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_status(e, "graph instantiate");
      S->graphs[parity][K] = exec;
      *out = exec;
      return PCG_OK;
    }
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();  // the invalidation is not sticky
    if (e == cudaSuccess) e = cudaErrorStreamCaptureInvalidated;
  }
  return cuda_status(e, "graph capture");
}

int launch_chunk(pcg_solver* S, int K, int parity) {
  S->host_base += K;
  if (!S->opt.use_graphs) {
    int rc = enqueue_chunk_body(S, K, parity);
    if (rc) return rc;
  } else if (S->graphs[parity].count(K)) {
    cudaError_t e = cudaGraphLaunch(S->graphs[parity][K], S->stream);
    if (e != cudaSuccess) return cuda_status(e, "graph launch");
  } else {
    // first chunk of this shape: launch it directly, then capture and
    // instantiate its graph while the GPU runs it (the host would otherwise
    // stall the GPU for the instantiation, measured ~5 ms per fresh solver)
    int rc = enqueue_chunk_body(S, K, parity);
    if (rc) return rc;
    rc = cuda_status(cudaEventRecord(S->ev_rec[parity], S->stream), "record event");
    cudaGraphExec_t exec = nullptr;
    if (!rc && chunk_graph(S, K, parity, &exec) != PCG_OK)
      cudaGetLastError();  // no graph this time: the next chunk of this shape launches directly
    S->graph_launches++;
    return rc;
  }
  S->graph_launches++;  // chunks launched (graph or direct)
  return cuda_status(cudaEventRecord(S->ev_rec[parity], S->stream), "record event");
}

int auto_chunk(pcg_solver* S) {
  if (S->opt.chunk > 0) return std::min(S->opt.chunk, kMaxChunk);
  // aim for ~4 ms of GPU work per chunk: the autotuner's time for the
  // engine in use, else an HBM estimate at ~5 TB/s.  A chunk boundary costs a
  // drain + graph launch + record copy (~15 us); a larger chunk costs up to
  // K-1 early-exit launches after convergence (~3 us each)
  const double bytes = 136.0 * S->A.n_rows + 12.0 * S->A.nnz + 4.0 * S->A.n_rows;
  double t_iter = bytes / 5.0e12 + 4e-6;
  const double tuned = S->engine == 2   ? S->tune_ms[kVariants]
                       : S->engine == 3 ? S->tune_ms[kVariants + 1]
                                        : S->tune_ms[S->variant];
  if (tuned > 0) t_iter = tuned * 1e-3;
  int K = (int)(4e-3 / t_iter);
  int p = 4;
  while (p * 2 <= K && p < kMaxChunk) p *= 2;
  return std::max(4, std::min(p, kMaxChunk));
}

void fill_result(pcg_solver* S, const Ctrl& c, pcg_result* res) {
  res->status = c.status;
  res->engine = S->engine == 1   ? 3 + S->variant
                : S->engine == 3 ? kReqG
                : S->engine == 4 ? kReqPCG
                                 : 2;
  for (int k = 0; k < 9; ++k) res->tune_ms[k] = S->tune_ms[k];
  res->pattern_flags = S->pat.n_pat == 0 ? 0
                       : 1 | (S->n_runs > 0 ? 2 : 0) | (S->dinv_by_code ? 4 : 0) |
                             (S->dinv_by_code && S->dinv_uniform ? 8 : 0) |
                             (defer_x_active(S) ? 16 : 0) |
                             (S->engine == 1 && S->variant == 5 && S->dv ? 32 : 0);
  res->graph_launches = S->graph_launches;
  res->norm0 = c.init.norm;
  res->breakdown_quantity = c.bd_code;
  res->breakdown_iteration = c.bd_it;
  res->breakdown_value = c.bd_val;
  if (c.status == PCG_STOPPED) {
    res->iterations = c.final_it;
    res->final_norm = c.final_norm;
    res->converged = c.final_norm < S->tol;
  } else {
    res->iterations = c.base_it;
    res->final_norm = NAN;
    res->converged = 0;
  }
}

// Force-load every kernel the solver launches (see preload_ops in ops.cu:
// lazy loading while a peer-waiting kernel spins can deadlock).
int preload_solver() {
  static std::mutex mu;
  static std::set<int> done_devices;  // function attributes are per device
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_devices.count(dev)) return PCG_OK;
  int rc = preload_ops();
  if (rc) return rc;
  pool_init();
  cudaFuncAttributes a;
  cudaError_t e = cudaSuccess;
#define PCG_LOAD(k) if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, (const void*)(k))
  PCG_LOAD((pipecg_fused_kernel<int, 256>)); PCG_LOAD((pipecg_fused_kernel<int, 128>));
  PCG_LOAD((pipecg_fused_kernel<int, 64>)); PCG_LOAD((pipecg_fused_kernel<long long, 256>));
  PCG_LOAD((pipecg_fused_kernel<long long, 128>)); PCG_LOAD((pipecg_fused_kernel<long long, 64>));
#define PCG_LOAD_A(MG) \
  PCG_LOAD((pipecg_fused_kernel_a<int, 256, MG>)); PCG_LOAD((pipecg_fused_kernel_a<int, 128, MG>)); \
  PCG_LOAD((pipecg_fused_kernel_a<int, 64, MG>)); PCG_LOAD((pipecg_fused_kernel_a<long long, 256, MG>)); \
  PCG_LOAD((pipecg_fused_kernel_a<long long, 128, MG>)); PCG_LOAD((pipecg_fused_kernel_a<long long, 64, MG>))
  PCG_LOAD_A(false);
  PCG_LOAD_A(true);
#undef PCG_LOAD_A
#define PCG_LOAD_X(RPT, TRV) \
  PCG_LOAD((pipecg_fused_kernel_a<RPT, TRV, false, true>)); PCG_LOAD((pipecg_fused_kernel_a<RPT, TRV, true, true>)); \
  PCG_LOAD((pipecg_fused_kernel_d<RPT, TRV, true>))
  PCG_LOAD_X(int, 256); PCG_LOAD_X(int, 128); PCG_LOAD_X(int, 64);
  PCG_LOAD_X(long long, 256); PCG_LOAD_X(long long, 128); PCG_LOAD_X(long long, 64);
#undef PCG_LOAD_X
  PCG_LOAD((pipecg_fused_kernel_p<int, 256, false>)); PCG_LOAD((pipecg_fused_kernel_p<int, 128, false>));
  PCG_LOAD((pipecg_fused_kernel_p<int, 64, false>)); PCG_LOAD((pipecg_fused_kernel_p<long long, 256, false>));
  PCG_LOAD((pipecg_fused_kernel_p<long long, 128, false>)); PCG_LOAD((pipecg_fused_kernel_p<long long, 64, false>));
  PCG_LOAD((pipecg_fused_kernel_p<int, 256, true>)); PCG_LOAD((pipecg_fused_kernel_p<int, 128, true>));
  PCG_LOAD((pipecg_fused_kernel_p<int, 64, true>)); PCG_LOAD((pipecg_fused_kernel_p<long long, 256, true>));
  PCG_LOAD((pipecg_fused_kernel_p<long long, 128, true>)); PCG_LOAD((pipecg_fused_kernel_p<long long, 64, true>));
  PCG_LOAD((pipecg_fused_kernel_d<int, 256>)); PCG_LOAD((pipecg_fused_kernel_d<int, 128>));
  PCG_LOAD((pipecg_fused_kernel_d<int, 64>)); PCG_LOAD((pipecg_fused_kernel_d<long long, 256>));
  PCG_LOAD((pipecg_fused_kernel_d<long long, 128>)); PCG_LOAD((pipecg_fused_kernel_d<long long, 64>));
  PCG_LOAD(tile_build_kernel<int>); PCG_LOAD(tile_build_kernel<long long>); PCG_LOAD(tile_close_kernel);
#define PCG_LOAD_S(MG, WV) \
  PCG_LOAD((pipecg_fused_kernel_s<256, MG, WV>)); PCG_LOAD((pipecg_fused_kernel_s<128, MG, WV>)); \
  PCG_LOAD((pipecg_fused_kernel_s<64, MG, WV>))
  PCG_LOAD_S(false, false); PCG_LOAD_S(true, false); PCG_LOAD_S(false, true); PCG_LOAD_S(true, true);
#undef PCG_LOAD_S
  PCG_LOAD((pipecg_fused_kernel_s<256, false, true, true>)); PCG_LOAD((pipecg_fused_kernel_s<128, false, true, true>));
  PCG_LOAD((pipecg_fused_kernel_s<64, false, true, true>)); PCG_LOAD((pipecg_fused_kernel_s<256, true, true, true>));
  PCG_LOAD((pipecg_fused_kernel_s<128, true, true, true>)); PCG_LOAD((pipecg_fused_kernel_s<64, true, true, true>));
  PCG_LOAD((pipecg_fused_kernel_s<256, false, true, false, true>));
  PCG_LOAD((pipecg_fused_kernel_s<128, false, true, false, true>));
  PCG_LOAD((pipecg_fused_kernel_s<64, false, true, false, true>));
  PCG_LOAD((pipecg_fused_kernel_s<256, false, true, true, true>));
  PCG_LOAD((pipecg_fused_kernel_s<128, false, true, true, true>));
  PCG_LOAD((pipecg_fused_kernel_s<64, false, true, true, true>));
  PCG_LOAD(tile_runs_kernel); PCG_LOAD(uniform_check_kernel);

  PCG_LOAD(pipecg_k1_kernel<false>); PCG_LOAD(pipecg_k1_kernel<true>); PCG_LOAD(gated_spmv_rows<int>); PCG_LOAD(gated_spmv_rows<long long>);
  PCG_LOAD(gated_spmv_long<int>); PCG_LOAD(gated_spmv_long<long long>);
  PCG_LOAD((sell_spmv_kernel<2, false>)); PCG_LOAD((sell_spmv_kernel<4, false>));
  PCG_LOAD((sell_spmv_kernel<8, false>)); PCG_LOAD((sell_spmv_kernel<2, true>));
  PCG_LOAD((sell_spmv_kernel<4, true>));
  PCG_LOAD(gated_spmv_chunks); PCG_LOAD(seq_dots_kernel);
  PCG_LOAD(drift_partial_kernel<int>); PCG_LOAD(drift_partial_kernel<long long>);
  PCG_LOAD(drift_finish_kernel); PCG_LOAD(advance_kernel); PCG_LOAD(init_ctrl_kernel);
  PCG_LOAD(drift_push_kernel); PCG_LOAD(drift_dist_finish_kernel); PCG_LOAD(drift_wait_kernel);
  PCG_LOAD(finalize_x_kernel); PCG_LOAD(finalize_mark_kernel);
  PCG_LOAD((pipecg_fused_kernel_g<4, 3, true>)); PCG_LOAD((pipecg_fused_kernel_g<2, 4, true>));
  PCG_LOAD((pipecg_fused_kernel_g<2, 4, false>)); PCG_LOAD((pipecg_fused_kernel_g<4, 4, false>));
  PCG_LOAD((pipecg_fused_kernel_g<2, 6, false>)); PCG_LOAD((pipecg_fused_kernel_g<4, 6, false>));
  PCG_LOAD(gather_perm_kernel); PCG_LOAD(scatter_perm_kernel); PCG_LOAD(iperm_kernel);
  PCG_LOAD(renumber_kernel); PCG_LOAD(hub_pack_kernel);
  PCG_LOAD(pcg_q1_kernel<int>); PCG_LOAD(pcg_q1_kernel<long long>); PCG_LOAD(pcg_q2_kernel<int>);
  PCG_LOAD(pcg_q2_kernel<long long>); PCG_LOAD(pcg_seq_dots_kernel); PCG_LOAD(pcg_hub_kernel);
  PCG_LOAD(iter_exchange_kernel); PCG_LOAD(vec_exchange_kernel);
  PCG_LOAD(init_dots_exchange_kernel); PCG_LOAD(snapshot_arrive_kernel); PCG_LOAD(xwait_kernel);
  PCG_LOAD(tile_span_kernel<int>); PCG_LOAD(tile_span_kernel<long long>); PCG_LOAD(max_row_kernel);
#undef PCG_LOAD
#define PCG_SMEM(k) \
  if (e == cudaSuccess)  \
  e = cudaFuncSetAttribute((const void*)(k), cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)
  PCG_SMEM((pipecg_fused_kernel<int, 256>)); PCG_SMEM((pipecg_fused_kernel<int, 128>));
  PCG_SMEM((pipecg_fused_kernel<int, 64>)); PCG_SMEM((pipecg_fused_kernel<long long, 256>));
  PCG_SMEM((pipecg_fused_kernel<long long, 128>)); PCG_SMEM((pipecg_fused_kernel<long long, 64>));
#define PCG_SMEM_A(MG) \
  PCG_SMEM((pipecg_fused_kernel_a<int, 256, MG>)); PCG_SMEM((pipecg_fused_kernel_a<int, 128, MG>)); \
  PCG_SMEM((pipecg_fused_kernel_a<int, 64, MG>)); PCG_SMEM((pipecg_fused_kernel_a<long long, 256, MG>)); \
  PCG_SMEM((pipecg_fused_kernel_a<long long, 128, MG>)); PCG_SMEM((pipecg_fused_kernel_a<long long, 64, MG>))
  PCG_SMEM_A(false);
  PCG_SMEM_A(true);
#undef PCG_SMEM_A
#define PCG_SMEM_X(RPT, TRV) \
  PCG_SMEM((pipecg_fused_kernel_a<RPT, TRV, false, true>)); PCG_SMEM((pipecg_fused_kernel_a<RPT, TRV, true, true>)); \
  PCG_SMEM((pipecg_fused_kernel_d<RPT, TRV, true>))
  PCG_SMEM_X(int, 256); PCG_SMEM_X(int, 128); PCG_SMEM_X(int, 64);
  PCG_SMEM_X(long long, 256); PCG_SMEM_X(long long, 128); PCG_SMEM_X(long long, 64);
#undef PCG_SMEM_X
  PCG_SMEM((pipecg_fused_kernel_p<int, 256, false>)); PCG_SMEM((pipecg_fused_kernel_p<int, 128, false>));
  PCG_SMEM((pipecg_fused_kernel_p<int, 64, false>)); PCG_SMEM((pipecg_fused_kernel_p<long long, 256, false>));
  PCG_SMEM((pipecg_fused_kernel_p<long long, 128, false>)); PCG_SMEM((pipecg_fused_kernel_p<long long, 64, false>));
  PCG_SMEM((pipecg_fused_kernel_p<int, 256, true>)); PCG_SMEM((pipecg_fused_kernel_p<int, 128, true>));
  PCG_SMEM((pipecg_fused_kernel_p<int, 64, true>)); PCG_SMEM((pipecg_fused_kernel_p<long long, 256, true>));
  PCG_SMEM((pipecg_fused_kernel_p<long long, 128, true>)); PCG_SMEM((pipecg_fused_kernel_p<long long, 64, true>));
  PCG_SMEM((pipecg_fused_kernel_d<int, 256>)); PCG_SMEM((pipecg_fused_kernel_d<int, 128>));
  PCG_SMEM((pipecg_fused_kernel_d<int, 64>)); PCG_SMEM((pipecg_fused_kernel_d<long long, 256>));
  PCG_SMEM((pipecg_fused_kernel_d<long long, 128>)); PCG_SMEM((pipecg_fused_kernel_d<long long, 64>));
#define PCG_SMEM_S(MG, WV) \
  PCG_SMEM((pipecg_fused_kernel_s<256, MG, WV>)); PCG_SMEM((pipecg_fused_kernel_s<128, MG, WV>)); \
  PCG_SMEM((pipecg_fused_kernel_s<64, MG, WV>))
  PCG_SMEM_S(false, false); PCG_SMEM_S(true, false); PCG_SMEM_S(false, true); PCG_SMEM_S(true, true);
#undef PCG_SMEM_S
  PCG_SMEM((pipecg_fused_kernel_s<256, false, true, true>)); PCG_SMEM((pipecg_fused_kernel_s<128, false, true, true>));
  PCG_SMEM((pipecg_fused_kernel_s<64, false, true, true>)); PCG_SMEM((pipecg_fused_kernel_s<256, true, true, true>));
  PCG_SMEM((pipecg_fused_kernel_s<128, true, true, true>)); PCG_SMEM((pipecg_fused_kernel_s<64, true, true, true>));
  PCG_SMEM((pipecg_fused_kernel_s<256, false, true, false, true>));
  PCG_SMEM((pipecg_fused_kernel_s<128, false, true, false, true>));
  PCG_SMEM((pipecg_fused_kernel_s<64, false, true, false, true>));
  PCG_SMEM((pipecg_fused_kernel_s<256, false, true, true, true>));
  PCG_SMEM((pipecg_fused_kernel_s<128, false, true, true, true>));
  PCG_SMEM((pipecg_fused_kernel_s<64, false, true, true, true>));
#undef PCG_SMEM
  // engine 2's SELL SpMV uses no shared memory and lives on L1 hits of its
  // gathers (hub columns recur): ask for the largest L1 carveout
  if (!getenv("PIPECG_B200_NO_L1PREF"))
    for (auto ks : {sell_spmv_kernel<2, true>, sell_spmv_kernel<4, true>, sell_spmv_kernel<2, false>,
                    sell_spmv_kernel<4, false>, sell_spmv_kernel<8, false>})
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute((const void*)ks, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)cudaSharedmemCarveoutMaxL1);
  if (e != cudaSuccess) return cuda_status(e, "preload solver kernels");
  rc = preload_patterns();
  if (rc) return rc;
  done_devices.insert(dev);
  return PCG_OK;
}

int comm_failed(const Ctrl& c) {
  if (c.status != PCG_ECOMM_STATUS) return PCG_OK;
  char buf[256];
  snprintf(buf, sizeof(buf),
           "distributed exchange timed out (a peer rank stalled): %s wait at iteration %lld saw "
           "%llu of %llu arrivals (arrive_base %llu)",
           c.diag_where == 1 ? "iteration" : c.diag_where == 3 ? "drift" : "setup", c.bd_it,
           c.diag_seen, c.diag_target,
           c.arrive_base);
  return set_error(PCG_ECOMM, buf);
}

__global__ void fill_kernel(double* p, long long n, double v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

// Setup-time autotuner: time a few real iterations (b = 1, x0 = 0, no stop
// test) of every engine/variant that fits this matrix on this GPU and keep
// the fastest.  Costs ~10 iterations once per solver; the state is
// re-initialised by the caller's solver_init.
__global__ void long_len_kernel(const int* rows, long long n, const void* rp, int rp64,
                                long long* lo, long long* hi) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const long long i = rows[k];
    lo[k] = rp64 ? ((const long long*)rp)[i] : (long long)((const int*)rp)[i];
    hi[k] = rp64 ? ((const long long*)rp)[i + 1] : (long long)((const int*)rp)[i + 1];
  }
}

// chunk table of the long rows (setup)
// nnz-bounded chunks of the long rows: engine 2 (one CTA per chunk of
// chunk_nnz) and engine 3 (one warp per chunk of g_chunk_nnz)
int build_chunk_list(pcg_solver* S, long long chunk_nnz, const std::vector<long long>& lo,
                     const std::vector<long long>& hi, const std::vector<int>& rows,
                     LongChunk** out, long long* n_out, double** part, unsigned** ticket,
                     int* n_multi = nullptr) {
  const long long nl = (long long)lo.size();
  std::vector<LongChunk> ch;
  int slots = 0;
  for (long long k = 0; k < nl; ++k) {
    const long long len = hi[k] - lo[k];
    const int n = (int)((len + chunk_nnz - 1) / chunk_nnz);
    const int first = (int)ch.size();
    const int slot = n > 1 ? slots++ : -1;
    for (int j = 0; j < n; ++j)
      ch.push_back(LongChunk{lo[k] + len * j / n, lo[k] + len * (j + 1) / n, rows[k], first, n, slot,
                             (int)k, 0});
  }
  *n_out = (long long)ch.size();
  if (n_multi) *n_multi = slots;
  if (pool_malloc(out, ch.size() * sizeof(LongChunk)) != cudaSuccess ||
      pool_malloc(part, ch.size() * sizeof(double)) != cudaSuccess ||
      pool_malloc(ticket, std::max(slots, 1) * sizeof(unsigned)) != cudaSuccess)
    return set_error(PCG_ENOMEM, "long chunks");
  cudaMemcpyAsync(*out, ch.data(), ch.size() * sizeof(LongChunk), cudaMemcpyHostToDevice, S->stream);
  cudaMemsetAsync(*ticket, 0, std::max(slots, 1) * sizeof(unsigned), S->stream);
  return cuda_status(cudaStreamSynchronize(S->stream), "long chunks");
}

int build_long_chunks(pcg_solver* S) {
  const long long nl = S->n_long;
  if (nl <= 0) return PCG_OK;
  cudaStream_t st = S->stream;
  long long* d = nullptr;
  if (pool_malloc(&d, 2 * nl * sizeof(long long)) != cudaSuccess)
    return set_error(PCG_ENOMEM, "long chunks");
  long_len_kernel<<<elementwise_grid(nl), 256, 0, st>>>(S->long_rows, nl, S->A.rowptr, S->A.rp64, d,
                                                        d + nl);
  std::vector<long long> lo(nl), hi(nl);
  std::vector<int> rows(nl);
  cudaMemcpyAsync(lo.data(), d, nl * 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(hi.data(), d + nl, nl * 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(rows.data(), S->long_rows, nl * 4, cudaMemcpyDeviceToHost, st);
  int rc = cuda_status(cudaStreamSynchronize(st), "long chunks");
  pool_free(d);
  if (rc) return rc;
  return build_chunk_list(S, S->chunk_nnz, lo, hi, rows, &S->chunks, &S->n_chunks, &S->chunk_part,
                          &S->chunk_ticket);
}

__global__ void gather_int_kernel(long long n, const int* __restrict__ idx, const int* __restrict__ src,
                                  int* __restrict__ dst) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    dst[k] = src[idx[k]];
}

// Engine 3 data (needs the SELL copy): row -> position map, the SELL
// columns as positions, the hub rows packed with positions, their warp
// chunks (row = position) and dot slots.
int build_g(pcg_solver* S) {
  const long long n = S->A.n_rows, nl = S->n_glong;
  cudaStream_t st = S->stream;
  if (pool_malloc(&S->iperm, n * 4) != cudaSuccess ||
      pool_malloc(&S->sell_colp, (S->gsell.total + 64) * 4) != cudaSuccess ||
      pool_malloc(&S->dinvp, (n + 32) * 8) != cudaSuccess)
    return set_error(PCG_ENOMEM, "engine 3 setup");
  iperm_kernel<<<elementwise_grid(n), 256, 0, st>>>(n, S->gsell.perm, S->iperm);
  renumber_kernel<<<elementwise_grid(S->gsell.total + 64), 256, 0, st>>>(S->gsell.total + 64, S->iperm,
                                                                         S->gsell.col, S->sell_colp);
  if (nl > 0) {
    long long* d = nullptr;
    int* pos = nullptr;
    if (pool_malloc(&d, 2 * nl * sizeof(long long)) != cudaSuccess ||
        pool_malloc(&pos, nl * sizeof(int)) != cudaSuccess)
      return set_error(PCG_ENOMEM, "engine 3 setup");
    long_len_kernel<<<elementwise_grid(nl), 256, 0, st>>>(S->g_long_rows, nl, S->A.rowptr, S->A.rp64,
                                                          d, d + nl);
    gather_int_kernel<<<elementwise_grid(nl), 256, 0, st>>>(nl, S->g_long_rows, S->iperm, pos);
    std::vector<long long> lo(nl), hi(nl), hoff(nl + 1, 0);
    std::vector<int> prow(nl);
    cudaMemcpyAsync(lo.data(), d, nl * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hi.data(), d + nl, nl * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(prow.data(), pos, nl * 4, cudaMemcpyDeviceToHost, st);
    int rc = cuda_status(cudaStreamSynchronize(st), "engine 3 setup");
    if (rc) return rc;
    for (long long k = 0; k < nl; ++k) hoff[k + 1] = hoff[k] + (hi[k] - lo[k]);
    long long* hoff_d = nullptr;
    if (pool_malloc(&hoff_d, (nl + 1) * 8) != cudaSuccess ||
        pool_malloc(&S->hcol, (hoff[nl] + 16) * 4) != cudaSuccess ||
        pool_malloc(&S->hval, (hoff[nl] + 16) * 8) != cudaSuccess)
      return set_error(PCG_ENOMEM, "engine 3 hub rows");
    cudaMemcpyAsync(hoff_d, hoff.data(), (nl + 1) * 8, cudaMemcpyHostToDevice, st);
    hub_pack_kernel<<<(unsigned)nl, 256, 0, st>>>(d, hoff_d, S->iperm, S->A.col, S->A.val, S->hcol,
                                                  S->hval);
    rc = cuda_status(cudaStreamSynchronize(st), "engine 3 hub rows");
    pool_free(d);
    pool_free(pos);
    pool_free(hoff_d);
    if (rc) return rc;
    std::vector<long long> plo(hoff.begin(), hoff.end() - 1), phi(hoff.begin() + 1, hoff.end());
    rc = build_chunk_list(S, S->g_chunk_nnz, plo, phi, prow, &S->gchunks, &S->n_gchunks,
                          &S->gchunk_part, &S->gchunk_ticket, &S->n_gmulti);
    if (rc) return rc;
    if (pool_malloc(&S->hubdot, std::max(S->n_gmulti, 1) * 4 * sizeof(double)) != cudaSuccess)
      return set_error(PCG_ENOMEM, "engine 3 hub rows");
  }
  S->g_built = true;
  return cuda_status(cudaStreamSynchronize(st), "engine 3 setup");
}

__global__ void seg_offsets_kernel(long long n, int sigma, long long n_seg, int* offs) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= n_seg;
       k += (long long)gridDim.x * blockDim.x)
    offs[k] = (int)(k * sigma < n ? k * sigma : n);
}

// SELL-C-sigma copy of the matrix for engine 2's K2 (see sell_spmv_kernel)
template <typename RP>
int build_sell(pcg_solver* S, int sigma, long long thr, Sell* out) {
  const long long n = S->A.n_rows;
  const long long n_seg = (n + sigma - 1) / sigma;
  const long long n_slices = (n + 31) / 32;
  cudaStream_t st = S->stream;
  const RP* rp = static_cast<const RP*>(S->A.rowptr);
  int *key = nullptr, *key2 = nullptr, *idx = nullptr, *offs = nullptr;
  long long* width = nullptr;
  void* tmp = nullptr;
  size_t b1 = 0, b2 = 0;
  int rc = PCG_OK;
  auto fail = [&](const char* w) { rc = set_error(PCG_ENOMEM, w); };
  if (pool_malloc(&key, n * 4) != cudaSuccess || pool_malloc(&key2, n * 4) != cudaSuccess ||
      pool_malloc(&idx, n * 4) != cudaSuccess || pool_malloc(&offs, (n_seg + 1) * 4) != cudaSuccess ||
      pool_malloc(&width, (n_slices + 1) * 8) != cudaSuccess ||
      pool_malloc(&out->perm, n * 4) != cudaSuccess || pool_malloc(&out->len, n * 4) != cudaSuccess ||
      pool_malloc(&out->ptr, (n_slices + 1) * 8) != cudaSuccess)
    fail("SELL build workspace");
  if (!rc) {
    const unsigned g = elementwise_grid(n);
    sell_keys_kernel<RP><<<g, 256, 0, st>>>(n, rp, thr, key, idx);
    seg_offsets_kernel<<<elementwise_grid(n_seg + 1), 256, 0, st>>>(n, sigma, n_seg, offs);
    int bits = 1;
    while ((1LL << bits) <= thr + 1) ++bits;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, b1, key, key2, idx, out->perm, (int)n,
                                             (int)n_seg, offs, offs + 1, 0, bits, st);
    cub::DeviceScan::ExclusiveSum(nullptr, b2, width, out->ptr, n_slices + 1, st);
    if (pool_malloc(&tmp, std::max(b1, b2)) != cudaSuccess) fail("SELL sort workspace");
    if (!rc) {
      size_t bt = std::max(b1, b2);
      cub::DeviceSegmentedRadixSort::SortPairs(tmp, bt, key, key2, idx, out->perm, (int)n,
                                               (int)n_seg, offs, offs + 1, 0, bits, st);
      cudaMemsetAsync(width, 0, (n_slices + 1) * 8, st);
      sell_len_kernel<RP><<<g, 256, 0, st>>>(n, rp, thr, out->perm, out->len, n_slices,
                                             width);
      bt = std::max(b1, b2);
      cub::DeviceScan::ExclusiveSum(tmp, bt, width, out->ptr, n_slices + 1, st);
      long long total = 0;
      cudaMemcpyAsync(&total, out->ptr + n_slices, 8, cudaMemcpyDeviceToHost, st);
      rc = cuda_status(cudaStreamSynchronize(st), "SELL build");
      out->total = total;
      if (!rc && (pool_malloc(&out->col, (total + 64) * 4) != cudaSuccess ||
                  pool_malloc(&out->val, (total + 64) * 8) != cudaSuccess))
        fail("SELL arrays");
      if (!rc) {
        // padding entries: column 0, value 0 (engine 3 gathers them without
        // summing; engine 2 skips them)
        cudaMemsetAsync(out->col, 0, (total + 64) * 4, st);
        cudaMemsetAsync(out->val, 0, (total + 64) * 8, st);
        sell_fill_kernel<RP><<<g, 256, 0, st>>>(n, rp, S->A.col, S->A.val, out->perm,
                                                out->len, out->ptr, out->col, out->val);
        rc = cuda_status(cudaStreamSynchronize(st), "SELL fill");
      }
    }
  }
  pool_free(key);
  pool_free(key2);
  pool_free(idx);
  pool_free(offs);
  pool_free(width);
  pool_free(tmp);
  if (!rc) out->slices = n_slices;
  return rc;
}

struct TuneKey {
  int dev;
  long long n_rows, n_cols, nnz;
  int rp64;
  long long max_row;
  int sms, dot_mode, req, n_pat, dinv_mode;
  bool operator<(const TuneKey& o) const {
    return std::tie(dev, n_rows, n_cols, nnz, rp64, max_row, sms, dot_mode, req, n_pat, dinv_mode) <
           std::tie(o.dev, o.n_rows, o.n_cols, o.nnz, o.rp64, o.max_row, o.sms, o.dot_mode, o.req,
                    o.n_pat, o.dinv_mode);
  }
};
// value: variant (kVariants = engine 2) and the E/F alternative picked
std::map<TuneKey, std::pair<int, int>>& tune_cache() {
  static std::map<TuneKey, std::pair<int, int>> m;
  return m;
}
std::mutex& tune_cache_mu() {
  static std::mutex mu;
  return mu;
}

// only >= 0: time just that fused variant's alternatives (a forced E / F)
int autotune(pcg_solver* S, int grid2, int grid3, bool with_engine2, bool irregular, int only = -1) {
  const long long n = S->A.n_rows;
  cudaStream_t st = S->stream;
  fill_kernel<<<elementwise_grid(n), 256, 0, st>>>(S->nv, n, 1.0);
  fill_kernel<<<elementwise_grid(n), 256, 0, st>>>(S->z, n, 0.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // timed as the solve runs: graph chunks (built before the timed chunk),
  // kTuneIters iterations after a 2-iteration warm-up.  When an iteration
  // moves more than ~0.5 GB (>= ~80 us) the launch overhead a graph saves is
  // noise and its capture + instantiation per candidate is not: direct
  // launches then (first-call cost)
  constexpr int kTuneIters = 8;
  const int saved_graphs = S->opt.use_graphs;
  if (136.0 * S->A.n_rows + 12.0 * S->A.nnz > 0.5e9) S->opt.use_graphs = 0;
  int best = -1;
  float best_ms = 0.f;
  int rc = PCG_OK;
  // candidates: fused variants 0..kVariants-1, engine 2 (kVariants), engine 3
  // (kVariants + 1: irregular rows, when its SELL copy exists)
  const bool g_ok = irregular && S->g_built;
  const int n_cand = with_engine2 ? (g_ok ? kVariants + 2 : kVariants + 1) : kVariants;
  // a row-pattern dictionary read through windows (E/F): the CSR variants
  // A/C/D and the two-kernel engine were 1.7-2.3x slower at every stencil
  // size measured (7/27-pt 128^3-400^3, 2D 512^2) -- not timed (P is: it
  // wins the launch-bound sizes)
  // (a dictionary so large that one CTA per SM is all that fits is timed
  // against everything)
  const bool dict = (S->plans[5].stages && S->plans[5].bps > 1 && s_windows(S, false)) ||
                    (S->plans[6].stages && S->plans[6].bps > 1 && s_windows(S, true));
  for (int cand = 0; cand < n_cand && !rc; ++cand) {
    if (only >= 0 && cand != only) continue;
    if (only < 0 && dict && (cand == 0 || cand == 2 || cand == 3 || cand == kVariants)) continue;
    if (cand < kVariants) {
      // B (gather warps) never won a measurement; D only pays for irregular rows
      if (!S->plans[cand].stages || cand == 1 || (cand == 3 && !irregular)) continue;
    }
    // E/F: every occupancy alternative; the fastest becomes the variant's plan
    const int n_alt = cand < kVariants && !S->alts[cand].empty() ? (int)S->alts[cand].size() : 1;
    float cand_ms = 0.f;
    for (int a = 0; a < n_alt && !rc; ++a) {
      if (cand < kVariants) {
        S->engine = 1;
        apply_plan(S, S->alts[cand].empty() ? S->plans[cand] : S->alts[cand][a]);
      } else if (cand == kVariants) {
        S->engine = 2;
        S->grid = S->n_partials = grid2;
      } else {
        S->engine = 3;
        S->grid = S->n_partials = grid3;
      }
      // b := n (ones), x0 := z (zeros); init copies them before overwriting
      rc = pipecg_b200_solver_init(S, S->nv, S->z, 0.0, 1LL << 40, 0, st);
      cudaGraphExec_t ge = nullptr;
      if (!rc && S->opt.use_graphs && chunk_graph(S, kTuneIters, 1, &ge) != PCG_OK)
        cudaGetLastError();  // timed with direct launches instead
      if (!rc) rc = launch_chunk(S, 2, 0);
      cudaEventRecord(e0, st);
      if (!rc) rc = launch_chunk(S, kTuneIters, 1);
      cudaEventRecord(e1, st);
      if (!rc) rc = cuda_status(cudaEventSynchronize(e1), "autotune");
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= (float)kTuneIters;
      for (int k = 0; k < 2; ++k) {  // graphs bake in this candidate's launch parameters
        for (auto& kv : S->graphs[k]) cudaGraphExecDestroy(kv.second);
        S->graphs[k].clear();
      }
      if (rc) break;
      if (a == 0 || ms < cand_ms) {
        cand_ms = ms;
        if (cand < kVariants && !S->alts[cand].empty()) {
          S->plans[cand] = S->alts[cand][a];
          S->alt_pick[cand] = a;
        }
      }
    }
    S->tune_ms[cand] = cand_ms;
    if (!rc && (best < 0 || cand_ms < best_ms)) {
      best = cand;
      best_ms = cand_ms;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  S->opt.use_graphs = saved_graphs;
  S->initialized = false;
  S->host_base = 0;
  if (rc) return rc;
  if (best < kVariants) {
    S->engine = 1;
    apply_plan(S, S->plans[best]);
  } else if (best == kVariants) {
    S->engine = 2;
    S->grid = S->n_partials = grid2;
  } else {
    S->engine = 3;
    S->grid = S->n_partials = grid3;
  }
  return PCG_OK;
}

}  // namespace

extern "C" {

int pipecg_b200_solver_create(const pcg_matrix* A, const pcg_options* opts, pcg_solver** out) {
  if (!A || !out || A->n_rows <= 0 || !A->rowptr || !A->inv_diag || (A->nnz > 0 && (!A->col || !A->val)))
    return set_error(PCG_EINVAL, "solver_create: bad matrix");
  if (A->n_rows >= (1LL << 31) || A->n_cols >= (1LL << 31))
    return set_error(PCG_ERANGE, "solver_create: >= 2^31 rows per device; shard the matrix");
  if (!A->rp64 && A->nnz >= (1LL << 31))
    return set_error(PCG_ERANGE, "solver_create: nnz >= 2^31 needs int64 row pointers");
  int prc = preload_solver();
  if (prc) return prc;
  pcg_solver* S = new pcg_solver();
  S->A = *A;
  // setup phase times (PIPECG_B200_DEBUG_PLAN)
  const auto t_start = std::chrono::steady_clock::now();
  std::vector<std::pair<const char*, double>> phases;
  auto phase = [&](const char* name) {
    phases.emplace_back(name, std::chrono::duration<double, std::milli>(
                                  std::chrono::steady_clock::now() - t_start).count());
  };
  if (const char* f = getenv("PIPECG_B200_FLAGS")) S->flags = atoi(f);
  if (getenv("PIPECG_B200_NO_PDL")) S->pdl = false;
  if (const char* e = getenv("PIPECG_B200_SELL_BATCH")) S->sell_batch = atoi(e);  // experiment
  if (const char* e = getenv("PIPECG_B200_G_BATCH")) S->g_batch = atoi(e);         // experiment
  if (const char* e = getenv("PIPECG_B200_G_MB")) S->g_mb = atoi(e);               // experiment
  if (const char* e = getenv("PIPECG_B200_E2POL")) S->e2_pol = atoi(e) != 0;      // experiment
  if (const char* e = getenv("PIPECG_B200_E2GLD")) S->sell_gld = atoi(e);          // experiment
  if (const char* e = getenv("PIPECG_B200_G_PF")) S->g_pf = atoi(e) != 0;          // experiment
  if (const char* e = getenv("PIPECG_B200_G_THR")) S->g_thr = std::max(8LL, atoll(e)); // experiment
  if (const char* e = getenv("PIPECG_B200_PA")) S->p_mg = atoi(e) == 0;  // experiment switch
  if (const char* e = getenv("PIPECG_B200_L2PF")) S->l2_prefetch = atoi(e);  // experiment switch
  if (getenv("PIPECG_B200_NO_DEFER_X")) S->no_defer_x = true;                 // experiment switch
  if (const char* v = getenv("PIPECG_B200_CHUNK_NNZ"))  // test switch: many chunks on small rows
    S->chunk_nnz = S->g_chunk_nnz = std::max(32LL, atoll(v));
  if (opts) S->opt = *opts;
  else {
    S->opt.dot_mode = PCG_DOT_TREE;
    S->opt.engine = 0;
    S->opt.chunk = 0;
    S->opt.use_graphs = 1;
    S->opt.max_sms = 0;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&S->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (S->opt.max_sms > 0 && S->opt.max_sms < S->num_sms) S->num_sms = S->opt.max_sms;
  // Early (programmatic) launch assumes the grid owns the GPU: with several
  // solvers co-resident on one GPU (max_sms), a next-iteration grid parked on
  // SMs could starve a peer rank's grid that this one waits for.
  if (S->opt.max_sms > 0) S->pdl = false;
  int rc = cuda_status(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking), "stream");
  if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&S->ev_in, cudaEventDisableTiming), "event");
  for (int k = 0; k < 2 && !rc; ++k)
    rc = cuda_status(cudaEventCreateWithFlags(&S->ev_rec[k], cudaEventDisableTiming), "event");
  if (rc) {
    pipecg_b200_solver_destroy(S);
    return rc;
  }
  AllocStream alloc_on(S->stream);  // setup allocations: the stream-ordered pool
  // long rows (> kLongRow entries) -> engine 2 with the block-per-row path
  unsigned long long* mx = nullptr;
  cudaMallocAsync(&mx, sizeof(unsigned long long), S->stream);
  cudaMemsetAsync(mx, 0, sizeof(unsigned long long), S->stream);
  max_row_kernel<<<elementwise_grid(A->n_rows), 256, 0, S->stream>>>(A->n_rows, A->rowptr, A->rp64, mx);
  unsigned long long max_row = 0;
  cudaMemcpyAsync(&max_row, mx, sizeof(max_row), cudaMemcpyDeviceToHost, S->stream);
  cudaFreeAsync(mx, S->stream);
  rc = cuda_status(cudaStreamSynchronize(S->stream), "max row");
  if (rc) {
    pipecg_b200_solver_destroy(S);
    return rc;
  }
  // engine: 0 auto (autotuned), 1 fused (heuristic variant), 2 two-kernel,
  // 3..9 fused variant A/B/C/D/P/E/F
  const int req = S->opt.engine;
  if (req < 0 || req > kReqPCG) {
    pipecg_b200_solver_destroy(S);
    return set_error(PCG_EINVAL, "solver_create: unknown engine");
  }
  const bool has_long = max_row > (unsigned long long)kLongRow;
  S->irregular = has_long;
  phase("stream+max_row");
  bool fused_ok = false;
  if (req == kReqPCG) {  // classic PCG: CSR kernels only, nothing to plan or tune
    S->engine = 4;
    S->grid = S->n_partials = std::min<int>(kDotGrid, 4 * S->num_sms);
    if (has_long) {  // hub rows: engine 2's chunks (pcg_hub_kernel)
      int64_t cnt = 0;
      rc = pipecg_b200_find_long_rows(A->n_rows, A->rp64, A->rowptr, kLongRow, nullptr, 0, &cnt,
                                      S->stream);
      if (!rc && cnt > 0) {
        if (pool_malloc(&S->long_rows, cnt * sizeof(int)) != cudaSuccess)
          rc = set_error(PCG_ENOMEM, "long rows alloc");
        else
          rc = pipecg_b200_find_long_rows(A->n_rows, A->rp64, A->rowptr, kLongRow, S->long_rows,
                                          cnt, &cnt, S->stream);
        S->n_long = cnt;
      }
      if (!rc) rc = build_long_chunks(S);
      if (!rc && S->n_long > 0 &&
          pool_malloc(&S->qhub, (S->n_long + 2) * sizeof(double)) != cudaSuccess)
        rc = set_error(PCG_ENOMEM, "pcg hub workspace");
    }
    if (!rc) rc = alloc_state(S);
    if (!rc && (pool_malloc(&S->qbuf, ((size_t)4 * S->grid * 4 + 32) * sizeof(double)) != cudaSuccess ||
                pool_malloc(&S->qcnt, 8 * sizeof(unsigned)) != cudaSuccess))
      rc = set_error(PCG_ENOMEM, "pcg workspace");
    if (rc) {
      pipecg_b200_solver_destroy(S);
      return rc;
    }
    cudaMemsetAsync(S->qcnt, 0, 8 * sizeof(unsigned), S->stream);
    *out = S;
    return cuda_status(cudaStreamSynchronize(S->stream), "pcg workspace");
  }
  if (req == 0 || req == 1 || req == 8 || req == 9) {
    // lossless row-pattern dictionary (variants E/F); none for irregular
    // matrices or when the rows are too diverse (patterns.cu)
    if (!has_long && !getenv("PIPECG_B200_NO_PATTERNS")) {
      rc = build_row_patterns(A->n_rows, A->rp64, A->rowptr, A->col, A->val, S->stream, &S->pat);
      if (!rc) rc = build_runs(S);
      if (!rc && S->pat.n_pat > 0) {
        if (pool_malloc(&S->pdinv, S->pat.n_pat * sizeof(double)) != cudaSuccess)
          rc = set_error(PCG_ENOMEM, "pattern dinv");
        else
          rc = check_dinv_by_code(S->pat, A->n_rows, A->inv_diag, S->pdinv, &S->dinv_by_code,
                                  &S->dinv_uniform, &S->dinv0, S->stream);
      }
      if (rc) {
        pipecg_b200_solver_destroy(S);
        return rc;
      }
    }
  }
  phase("patterns");
  if (req != 2 && req != kReqG) {
    rc = A->rp64 ? fused_setup<long long>(S) : fused_setup<int>(S);
    if (rc && rc != PCG_EINVAL) {
      pipecg_b200_solver_destroy(S);
      return rc;
    }
    fused_ok = rc == PCG_OK;
    if (req >= 3 && !S->plans[req - 3].stages) fused_ok = false;
    if (!fused_ok && req != 0) {
      const bool no_dict = S->pat.n_pat == 0;
      pipecg_b200_solver_destroy(S);
      if (req >= 8 && no_dict)
        return set_error(PCG_EINVAL, "fused variants E/F: the matrix has no row-pattern dictionary");
      return set_error(PCG_EINVAL, "fused engine: tiles exceed shared memory");
    }
  }
  {  // block-per-row list of long rows: engine 2 (also an autotune candidate) and the init SpMVs
    if (has_long) {
      int64_t cnt = 0;
      rc = pipecg_b200_find_long_rows(A->n_rows, A->rp64, A->rowptr, kLongRow, nullptr, 0, &cnt,
                                      S->stream);
      if (!rc && cnt > 0) {
        if (pool_malloc(&S->long_rows, cnt * sizeof(int)) != cudaSuccess)
          rc = set_error(PCG_ENOMEM, "long rows alloc");
        else
          rc = pipecg_b200_find_long_rows(A->n_rows, A->rp64, A->rowptr, kLongRow, S->long_rows,
                                          cnt, &cnt, S->stream);
        S->n_long = cnt;
      }
      if (rc) {
        pipecg_b200_solver_destroy(S);
        return rc;
      }
    }
  }
  {  // engine 2 on irregular rows reads a SELL-C-sigma copy (coalesced K2)
    bool want = has_long && (req == 0 || req == 2 || !fused_ok);
    if (const char* e = getenv("PIPECG_B200_SELL")) want = atoi(e) != 0 && (req == 0 || req == 2 || !fused_ok);
    if (want) {
      rc = A->rp64 ? build_sell<long long>(S, kSellSigma, kLongRow, &S->sell2)
                   : build_sell<int>(S, kSellSigma, kLongRow, &S->sell2);
      S->sell = rc == PCG_OK;
      if (!rc && !getenv("PIPECG_B200_NO_CHUNKS")) rc = build_long_chunks(S);
      if (rc) {
        pipecg_b200_solver_destroy(S);
        return rc;
      }
    }
  }
  // engine 3: an autotune candidate for irregular rows (req 0), or asked for
  if (req == kReqG || (req == 0 && has_long && !getenv("PIPECG_B200_NO_G"))) {
    int64_t cnt = 0;
    rc = pipecg_b200_find_long_rows(A->n_rows, A->rp64, A->rowptr, S->g_thr, nullptr, 0, &cnt, S->stream);
    if (!rc && cnt > 0) {
      if (pool_malloc(&S->g_long_rows, cnt * sizeof(int)) != cudaSuccess)
        rc = set_error(PCG_ENOMEM, "engine 3 long rows");
      else
        rc = pipecg_b200_find_long_rows(A->n_rows, A->rp64, A->rowptr, S->g_thr, S->g_long_rows, cnt,
                                        &cnt, S->stream);
    }
    S->n_glong = cnt;
    if (!rc)
      rc = A->rp64 ? build_sell<long long>(S, kGRows, S->g_thr, &S->gsell)
                   : build_sell<int>(S, kGRows, S->g_thr, &S->gsell);
    if (!rc) rc = build_g(S);
    if (rc) {
      pipecg_b200_solver_destroy(S);
      return rc;
    }
  }
  const int grid2 = std::min<int>(kDotGrid, 4 * S->num_sms);
  int grid3 = 0;  // engine 3: resident CTAs (256 threads each), at most one per window
  if (S->g_built) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, g_kernel(S), kGRows, 0);
    const long long n_win = (A->n_rows + kGRows - 1) / kGRows;  // 8 slices (warps) each
    grid3 = (int)std::max<long long>(1, std::min<long long>((long long)std::max(occ, 1) * S->num_sms,
                                                            n_win));
  }
  S->grid = std::max(grid2, grid3);
  // partials are sized for the largest grid any candidate (plan or autotune
  // alternative) can launch with
  for (int v = 0; v < kVariants; ++v) {
    S->grid = std::max(S->grid, S->plans[v].grid);
    for (const FusedPlan& p : S->alts[v]) S->grid = std::max(S->grid, p.grid);
  }
  phase("fused_setup+long+sell");
  rc = alloc_state(S);
  phase("alloc_state");
  if (rc) {
    pipecg_b200_solver_destroy(S);
    return rc;
  }
  if (req == kReqG) {
    S->engine = 3;
    S->grid = S->n_partials = grid3;
  } else if (!fused_ok) {
    S->engine = 2;
    S->grid = S->n_partials = grid2;
  } else if (req >= 3) {
    S->engine = 1;
    apply_plan(S, S->plans[req - 3]);
    // a forced E / F still picks the fastest of its own occupancy / stage
    // alternatives (process-cached like the full autotune)
    if (A->n_rows >= kTuneRows && S->alts[req - 3].size() > 1) {
      const TuneKey key{dev, A->n_rows, A->n_cols, A->nnz, A->rp64, (long long)max_row,
                        S->num_sms, S->opt.dot_mode, req, S->pat.n_pat,
                        (S->dinv_by_code ? 1 : 0) + (S->dinv_uniform ? 2 : 0)};
      int cached = -1, cached_alt = 0;
      if (!getenv("PIPECG_B200_NO_TUNE_CACHE")) {
        std::lock_guard<std::mutex> lk(tune_cache_mu());
        auto it = tune_cache().find(key);
        if (it != tune_cache().end()) std::tie(cached, cached_alt) = it->second;
      }
      if (cached == req - 3 && cached_alt < (int)S->alts[cached].size()) {
        apply_plan(S, S->alts[cached][cached_alt]);
      } else {
        rc = autotune(S, grid2, grid3, false, has_long, req - 3);
        if (rc) {
          pipecg_b200_solver_destroy(S);
          return rc;
        }
        std::lock_guard<std::mutex> lk(tune_cache_mu());
        tune_cache()[key] = std::make_pair(S->variant, S->alt_pick[S->variant]);
      }
    }
  } else if (A->n_rows < kTuneRows) {
    // small: no autotune.  Irregular rows -> D (balanced tiles); else P, then
    // C for wide rows (> 12 nnz/row, one gather per nonzero) or A
    const bool wide = A->nnz > 12 * A->n_rows;
    // small problems are launch-latency bound: P (one launch per chunk) first
    int order[kVariants] = {4, 0, 2, 3, 1, 5, 6};
    if (has_long) order[0] = 3, order[1] = 4, order[2] = 2, order[3] = 0;
    else if (wide) order[1] = 2, order[2] = 0;
    S->engine = 1;
    for (int k = 0; k < kVariants; ++k)
      if (S->plans[order[k]].stages) {
        apply_plan(S, S->plans[order[k]]);
        break;
      }
  } else {
    // process-level tuning cache (like a BLAS heuristics cache): a matrix
    // with the same shape and row-length profile on the same device reuses
    // the measured choice instead of re-timing every candidate
    const TuneKey key{dev, A->n_rows, A->n_cols, A->nnz, A->rp64, (long long)max_row,
                      S->num_sms, S->opt.dot_mode, req, S->pat.n_pat,
                      (S->dinv_by_code ? 1 : 0) + (S->dinv_uniform ? 2 : 0)};
    int cached = -1, cached_alt = 0;
    if (!getenv("PIPECG_B200_NO_TUNE_CACHE")) {
      std::lock_guard<std::mutex> lk(tune_cache_mu());
      auto it = tune_cache().find(key);
      if (it != tune_cache().end()) std::tie(cached, cached_alt) = it->second;
    }
    if (cached >= 0 && cached < kVariants && cached_alt < (int)S->alts[cached].size())
      S->plans[cached] = S->alts[cached][cached_alt];
    if (cached >= 0 && (cached == kVariants ||
                        (cached == kVariants + 1 && S->g_built) ||
                        (cached < kVariants && S->plans[cached].stages))) {
      if (cached < kVariants) {
        S->engine = 1;
        apply_plan(S, S->plans[cached]);
      } else if (cached == kVariants) {
        S->engine = 2;
        S->grid = S->n_partials = grid2;
      } else {
        S->engine = 3;
        S->grid = S->n_partials = grid3;
      }
    } else {
      rc = autotune(S, grid2, grid3, req == 0, has_long);
      if (rc) {
        pipecg_b200_solver_destroy(S);
        return rc;
      }
      std::lock_guard<std::mutex> lk(tune_cache_mu());
      tune_cache()[key] = S->engine == 2   ? std::make_pair(kVariants, 0)
                          : S->engine == 3 ? std::make_pair(kVariants + 1, 0)
                                           : std::make_pair(S->variant, S->alt_pick[S->variant]);
    }
  }
  phase("engine choice");
  if (getenv("PIPECG_B200_DEBUG_PLAN")) {  // experiment aid: the plan in use + the E/F alternatives
    for (auto& ph : phases) fprintf(stderr, "[pipecg_b200] t=%.2f ms after %s\n", ph.second, ph.first);
    fprintf(stderr, "[pipecg_b200] engine %d variant %d tr %d stages %d grid %d smem %zu n_pat %d "
            "runs %d dinv_by_code %d uniform %d\n", S->engine, S->variant, S->tr, S->stages, S->grid,
            S->smem, S->pat.n_pat, S->n_runs, (int)S->dinv_by_code, (int)S->dinv_uniform);
    if (S->g_built)
      fprintf(stderr, "[pipecg_b200] engine 3: lane rows <= %lld, %lld warp-chunk rows (%lld chunks, %d "
              "multi-chunk), SELL %lld slices %lld elements, grid %d\n", S->g_thr, S->n_glong,
              S->n_gchunks, S->n_gmulti, S->gsell.slices, S->gsell.total, S->engine == 3 ? S->grid : 0);
    for (int v = 5; v <= 6; ++v)
      for (const FusedPlan& p : S->alts[v])
        fprintf(stderr, "[pipecg_b200]   alt %c: tr %d bps %d stages %d grid %d smem %zu\n",
                v == 5 ? 'E' : 'F', p.tr, p.bps, p.stages, p.grid, p.smem);
  }
  *out = S;
  return PCG_OK;
}

// cudaFree synchronises the whole device.  While a connected solver of
// this process may be running, its kernels can be spinning on a peer
// rank's arrival -- and that peer's host thread may be the one that would
// block in cudaFree (a virtual rank sharing the GPU, or a thread of
// pipecg_solve_devices collecting garbage), which stalls the exchange until
// the spin timeout.  So the IPC-exported buffers (plain cudaMalloc, no
// stream-ordered free) of a destroyed solver are parked here while any
// connected solver is alive and freed when the last one goes.
struct DeferredFrees {
  std::mutex mu;
  std::vector<std::pair<int, void*>> ptrs;  // (device, pointer)
  int connected = 0;
};
DeferredFrees& deferred_frees() {
  static DeferredFrees d;
  return d;
}
void free_exported(pcg_solver* S) {
  DeferredFrees& D = deferred_frees();
  std::lock_guard<std::mutex> lk(D.mu);
  if (S->connected) --D.connected;
  int dev = 0;
  cudaGetDevice(&dev);
  if (D.connected > 0 && !getenv("PIPECG_B200_EAGER_FREE")) {  // (env: regression check)
    for (void* p : {static_cast<void*>(S->vbuf), static_cast<void*>(S->comm)}) {
      if (!p) continue;
      cudaPointerAttributes a{};
      const bool known = cudaPointerGetAttributes(&a, p) == cudaSuccess;
      D.ptrs.emplace_back(known ? a.device : dev, p);  // freed on its own device later
    }
    cudaGetLastError();
    return;
  }
  cudaFree(S->vbuf);
  cudaFree(S->comm);
  for (auto& dp : D.ptrs) {
    cudaSetDevice(dp.first);
    cudaFree(dp.second);
  }
  D.ptrs.clear();
  cudaSetDevice(dev);
}

int pipecg_b200_solver_destroy(pcg_solver* S) {
  if (!S) return PCG_OK;
  if (S->stream) cudaStreamSynchronize(S->stream);
  AllocStream alloc_on(S->stream);  // (null stream: plain cudaFree)
  for (int k = 0; k < 2; ++k) {
    for (auto& kv : S->graphs[k]) cudaGraphExecDestroy(kv.second);
    if (S->rec_host[k]) pinned_record_release(S->rec_host[k]);
    if (S->ev_rec[k]) cudaEventDestroy(S->ev_rec[k]);
  }
  free_exported(S);  // vbuf, comm
  pool_free(S->partials);
  pool_free(S->fin);
  pool_free(S->gbar);
  pool_free(S->counter);
  pool_free(S->seqbuf);
  pool_free(S->dpart);
  pool_free(S->dots_ws);
  pool_free(S->dots4);
  pool_free(S->rec_dev);
  pool_free(S->long_rows);
  pool_free(S->chunks);
  pool_free(S->chunk_part);
  pool_free(S->chunk_ticket);
  pool_free(S->hubdot);
  pool_free(S->gchunks);
  pool_free(S->iperm);
  pool_free(S->sell_colp);
  pool_free(S->hcol);
  pool_free(S->hval);
  pool_free(S->dinvp);
  pool_free(S->natbuf);
  pool_free(S->qbuf);
  pool_free(S->qcnt);
  pool_free(S->qhub);
  pool_free(S->gchunk_part);
  pool_free(S->gchunk_ticket);
  for (Sell* c : {&S->sell2, &S->gsell}) {
    pool_free(c->ptr);
    pool_free(c->perm);
    pool_free(c->len);
    pool_free(c->col);
    pool_free(c->val);
  }
  pool_free(S->g_long_rows);
  pool_free(S->x_ptr);
  pool_free(S->x_row);
  pool_free(S->x_peer);
  pool_free(S->x_dst);
  for (int v = 0; v < kVariants; ++v) {
    pool_free(S->plans[v].tile_row);
    pool_free(S->plans[v].tile_e);
  }
  free_row_patterns(&S->pat);
  pool_free(S->pwin);
  for (int k = 0; k < 3; ++k) pool_free(S->tile_runs[k]);
  pool_free(S->pdinv);

  if (S->ev_in) cudaEventDestroy(S->ev_in);
  if (S->stream) cudaStreamDestroy(S->stream);
  delete S;
  return PCG_OK;
}

int pipecg_b200_solver_comm_info(pcg_solver* S, void** vbuf, int64_t* ld, void** comm) {
  if (!S) return set_error(PCG_EINVAL, "solver_comm_info: null solver");
  if (vbuf) *vbuf = S->vbuf;
  if (ld) *ld = (int64_t)S->ld;
  if (comm) *comm = S->comm;
  return PCG_OK;
}

int pipecg_b200_ipc_get_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return set_error(PCG_EINVAL, "ipc_get_handle: null");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
  if (e != cudaSuccess) return cuda_status(e, "cudaIpcGetMemHandle");
  memcpy(handle_out, &h, sizeof(h));
  return PCG_OK;
}

int pipecg_b200_ipc_open(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return set_error(PCG_EINVAL, "ipc_open: null");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess),
                     "cudaIpcOpenMemHandle");
}

int pipecg_b200_ipc_close(void* dev_ptr) {
  return cuda_status(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
}

int pipecg_b200_enable_peer_access(int device, int peer) {
  int prev = 0, can = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaDeviceCanAccessPeer(&can, device, peer);
  if (e != cudaSuccess) return cuda_status(e, "cudaDeviceCanAccessPeer");
  if (!can) return set_error(PCG_EINVAL, "enable_peer_access: the devices cannot access each other");
  e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky-free status
    e = cudaSuccess;
  }
  cudaSetDevice(prev);
  return cuda_status(e, "cudaDeviceEnablePeerAccess");
}

// Per-tile send lists for the fused exchange: the plan's send entries sorted
// by local row, and for every tile of the applied plan the range of entries
// whose row it owns.
int build_tile_sends(pcg_solver* S) {
  const long long ns = S->cp.n_send, nt = S->n_tiles, n = S->A.n_rows;
  std::vector<int> row(ns), peer(ns);
  std::vector<long long> dst(ns);
  cudaStream_t st = S->stream;
  if (ns) {
    cudaMemcpyAsync(row.data(), S->cp.send_row, ns * sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(peer.data(), S->cp.send_peer, ns * sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(dst.data(), S->cp.send_dst, ns * sizeof(long long), cudaMemcpyDeviceToHost, st);
  }
  std::vector<int> tstart(nt + 1);
  if (S->variant == 3) {
    cudaMemcpyAsync(tstart.data(), S->tile_row, (nt + 1) * sizeof(int), cudaMemcpyDeviceToHost, st);
  } else {
    for (long long t = 0; t <= nt; ++t) tstart[t] = (int)std::min<long long>(t * S->tr, n);
  }
  int rc = cuda_status(cudaStreamSynchronize(st), "fused exchange plan");
  if (rc) return rc;
  std::vector<long long> ord(ns);
  for (long long e = 0; e < ns; ++e) ord[e] = e;
  std::stable_sort(ord.begin(), ord.end(), [&](long long a, long long b) { return row[a] < row[b]; });
  std::vector<int> srow(ns), speer(ns), ptr(nt + 1);
  std::vector<long long> sdst(ns);
  for (long long e = 0; e < ns; ++e) {
    srow[e] = row[ord[e]];
    speer[e] = peer[ord[e]];
    sdst[e] = dst[ord[e]];
  }
  for (long long t = 0; t <= nt; ++t)
    ptr[t] = (int)(std::lower_bound(srow.begin(), srow.end(), tstart[t]) - srow.begin());
  pool_free(S->x_ptr);
  pool_free(S->x_row);
  pool_free(S->x_peer);
  pool_free(S->x_dst);
  S->x_ptr = S->x_row = S->x_peer = nullptr;
  S->x_dst = nullptr;
  if (pool_malloc(&S->x_ptr, (nt + 1) * sizeof(int)) != cudaSuccess ||
      pool_malloc(&S->x_row, std::max<long long>(ns, 1) * sizeof(int)) != cudaSuccess ||
      pool_malloc(&S->x_peer, std::max<long long>(ns, 1) * sizeof(int)) != cudaSuccess ||
      pool_malloc(&S->x_dst, std::max<long long>(ns, 1) * sizeof(long long)) != cudaSuccess)
    return set_error(PCG_ENOMEM, "fused exchange lists");
  cudaMemcpyAsync(S->x_ptr, ptr.data(), (nt + 1) * sizeof(int), cudaMemcpyHostToDevice, st);
  if (ns) {
    cudaMemcpyAsync(S->x_row, srow.data(), ns * sizeof(int), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(S->x_peer, speer.data(), ns * sizeof(int), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(S->x_dst, sdst.data(), ns * sizeof(long long), cudaMemcpyHostToDevice, st);
  }
  return cuda_status(cudaStreamSynchronize(st), "fused exchange lists");
}

// every inv_diag entry of [0, n_cols) (owned + halo) equal to dinv0?
// Stream-ordered allocation only: solver_init calls this while a peer rank
// sharing the GPU may already be spinning in its iteration kernel, and a
// plain cudaFree would wait for that kernel (device-wide sync -> the peer
// times out waiting for this rank).
int uniform_dinv(pcg_solver* S, int* bad) {
  int* d = nullptr;
  if (cudaMallocAsync(&d, sizeof(int), S->stream) != cudaSuccess)
    return set_error(PCG_ENOMEM, "dinv check");
  cudaMemsetAsync(d, 0, sizeof(int), S->stream);
  uniform_check_kernel<<<elementwise_grid(S->A.n_cols), 256, 0, S->stream>>>(
      S->A.n_cols, S->A.inv_diag, S->dinv0, d);
  cudaMemcpyAsync(bad, d, sizeof(int), cudaMemcpyDeviceToHost, S->stream);
  cudaFreeAsync(d, S->stream);
  return cuda_status(cudaStreamSynchronize(S->stream), "dinv check");
}

int pipecg_b200_solver_connect(pcg_solver* S, int rank, int world, void* const* peer_vbuf,
                               const int64_t* peer_ld, void* const* peer_comm, int64_t n_send,
                               const int32_t* send_row, const int32_t* send_peer,
                               const int64_t* send_dst) {
  if (!S || world < 1 || world > kMaxRanks || rank < 0 || rank >= world || !peer_vbuf ||
      !peer_ld || !peer_comm || (n_send > 0 && (!send_row || !send_peer || !send_dst)))
    return set_error(PCG_EINVAL, "solver_connect: bad arguments");
  if (S->engine != 1)
    return set_error(PCG_EINVAL, "solver_connect: distributed mode needs the fused engine");
  S->rank = rank;
  S->world = world;
  CommParams cp{};
  cp.rank = rank;
  cp.world = world;
  for (int q = 0; q < world; ++q) {
    cp.peer_vbuf[q] = static_cast<char*>(peer_vbuf[q]);
    cp.peer_ld[q] = peer_ld[q];
    cp.peer_comm[q] = static_cast<char*>(peer_comm[q]);
  }
  cp.n_send = n_send;
  cp.send_row = send_row;
  cp.send_peer = send_peer;
  cp.send_dst = reinterpret_cast<const long long*>(send_dst);
  S->cp = cp;
  if (!S->connected) {
    std::lock_guard<std::mutex> lk(deferred_frees().mu);
    ++deferred_frees().connected;
  }
  S->connected = true;
  AllocStream alloc_on(S->stream);
  // The shard's row-pattern dictionary is valid in its [owned | halo]
  // column space (the halo mapping is affine per contiguous halo range), so
  // E/F keep running with windows and the fused exchange.  E needs one dinv
  // for every column, halo included (it never sees the halo rows' codes).
  // Otherwise -> the CSR variant of the same exchange class (E -> A, F -> C,
  // both push the same vector) in per-iteration launches (P -> C).
  bool keep = S->engine == 1 && (S->variant == 5 || S->variant == 6) && S->n_runs > 0 &&
              !getenv("PIPECG_B200_SEPARATE_XCHG");
  if (keep && S->variant == 5) {
    int bad = 1;
    int rc = uniform_dinv(S, &bad);
    if (rc) return rc;
    keep = S->dinv_by_code && S->dinv_uniform && !bad;
  }
  // E's consumer-loaded layout (dv) is the single-GPU autotuner's pick at
  // 7-pt, but with the fused exchange the staged layout is faster (3D 7-pt
  // 256^3, one connected rank: 0.358 vs 0.535 ms per iteration,
  // tools/dist1.py): take E's first staged alternative
  if (keep && S->variant == 5 && S->dv && !getenv("PIPECG_B200_DIST_KEEP_DV"))
    for (const FusedPlan& q : S->alts[5])
      if (!q.dv) {
        apply_plan(S, q);
        break;
      }
  if (S->engine == 1 && S->variant >= 4 && !keep) {
    const FusedPlan& csr = S->plans[S->variant == 5 ? 0 : 2];
    if (!csr.stages) return set_error(PCG_EINVAL, "solver_connect: no CSR variant fits this shard");
    apply_plan(S, csr);
  }
  // fused exchange for variants A, C, D (B keeps the separate exchange kernel)
  S->fused_xchg = S->variant != 1 && !getenv("PIPECG_B200_SEPARATE_XCHG");
  if (S->fused_xchg) {
    int rc = build_tile_sends(S);
    if (rc) return rc;
  }
  for (int k = 0; k < 2; ++k) {  // graphs captured without the exchange are stale
    for (auto& kv : S->graphs[k]) cudaGraphExecDestroy(kv.second);
    S->graphs[k].clear();
  }
  return PCG_OK;
}

int pipecg_b200_solver_init(pcg_solver* S, const double* b, const double* x0, double tolerance,
                            int64_t max_iterations, int64_t drift_check_interval, void* stream) {
  if (!S || !b || !x0) return set_error(PCG_EINVAL, "solver_init: bad arguments");
  if (max_iterations < 1) return set_error(PCG_EINVAL, "solver_init: max_iterations < 1");
  cudaStream_t st = S->stream;
  cudaEventRecord(S->ev_in, (cudaStream_t)stream);
  cudaStreamWaitEvent(st, S->ev_in, 0);
  const long long n = S->A.n_rows;
  const size_t bytes = (size_t)n * sizeof(double);
  S->tol = tolerance;
  S->max_it = max_iterations;
  if ((drift_check_interval > 0) != (S->drift_k > 0)) {
    // the chunk graphs bake in the drift kernels and the deferred-x mode
    for (int k = 0; k < 2; ++k) {
      for (auto& kv : S->graphs[k]) cudaGraphExecDestroy(kv.second);
      S->graphs[k].clear();
    }
  }
  S->drift_k = drift_check_interval;
  Record R = record_at(S->rec_dev);
  cudaMemsetAsync(&R.C->comm_error, 0, sizeof(int), st);
  cudaMemsetAsync(S->counter, 0, 2 * sizeof(unsigned), st);
  // solvers.py:305-321
  cudaMemcpyAsync(S->b, b, bytes, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(S->x, x0, bytes, cudaMemcpyDeviceToDevice, st);
  if (S->pat.n_pat > 0) {  // is dinv still a function of the row's code? (E/F read it so)
    bool dbc = false, uni = false;
    double d0 = 0.0;
    int rc = check_dinv_by_code(S->pat, n, S->A.inv_diag, S->pdinv, &dbc, &uni, &d0, st);
    if (rc) return rc;
    if (S->connected && S->engine == 1 && S->variant == 5) {
      // E reads one dinv for every column, the halo columns included: the
      // owned rows (check_dinv_by_code) and all n_cols entries must still
      // hold the number solver_connect checked
      int bad = 0;
      if (dbc && uni && std::memcmp(&d0, &S->dinv0, sizeof(double)) == 0) {
        rc = uniform_dinv(S, &bad);
        if (rc) return rc;
      }
      if (!dbc || !uni || bad || std::memcmp(&d0, &S->dinv0, sizeof(double)) != 0)
        return set_error(PCG_ESTATE, "solver_init: inv_diag changed after solver_connect "
                                     "(variant E reads one dinv for every column)");
    }
    if (dbc != S->dinv_by_code || uni != S->dinv_uniform ||
        std::memcmp(&d0, &S->dinv0, sizeof(double)) != 0) {
      S->dinv_by_code = dbc;
      S->dinv_uniform = uni;
      S->dinv0 = d0;
      // an E plan without the streamed vectors in its stages only fits the
      // window layout: without windows (dinv no longer by code) take E's
      // plan that stages them
      if (S->engine == 1 && S->variant == 5 && S->dv && !s_windows(S, false))
        for (const FusedPlan& q : S->alts[5])
          if (!q.dv) {
            apply_plan(S, q);
            break;
          }
      for (int k = 0; k < 2; ++k) {  // graphs bake the kernel choice in
        for (auto& kv : S->graphs[k]) cudaGraphExecDestroy(kv.second);
        S->graphs[k].clear();
      }
    }
  }
  if (S->connected) {  // x halo (r = b - A x reads it)
    snapshot_arrive_kernel<<<1, 32, 0, st>>>(R.C, S->comm);
    vec_exchange_kernel<<<kXchgBlocks, 256, 0, st>>>(S->cp, 4, S->x);
    S->xtarget += (unsigned long long)S->world * kXchgBlocks;
    xwait_kernel<<<1, 32, 0, st>>>(S->comm, S->xtarget, R.C);
  }
  int rc = spmv_any(n, S->A.rp64, S->A.rowptr, S->A.col, S->A.val, S->x, S->b, S->r,
                    S->long_rows, S->n_long, 1, st);  // r = b - A x
  if (rc) return rc;
  rc = pipecg_b200_jacobi_apply(n, S->A.inv_diag, S->r, S->u, st);  // u = M^-1 r
  if (rc) return rc;
  if (S->engine == 4) {  // classic PCG (solvers.py:223-231): p = 0, gamma, norm, b_norm
    cudaMemsetAsync(S->p, 0, bytes, st);
    cudaMemsetAsync(S->qcnt, 0, 8 * sizeof(unsigned), st);
    const double* qa[4] = {S->r, S->u, S->u, S->b};
    const double* qb[4] = {S->u, S->u, S->u, S->b};
    rc = dots_any(n, 4, qa, qb, S->opt.dot_mode, S->dots4, S->dots_ws, st);
    if (rc) return rc;
    init_ctrl_kernel<<<1, 256, 0, st>>>(R.C, S->dots4, 1, tolerance, max_iterations,
                                        drift_check_interval, R.hist, R.dit, nullptr);
    S->host_base = 0;
    S->initialized = true;
    return cuda_status(cudaGetLastError(), "solver_init");
  }
  if (S->connected) {  // u halo (w = A u reads it)
    vec_exchange_kernel<<<kXchgBlocks, 256, 0, st>>>(S->cp, 6, S->u);
    S->xtarget += (unsigned long long)S->world * kXchgBlocks;
    xwait_kernel<<<1, 32, 0, st>>>(S->comm, S->xtarget, R.C);
  }
  rc = spmv_any(n, S->A.rp64, S->A.rowptr, S->A.col, S->A.val, S->u, nullptr, S->w[0],
                S->long_rows, S->n_long, 0, st);  // w = A u
  if (rc) return rc;
  const bool stored_m = S->engine == 2 || stored_m_fused(S);
  if (stored_m_fused(S)) {
    rc = pipecg_b200_jacobi_apply(n, S->A.inv_diag, S->w[0], S->m, st);  // m = M^-1 w
    if (rc) return rc;
  }
  if (S->connected) {  // halo of what F(0) gathers: w (A/B) or the stored m (C)
    vec_exchange_kernel<<<kXchgBlocks, 256, 0, st>>>(S->cp, stored_m ? 9 : 7,
                                                     stored_m ? S->m : S->w[0]);
    S->xtarget += (unsigned long long)S->world * kXchgBlocks;
    xwait_kernel<<<1, 32, 0, st>>>(S->comm, S->xtarget, R.C);
  }
  if (S->engine == 3) {  // the kernel gathers the stored m (n = A m is formed in the kernel)
    rc = pipecg_b200_jacobi_apply(n, S->A.inv_diag, S->w[0], S->m, st);  // m = M^-1 w
    if (rc) return rc;
  }
  if (S->engine == 2) {
    rc = pipecg_b200_jacobi_apply(n, S->A.inv_diag, S->w[0], S->m, st);  // m = M^-1 w
    if (rc) return rc;
    rc = spmv_any(n, S->A.rp64, S->A.rowptr, S->A.col, S->A.val, S->m, nullptr, S->nv,
                  S->long_rows, S->n_long, 0, st);  // n = A m
    if (rc) return rc;
  }
  S->mn_valid = S->engine == 2 && !S->connected;
  cudaMemsetAsync(S->z, 0, bytes, st);
  cudaMemsetAsync(S->q, 0, bytes, st);
  cudaMemsetAsync(S->s, 0, bytes, st);
  cudaMemsetAsync(S->p, 0, bytes, st);
  const double* da[4] = {S->r, S->w[0], S->u, S->b};
  const double* db[4] = {S->u, S->u, S->u, S->b};
  rc = dots_any(n, 4, da, db, S->opt.dot_mode, S->dots4, S->dots_ws, st);
  if (rc) return rc;
  if (S->engine == 3) {  // the state moves into SELL order (b stays natural)
    const unsigned g = elementwise_grid(n);
    gather_perm_kernel<<<g, 256, 0, st>>>(n, S->gsell.perm, S->A.inv_diag, S->dinvp);
    double* vs[5] = {S->x, S->r, S->u, S->w[0], S->m};
    for (double* v : vs) {
      cudaMemcpyAsync(S->nv, v, bytes, cudaMemcpyDeviceToDevice, st);
      gather_perm_kernel<<<g, 256, 0, st>>>(n, S->gsell.perm, S->nv, v);
    }
  }
  if (S->connected) {
    init_dots_exchange_kernel<<<1, 32, 0, st>>>(S->cp, S->dots4);
    S->xtarget += (unsigned long long)S->world;
    xwait_kernel<<<1, 32, 0, st>>>(S->comm, S->xtarget, R.C);
    init_ctrl_kernel<<<1, 256, 0, st>>>(
        R.C, reinterpret_cast<const double*>(S->comm + kCommISlots), S->world, tolerance,
        max_iterations, drift_check_interval, R.hist, R.dit,
        reinterpret_cast<const unsigned long long*>(S->comm));
  } else {
    init_ctrl_kernel<<<1, 256, 0, st>>>(R.C, S->dots4, 1, tolerance, max_iterations,
                                        drift_check_interval, R.hist, R.dit, nullptr);
  }
  S->host_base = 0;
  S->initialized = true;
  return cuda_status(cudaGetLastError(), "solver_init");
}

int pipecg_b200_solver_run(pcg_solver* S, pcg_result* res, double* history_host, int64_t hist_cap,
                           int64_t* drift_it_host, double* drift_val_host, int64_t drift_cap) {
  if (!S || !res) return set_error(PCG_EINVAL, "solver_run: bad arguments");
  if (!S->initialized) return set_error(PCG_ESTATE, "solver_run before solver_init");
  memset(res, 0, sizeof(*res));
  const int K = auto_chunk(S);
  long long hist_n = 0, drift_n = 0;
  long long next_hist = 1;  // next history index to collect (0 = init norm)
  long long chunk_lo[2] = {0, 0};
  int cur = S->rec_parity;
  chunk_lo[cur] = S->host_base;
  int rc = launch_chunk(S, K, cur);
  if (rc) return rc;
  Ctrl c{};
  bool first = true;
  while (true) {
    const int nxt = cur ^ 1;
    const bool more = S->host_base <= S->max_it;  // F(max_it) must run to stop
    if (more) {
      chunk_lo[nxt] = S->host_base;
      rc = launch_chunk(S, K, nxt);
      if (rc) return rc;
    }
    cudaError_t e = cudaEventSynchronize(S->ev_rec[cur]);
    if (e != cudaSuccess) return cuda_status(e, "chunk wait");
    const Record R = record_at(S->rec_host[cur]);
    c = *R.C;
    if (first) {
      if (history_host && hist_cap > 0) history_host[0] = c.init.norm;
      hist_n = 1;
      first = false;
    }
    long long hi = chunk_lo[cur] + K - 1;  // last iteration whose entry this chunk ran
    if (c.status == PCG_STOPPED) hi = std::min(hi, c.final_it);
    if (c.status == PCG_BREAKDOWN) hi = std::min(hi, c.bd_it);
    if (c.status == PCG_ECOMM_STATUS) hi = -1;
    for (long long itx = next_hist; itx <= hi; ++itx) {
      if (history_host && hist_n < hist_cap) history_host[hist_n] = R.hist[itx & (kHistRing - 1)];
      hist_n++;
    }
    if (S->drift_k > 0) {
      for (long long itx = std::max(chunk_lo[cur], 1LL); itx <= hi; ++itx) {
        if (itx % S->drift_k) continue;
        const int slot = (int)(itx & (kHistRing - 1));
        if (R.dit[slot] != itx) continue;
        if (drift_n < drift_cap) {
          if (drift_it_host) drift_it_host[drift_n] = itx;
          if (drift_val_host) drift_val_host[drift_n] = R.dval[slot];
        }
        drift_n++;
      }
    }
    next_hist = std::max(next_hist, hi + 1);
    if (c.status != PCG_RUNNING || !more) break;
    cur = nxt;
  }
  if (defer_x_active(S)) {  // after every queued iteration kernel (stream order)
    Ctrl* Cd = record_at(S->rec_dev).C;
    finalize_x_kernel<<<elementwise_grid(S->A.n_rows), 256, 0, S->stream>>>(Cd, S->A.n_rows,
                                                                            S->x, S->p);
    finalize_mark_kernel<<<1, 32, 0, S->stream>>>(Cd);
  }
  {
    cudaError_t e = cudaStreamSynchronize(S->stream);
    if (e != cudaSuccess) return cuda_status(e, "solve sync");
  }
  S->rec_parity = cur ^ 1;
  fill_result(S, c, res);
  res->n_history = hist_n;
  res->n_drift = drift_n;
  S->mn_valid = false;
  return comm_failed(c);
}

int pipecg_b200_solver_prepare(pcg_solver* S, int64_t count) {
  if (!S) return set_error(PCG_EINVAL, "solver_prepare: null handle");
  if (!S->opt.use_graphs || count <= 0) return PCG_OK;
  const int K = auto_chunk(S);
  const int sizes[2] = {(int)std::min<int64_t>(count, K), (int)(count % K)};
  for (int k : sizes)
    for (int parity = 0; parity < 2 && k > 0; ++parity) {
      cudaGraphExec_t exec = nullptr;
      if (chunk_graph(S, k, parity, &exec) != PCG_OK)
        cudaGetLastError();  // launched directly instead (see chunk_graph)
    }
  return PCG_OK;
}

int pipecg_b200_solver_enqueue(pcg_solver* S, int64_t count) {
  if (!S || !S->initialized) return set_error(PCG_ESTATE, "solver_enqueue before init");
  const int K = auto_chunk(S);
  while (count > 0) {
    const int k = (int)std::min<int64_t>(count, K);
    int rc = launch_chunk(S, k, S->rec_parity);
    if (rc) return rc;
    S->rec_parity ^= 1;
    count -= k;
  }
  S->mn_valid = false;
  return PCG_OK;
}

double* pipecg_b200_solver_x(pcg_solver* S) {
  if (!S) return nullptr;
  if (S->engine == 3 && S->initialized) {  // SELL order -> natural order (into the unused n)
    scatter_perm_kernel<<<elementwise_grid(S->A.n_rows), 256, 0, S->stream>>>(S->A.n_rows, S->gsell.perm,
                                                                              S->x, S->nv);
    cudaStreamSynchronize(S->stream);
    return S->nv;
  }
  return S->x;
}

void* pipecg_b200_solver_stream(pcg_solver* S) { return S ? (void*)S->stream : nullptr; }

int pipecg_b200_solver_poll(pcg_solver* S, pcg_result* res) {
  if (!S || !res) return set_error(PCG_EINVAL, "solver_poll: bad arguments");
  cudaError_t e = cudaStreamSynchronize(S->stream);
  if (e != cudaSuccess) return cuda_status(e, "poll sync");
  Ctrl c{};
  e = cudaMemcpy(&c, S->rec_dev, sizeof(Ctrl), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e, "poll copy");
  memset(res, 0, sizeof(*res));
  fill_result(S, c, res);
  return comm_failed(c);
}

void pipecg_b200_tune_cache_clear(void) {
  std::lock_guard<std::mutex> lock(tune_cache_mu());
  tune_cache().clear();
}

int pipecg_b200_solver_state(pcg_solver* S, double** ptrs) {
  if (!S || !ptrs) return set_error(PCG_EINVAL, "solver_state: bad arguments");
  if (S->connected) return set_error(PCG_EINVAL, "solver_state: single-GPU only");
  Ctrl c{};
  cudaError_t e = cudaStreamSynchronize(S->stream);
  if (e == cudaSuccess) e = cudaMemcpy(&c, S->rec_dev, sizeof(Ctrl), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e, "solver_state");
  const long long done = c.status == PCG_STOPPED ? c.final_it : c.base_it;
  double* w = S->engine == 1 ? S->w[done & 1] : S->w[0];
  const long long n = S->A.n_rows;
  if (S->engine == 3) {  // natural-order copies of the SELL-order state
    if (!S->natbuf && pool_malloc(&S->natbuf, S->ld * 10 * sizeof(double)) != cudaSuccess)
      return set_error(PCG_ENOMEM, "solver_state: natural-order copies");
    double* src[10] = {S->x, S->r, S->u, S->w[0], nullptr, nullptr, S->z, S->q, S->s, S->p};
    const unsigned g = elementwise_grid(n);
    for (int k = 0; k < 10; ++k) {
      ptrs[k] = S->natbuf + (size_t)k * S->ld;
      if (src[k])
        scatter_perm_kernel<<<g, 256, 0, S->stream>>>(n, S->gsell.perm, src[k], (double*)ptrs[k]);
    }
    int rc = pipecg_b200_jacobi_apply(n, S->A.inv_diag, (double*)ptrs[3], (double*)ptrs[4], S->stream);
    if (!rc)
      rc = spmv_any(n, S->A.rp64, S->A.rowptr, S->A.col, S->A.val, (double*)ptrs[4], nullptr,
                    (double*)ptrs[5], S->long_rows, S->n_long, 0, S->stream);
    if (rc) return rc;
    return cuda_status(cudaStreamSynchronize(S->stream), "solver_state");
  }
  if (!S->mn_valid) {
    int rc = pipecg_b200_jacobi_apply(n, S->A.inv_diag, w, S->m, S->stream);
    if (!rc)
      rc = spmv_any(n, S->A.rp64, S->A.rowptr, S->A.col, S->A.val, S->m, nullptr, S->nv,
                    S->long_rows, S->n_long, 0, S->stream);
    if (rc) return rc;
    e = cudaStreamSynchronize(S->stream);
    if (e != cudaSuccess) return cuda_status(e, "solver_state m/n");
    S->mn_valid = true;
  }
  double* v[10] = {S->x, S->r, S->u, w, S->m, S->nv, S->z, S->q, S->s, S->p};
  for (int k = 0; k < 10; ++k) ptrs[k] = v[k];
  return PCG_OK;
}

}  // extern "C"
