// ravnest_b200 -- sm_100a kernels and C ABI for the Parallel Multi-Ring
// All-Reduce of Ravnest (arXiv 2401.01728).  See include/ravnest_b200.h for
// the contract and DESIGN.md for the data layout and roofline.
//
// Reference arithmetic (/root/reference/pkg/src/ravnest/multiring.py):
//   * chunk split       :134-144  chunk i of a ring gets base + (i < rem)
//   * reduce-scatter    :216-219  seg += payload, last RS round seg /= C
//   * all-gather        :220-221  seg = payload
// Closed form (SURVEY.md headline fact 3): chunk k of every member ends as
//   fl(fl(...fl(x_k + x_{k+1}) ... + x_{k+C-1}) / C), indices mod C.
//
// One kernel does the whole cycle for the chunks hosted on this device: it
// reads chunk k from the C member buffers (local HBM or NVLink peer memory),
// folds in ring order, divides by C and stores the mean into all C member
// buffers.  Chunk k is read and written only by its owner, so in-place
// averaging needs no mid-cycle barrier; cross-device ordering uses
// release/acquire flags at system scope (arrive before the first read,
// depart after the last write).

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ravnest_b200.h"

namespace {

// ---------------------------------------------------------------------------
// error plumbing

thread_local std::string g_err;

int set_err(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define RV_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return set_err(RV_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));   \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ---------------------------------------------------------------------------
// device-side types

constexpr int kThreads = 256;
constexpr unsigned kStatusTimeout = 1u;
constexpr int64_t kUnitBytes = 256 * 1024;    // push protocol: largest flagged unit
constexpr int64_t kMinUnitBytes = 16 * 1024;  // push protocol: smallest flagged unit

struct Seg {
  int64_t lo, hi;            // chunk [lo, hi) in elements
  int64_t body_lo, body_hi;  // 16-byte aligned vector body inside it
  int64_t stage_off;         // push: element offset of this chunk in the owner's staging slot
  int64_t unit0;             // push: first unit index of this chunk (per owner, per lane)
  int32_t k;                 // fold start position = owner position (chunk index in its ring)
  int32_t ring;
};

struct LaneState {
  unsigned long long epoch;     // cycles completed on this lane
  unsigned long long signaled;  // last epoch whose arrive flags were posted
  unsigned int done;            // blocks finished in the running cycle
  unsigned int pad;
};

struct CycleParams {
  const void *src[RV_MAX_CLUSTERS];
  void *dst[RV_MAX_CLUSTERS];
  void *stage[RV_MAX_CLUSTERS];                 // push: owner q's staging area (as mapped here)
  unsigned long long *pflags[RV_MAX_CLUSTERS];  // push: owner q's unit flags (as mapped here)
  unsigned long long *peer_flags[RV_MAX_RANKS]; // rank r's barrier flag area (as mapped here)
  const Seg *segs;             // pull: this device's chunks; push: every owner's, owner-major
  const int64_t *tile_prefix;  // pull: nseg + 1 entries
  unsigned long long *my_flags;
  LaneState *state;
  unsigned int *status;        // [0] code, [1] diag
  unsigned long long *trace;   // optional: [start, ready, work done, departed] (globaltimer ns)
  int64_t n_tiles;             // pull
  int64_t stride;              // push: staging elements per writer slot
  int64_t units_max;           // push: unit-flag slots per (lane, writer)
  int64_t scatter_umax;        // push: max units over the other owners
  int64_t unit_vecs;           // push: vectors per unit
  int64_t ounits[RV_MAX_CLUSTERS];
  int oseg_base[RV_MAX_CLUSTERS + 1];
  unsigned long long timeout_ns;
  double inv_c;
  int C, nseg, rank, n_ranks, lane, pow2, me;
};

// flag slot of (lane, sender rank, phase) inside a receiver's barrier area
__host__ __device__ inline size_t flag_index(int lane, int sender, int phase) {
  return ((size_t)lane * RV_MAX_RANKS + (size_t)sender) * 2 + (size_t)phase;
}

// push: flag slot of (lane, writer, unit) inside an owner's unit-flag area
__host__ __device__ inline size_t pflag_index(int lane, int c, int writer, int64_t units_max, int64_t u) {
  return ((size_t)lane * c + (size_t)writer) * (size_t)units_max + (size_t)u;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Spin until *f >= e.  Returns false on timeout (status set, diag recorded)
// or when another block already failed.
__device__ bool wait_flag(const CycleParams &p, const unsigned long long *f, unsigned long long e,
                          unsigned long long t0, unsigned diag) {
  unsigned spins = 0;
  while (ld_acquire_sys(f) < e) {
    if ((++spins & 255u) == 0) {
      if (*(volatile unsigned *)p.status != 0) return false;
      if (globaltimer() - t0 > p.timeout_ns) {
        if (atomicCAS(p.status, 0u, kStatusTimeout) == 0u) p.status[1] = diag;
        return false;
      }
    }
  }
  return true;
}

// Wait until every peer posted `phase` for epoch e.
__device__ bool wait_peers(const CycleParams &p, int phase, unsigned long long e) {
  const unsigned long long t0 = globaltimer();
  for (int r = 0; r < p.n_ranks; ++r) {
    if (r == p.rank) continue;
    const unsigned diag = ((unsigned)phase << 16) | ((unsigned)p.lane << 8) | (unsigned)r;
    if (!wait_flag(p, p.my_flags + flag_index(p.lane, r, phase), e, t0, diag)) return false;
  }
  return true;
}

__device__ void post_peers(const CycleParams &p, int phase, unsigned long long e) {
  for (int r = 0; r < p.n_ranks; ++r) {
    if (r == p.rank) continue;
    st_release_sys(p.peer_flags[r] + flag_index(p.lane, p.rank, phase), e);
  }
}

// Optional phase trace (thread 0 of each block): earliest start, latest
// "ready for data" (pull: arrive barrier passed), latest end of data work,
// and the moment the depart barrier completed.
__device__ __forceinline__ void trace_min(const CycleParams &p, int slot) {
  if (p.trace) atomicMin(p.trace + slot, globaltimer());
}
__device__ __forceinline__ void trace_max(const CycleParams &p, int slot) {
  if (p.trace) atomicMax(p.trace + slot, globaltimer());
}

// Exit barrier: the last block of this launch tells every peer that all of
// this device's stores (local and remote) are done, then waits for theirs,
// so nobody resumes training on a buffer a peer is still writing.
__device__ void depart(const CycleParams &p, unsigned long long epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    trace_max(p, 2);
    __threadfence_system();
    const unsigned prev = atomicAdd(&p.state->done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      post_peers(p, 1, epoch);
      if (*(volatile unsigned *)p.status == 0) wait_peers(p, 1, epoch);
      trace_max(p, 3);
      p.state->done = 0u;
      *(volatile unsigned long long *)&p.state->epoch = epoch;
      __threadfence();
    }
  }
}

template <int VB>
struct RawVec;
template <>
struct RawVec<16> {
  using type = uint4;
};
template <>
struct RawVec<8> {
  using type = uint2;
};
template <>
struct RawVec<4> {
  using type = unsigned int;
};

template <typename T, int VB>
union Lanes {
  typename RawVec<VB>::type raw;
  T v[VB / sizeof(T)];
};

template <typename T, typename Acc>
__device__ __forceinline__ T finish(Acc acc, const CycleParams &p) {
  // IEEE true division by C (multiring.py:219).  For C a power of two the
  // product with the exact reciprocal is the same correctly rounded value.
  const Acc q = p.pow2 ? acc * (Acc)p.inv_c : acc / (Acc)p.C;
  return (T)q;
}

// Element i of member m as this device reads it.  Pull: the member's own
// buffer (local or peer).  Push: the owner's own buffer for m == me, else the
// staging slot member m pushed into.
template <typename T, bool PUSH>
__device__ __forceinline__ const T *member_elem(const CycleParams &p, const Seg &s, int m, int64_t i) {
  if (!PUSH || m == p.me) return static_cast<const T *>(p.src[m]) + i;
  return static_cast<const T *>(p.stage[p.me]) + ((int64_t)m * p.stride + s.stage_off + (i - s.lo));
}

// Fold of one element (chunk edges, misaligned buffers): ring order from s.k.
template <typename T, typename Acc, bool PUSH>
__device__ __forceinline__ void fold_scalar(const CycleParams &p, const Seg &s, int64_t i) {
  int m = s.k;
  Acc acc = (Acc)__ldcs(member_elem<T, PUSH>(p, s, m, i));
  for (int q = 1; q < p.C; ++q) {
    m = (m + 1 == p.C) ? 0 : m + 1;
    acc = acc + (Acc)__ldcs(member_elem<T, PUSH>(p, s, m, i));
  }
  const T out = finish<T, Acc>(acc, p);
  for (int q = 0; q < p.C; ++q) __stcs(static_cast<T *>(p.dst[q]) + i, out);
}

// Fold one pass of chunk s: this thread takes vectors j0 + u*kThreads
// (u < U, below jend), loads all C members of each (U*C loads in flight),
// folds in ring order, divides, and stores the mean into all C buffers.
template <typename T, typename Acc, int CB, int VB, int U, bool PUSH>
__device__ __forceinline__ void fold_pass(const CycleParams &p, const Seg &s, int64_t j0, int64_t jend) {
  constexpr int N = VB / sizeof(T);
  using Raw = typename RawVec<VB>::type;
  Lanes<T, VB> x[U][CB];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t j = j0 + (int64_t)u * kThreads;
    if (j < jend) {
      const int64_t i = s.body_lo + j * N;
#pragma unroll
      for (int q = 0; q < CB; ++q) {
        if (q < p.C) {
          int m = s.k + q;
          if (m >= p.C) m -= p.C;
          x[u][q].raw = __ldcs(reinterpret_cast<const Raw *>(member_elem<T, PUSH>(p, s, m, i)));
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t j = j0 + (int64_t)u * kThreads;
    if (j < jend) {
      Lanes<T, VB> out;
#pragma unroll
      for (int e = 0; e < N; ++e) {
        Acc acc = (Acc)x[u][0].v[e];
#pragma unroll
        for (int q = 1; q < CB; ++q)
          if (q < p.C) acc = acc + (Acc)x[u][q].v[e];
        out.v[e] = finish<T, Acc>(acc, p);
      }
      const int64_t i = s.body_lo + j * N;
#pragma unroll
      for (int q = 0; q < CB; ++q)
        if (q < p.C) __stcs(reinterpret_cast<Raw *>(static_cast<T *>(p.dst[q]) + i), out.raw);
    }
  }
}

// ---------------------------------------------------------------------------
// pull protocol: the owner of chunk k reads chunk k of every member (local
// HBM or NVLink peer loads) and pushes the mean into every member.  Arrive
// barrier first (peers' inputs final), depart barrier last.

// Two 256-thread blocks per SM (<= 128 registers): measured 1.18 ms vs
// 1.47 ms at one block per SM on the co-resident BERT cycle.
template <typename T, typename Acc, int CB, int VB, int U, int MINB = 2>
__global__ void __launch_bounds__(kThreads, MINB)
ring_cycle_kernel(const __grid_constant__ CycleParams p) {
  constexpr int N = VB / sizeof(T);
  __shared__ int s_go;
  unsigned long long epoch = 0;

  if (threadIdx.x == 0) trace_min(p, 0);
  if (p.n_ranks > 1) {
    if (threadIdx.x == 0) {
      epoch = *(volatile unsigned long long *)&p.state->epoch + 1ull;
      int go = (*(volatile unsigned *)p.status == 0);
      if (go) {
        // first block of this launch posts "inputs final" to every peer
        if (atomicCAS(&p.state->signaled, epoch - 1ull, epoch) == epoch - 1ull) {
          __threadfence_system();
          post_peers(p, 0, epoch);
        }
        go = wait_peers(p, 0, epoch);
      }
      trace_max(p, 1);
      s_go = go;
    }
    __syncthreads();
  } else {
    if (threadIdx.x == 0) s_go = 1;
    __syncthreads();
  }

  if (s_go) {
    const int64_t tile_vecs = (int64_t)kThreads * U;
    for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
      int a = 0, b = p.nseg - 1;
      while (a < b) {
        const int mid = (a + b + 1) >> 1;
        if (__ldg(p.tile_prefix + mid) <= t) a = mid; else b = mid - 1;
      }
      const Seg s = p.segs[a];
      const int64_t local_tile = t - __ldg(p.tile_prefix + a);
      const int64_t nvec = (s.body_hi - s.body_lo) / N;
      const int64_t jbeg = local_tile * tile_vecs;
      fold_pass<T, Acc, CB, VB, U, false>(p, s, jbeg + threadIdx.x, min(nvec, jbeg + tile_vecs));
      if (local_tile == 0) {
        const int64_t nhead = s.body_lo - s.lo, ntail = s.hi - s.body_hi;
        if ((int64_t)threadIdx.x < nhead + ntail) {
          const int64_t i = (int64_t)threadIdx.x < nhead ? s.lo + threadIdx.x
                                                          : s.body_hi + ((int64_t)threadIdx.x - nhead);
          fold_scalar<T, Acc, false>(p, s, i);
        }
      }
    }
  }
  if (p.n_ranks > 1) {
    depart(p, epoch);
  } else if (p.trace) {
    __syncthreads();
    if (threadIdx.x == 0) trace_max(p, 2);
  }
}

// ---------------------------------------------------------------------------
// push protocol (one position per rank, rank == position): NVLink carries
// stores only.  Scatter: this rank copies its chunk-q slice of every ring into
// owner q's staging slot and raises one release flag per 256 KB unit.  Fold:
// for its own chunk, once every writer's flag for a unit is up, the owner
// folds its own values and the staged ones in ring order and pushes the mean
// into all members.  No arrive barrier is needed: a member's chunk reaches
// the owner only after its kernel started (inputs final), and the owner
// writes a member's buffer only after receiving that member's data for the
// same unit.  The depart barrier still closes the cycle.

template <typename T>
__device__ __forceinline__ Seg find_unit(const Seg *segs, int nseg, int64_t u) {
  int a = 0, b = nseg - 1;
  while (a < b) {
    const int mid = (a + b + 1) >> 1;
    if (segs[mid].unit0 <= u) a = mid; else b = mid - 1;
  }
  return segs[a];
}

template <typename T, typename Acc, int CB, int VB, int U>
__global__ void __launch_bounds__(kThreads, 2)
ring_push_kernel(const __grid_constant__ CycleParams p) {
  constexpr int N = VB / sizeof(T);
  constexpr int KC = (U * CB) < 8 ? (U * CB) : 8;  // vectors in flight per thread when copying
  using Raw = typename RawVec<VB>::type;
  __shared__ int s_ok;
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) {
    trace_min(p, 0);
    trace_max(p, 1);
    s_epoch = *(volatile unsigned long long *)&p.state->epoch + 1ull;
    s_ok = (*(volatile unsigned *)p.status == 0);
  }
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  const int C = p.C, me = p.me;
  const int64_t n_scatter = (int64_t)(C - 1) * p.scatter_umax;
  const int64_t n_work = n_scatter + p.ounits[me];
  const unsigned long long t0 = globaltimer();

  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    if (!s_ok) break;
    if (w < n_scatter) {
      const int r = (int)(w % (C - 1));
      const int64_t u = w / (C - 1);
      int q = me + 1 + r;
      if (q >= C) q -= C;
      if (u >= p.ounits[q]) continue;
      const Seg s = find_unit<T>(p.segs + p.oseg_base[q], p.oseg_base[q + 1] - p.oseg_base[q], u);
      const int64_t uu = u - s.unit0;
      const int64_t nvec = (s.body_hi - s.body_lo) / N;
      const int64_t jbeg = uu * p.unit_vecs, jend = min(nvec, jbeg + p.unit_vecs);
      const T *src = static_cast<const T *>(p.src[me]);
      T *stg = static_cast<T *>(p.stage[q]) + ((int64_t)me * p.stride + s.stage_off - s.lo);
      for (int64_t j0 = jbeg + threadIdx.x; j0 < jend; j0 += (int64_t)kThreads * KC) {
        Raw v[KC];
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          const int64_t j = j0 + (int64_t)c * kThreads;
          if (j < jend) v[c] = __ldcs(reinterpret_cast<const Raw *>(src + s.body_lo + j * N));
        }
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          const int64_t j = j0 + (int64_t)c * kThreads;
          if (j < jend) __stcs(reinterpret_cast<Raw *>(stg + s.body_lo + j * N), v[c]);
        }
      }
      if (uu == 0) {
        const int64_t nhead = s.body_lo - s.lo, ntail = s.hi - s.body_hi;
        if ((int64_t)threadIdx.x < nhead + ntail) {
          const int64_t i = (int64_t)threadIdx.x < nhead ? s.lo + threadIdx.x
                                                          : s.body_hi + ((int64_t)threadIdx.x - nhead);
          stg[i] = src[i];
        }
      }
      __threadfence_system();  // this thread's stores, before the unit flag
      __syncthreads();
      if (threadIdx.x == 0)
        st_release_sys(p.pflags[q] + pflag_index(p.lane, C, me, p.units_max, u), epoch);
    } else {
      const int64_t u = w - n_scatter;
      const Seg s = find_unit<T>(p.segs + p.oseg_base[me], p.oseg_base[me + 1] - p.oseg_base[me], u);
      if (threadIdx.x == 0) {
        for (int m = 0; m < C && s_ok; ++m) {
          if (m == me) continue;
          const unsigned diag = (2u << 16) | ((unsigned)p.lane << 8) | (unsigned)m;
          if (!wait_flag(p, p.pflags[me] + pflag_index(p.lane, C, m, p.units_max, u), epoch, t0, diag)) s_ok = 0;
        }
      }
      __syncthreads();
      if (!s_ok) break;
      const int64_t uu = u - s.unit0;
      const int64_t nvec = (s.body_hi - s.body_lo) / N;
      const int64_t jbeg = uu * p.unit_vecs, jend = min(nvec, jbeg + p.unit_vecs);
      for (int64_t j0 = jbeg + threadIdx.x; j0 < jend; j0 += (int64_t)kThreads * U)
        fold_pass<T, Acc, CB, VB, U, true>(p, s, j0, jend);
      if (uu == 0) {
        const int64_t nhead = s.body_lo - s.lo, ntail = s.hi - s.body_hi;
        if ((int64_t)threadIdx.x < nhead + ntail) {
          const int64_t i = (int64_t)threadIdx.x < nhead ? s.lo + threadIdx.x
                                                          : s.body_hi + ((int64_t)threadIdx.x - nhead);
          fold_scalar<T, Acc, true>(p, s, i);
        }
      }
      __syncthreads();  // s_ok is re-armed by thread 0 for the next unit
    }
  }
  depart(p, epoch);
}

// ---------------------------------------------------------------------------
// co-resident TMA path (all C members on this device, 16-byte congruent
// buffers): HBM-bound, so tiles stream through shared memory with bulk async
// copies.  Warp 0 / lane 0 produces: for each tile it loads the tile of all C
// members (cp.async.bulk global->shared, completion on a per-stage mbarrier)
// into a STAGES-deep ring.  Warps 1..8 consume: fold from shared memory in
// ring order, write the mean tile to shared memory, and one consumer issues
// C bulk stores (shared->global) of it, double-buffered.  No register
// staging of loads, so each SM keeps STAGES * C * TV * 16 bytes in flight.

constexpr int kTmaConsumers = 256;

__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_load(void *smem, const void *gmem, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void bulk_store(void *gmem, const void *smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_addr(smem)),
               "r"(bytes)
               : "memory");
}

template <typename T, typename Acc, int CB, int TV, int STAGES>
__global__ void __launch_bounds__(kTmaConsumers + 32, 2)
ring_tma_kernel(const __grid_constant__ CycleParams p) {
  constexpr int N = 16 / sizeof(T);
  extern __shared__ __align__(128) unsigned char smem[];
  uint4 *in = reinterpret_cast<uint4 *>(smem);                       // [STAGES][CB][TV]
  uint4 *out = in + (size_t)STAGES * CB * TV;                          // [2][TV]
  __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
  const int tid = threadIdx.x;
  const int C = p.C;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    trace_min(p, 0);
    trace_max(p, 1);
  }
  __syncthreads();

  // the tiles this block owns: t = blockIdx.x + i * gridDim.x
  auto seg_of = [&](int64_t t, int64_t *local) -> Seg {
    int a = 0, b = p.nseg - 1;
    while (a < b) {
      const int mid = (a + b + 1) >> 1;
      if (__ldg(p.tile_prefix + mid) <= t) a = mid; else b = mid - 1;
    }
    *local = t - __ldg(p.tile_prefix + a);
    return p.segs[a];
  };

  if (tid < 32) {
    if (tid == 0) {  // producer
      int stage = 0;
      unsigned phase = 0;
      int64_t n = 0;
      for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++n) {
        int64_t lt;
        const Seg s = seg_of(t, &lt);
        const int64_t nvec = (s.body_hi - s.body_lo) / N;
        const int64_t j0 = lt * TV;
        const int cnt = (int)max((int64_t)0, min((int64_t)TV, nvec - j0));
        if (n >= STAGES) mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], (unsigned)(cnt * 16 * C));
        if (cnt > 0) {
          for (int q = 0; q < C; ++q) {
            int m = s.k + q;
            if (m >= C) m -= C;
            bulk_load(in + ((size_t)stage * CB + q) * TV, static_cast<const T *>(p.src[m]) + s.body_lo + j0 * N,
                      (unsigned)(cnt * 16), &full[stage]);
          }
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  // consumers (256 threads)
  const int c = tid - 32;
  int stage = 0;
  unsigned phase = 0;
  int ob = 0;
  for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
    int64_t lt;
    const Seg s = seg_of(t, &lt);
    const int64_t nvec = (s.body_hi - s.body_lo) / N;
    const int64_t j0 = lt * TV;
    const int cnt = (int)max((int64_t)0, min((int64_t)TV, nvec - j0));
    mbar_wait(&full[stage], phase);
    // consumer 0 finished the previous tile's store bookkeeping (out[ob] free)
    asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers) : "memory");
    for (int v = c; v < cnt; v += kTmaConsumers) {
      Lanes<T, 16> x, o;
      Acc acc[N];
      x.raw = in[((size_t)stage * CB + 0) * TV + v];
#pragma unroll
      for (int e = 0; e < N; ++e) acc[e] = (Acc)x.v[e];
#pragma unroll
      for (int q = 1; q < CB; ++q) {
        if (q < C) {
          x.raw = in[((size_t)stage * CB + q) * TV + v];
#pragma unroll
          for (int e = 0; e < N; ++e) acc[e] = acc[e] + (Acc)x.v[e];
        }
      }
#pragma unroll
      for (int e = 0; e < N; ++e) o.v[e] = finish<T, Acc>(acc[e], p);
      out[ob * TV + v] = o.raw;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers) : "memory");
    if (c == 0) {
      mbar_arrive(&empty[stage]);  // every consumer has read this stage
      if (cnt > 0) {
        for (int q = 0; q < C; ++q)
          bulk_store(static_cast<T *>(p.dst[q]) + s.body_lo + j0 * N, out + ob * TV, (unsigned)(cnt * 16));
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // out[ob ^ 1] reusable
    }
    if (lt == 0) {
      const int64_t nhead = s.body_lo - s.lo, ntail = s.hi - s.body_hi;
      if ((int64_t)c < nhead + ntail) {
        const int64_t i = (int64_t)c < nhead ? s.lo + c : s.body_hi + ((int64_t)c - nhead);
        fold_scalar<T, Acc, false>(p, s, i);
      }
    }
    ob ^= 1;
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
  if (c == 0) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    trace_max(p, 2);
  }
}

// live <- mean + (live - snap); exactly mean where live == snap bitwise.
template <typename T, typename U>
__global__ void __launch_bounds__(kThreads)
blend_kernel(T *__restrict__ live, const T *__restrict__ snap, const T *__restrict__ mean, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const T l = live[i], s = snap[i], m = __ldcs(mean + i);
    U lb, sb;
    memcpy(&lb, &l, sizeof(T));
    memcpy(&sb, &s, sizeof(T));
    live[i] = (lb == sb) ? m : (m + (l - s));
  }
}

template <typename T, typename U>
__global__ void __launch_bounds__(kThreads)
blend_kernel_v4(T *__restrict__ live, const T *__restrict__ snap, const T *__restrict__ mean, int64_t nvec) {
  constexpr int N = 16 / sizeof(T);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nvec; j += stride) {
    Lanes<T, 16> l, s, m, o;
    l.raw = *reinterpret_cast<const uint4 *>(live + j * N);
    s.raw = __ldcs(reinterpret_cast<const uint4 *>(snap + j * N));
    m.raw = __ldcs(reinterpret_cast<const uint4 *>(mean + j * N));
#pragma unroll
    for (int e = 0; e < N; ++e) {
      U lb, sb;
      memcpy(&lb, &l.v[e], sizeof(T));
      memcpy(&sb, &s.v[e], sizeof(T));
      o.v[e] = (lb == sb) ? m.v[e] : (m.v[e] + (l.v[e] - s.v[e]));
    }
    *reinterpret_cast<uint4 *>(live + j * N) = o.raw;
  }
}

// ---------------------------------------------------------------------------
// kernel dispatch

using KernelFn = void (*)(CycleParams);

enum Mode { kF32Acc64 = 0, kF32Native = 1, kF64 = 2 };

// Vectors per thread per pass: U*C 16-byte loads in flight, kept within the
// 128-register budget (fp64 storage and the push kernel's staging addresses
// take more registers, so they run at half U).
template <typename T, typename Acc, int VB>
KernelFn pick_cb(int c, bool push, int *u_out) {
  constexpr bool wide = sizeof(T) == 8;
  if (push) {
    if (c <= 2) { *u_out = 4; return ring_push_kernel<T, Acc, 2, VB, 4>; }
    if (c <= 4) { *u_out = 2; return ring_push_kernel<T, Acc, 4, VB, 2>; }
    if (c <= 8) { *u_out = 1; return ring_push_kernel<T, Acc, 8, VB, 1>; }
    *u_out = 1;
    return ring_push_kernel<T, Acc, 16, VB, 1>;
  }
  if constexpr (wide) {
    if (c <= 2) { *u_out = 4; return ring_cycle_kernel<T, Acc, 2, VB, 4>; }
    if (c <= 4) { *u_out = 2; return ring_cycle_kernel<T, Acc, 4, VB, 2>; }
    if (c <= 8) { *u_out = 1; return ring_cycle_kernel<T, Acc, 8, VB, 1>; }
  } else {
    if (c <= 2) { *u_out = 8; return ring_cycle_kernel<T, Acc, 2, VB, 8>; }
    if (c <= 4) { *u_out = 4; return ring_cycle_kernel<T, Acc, 4, VB, 4>; }
    if (c <= 8) { *u_out = 2; return ring_cycle_kernel<T, Acc, 8, VB, 2>; }
  }
  *u_out = 1;
  return ring_cycle_kernel<T, Acc, 16, VB, 1>;
}

// Tuning variants of the f32 / f64-fold vector pull kernel (RAVNEST_B200_VARIANT,
// experiments only): 1 = half the vectors per thread, >= 3 blocks/SM;
// 2 = half, >= 4 blocks/SM; 3 = same vectors, no register cap (1 block/SM).
template <int CB, int U>
KernelFn pick_variant(int v, int *u_out) {
  constexpr int H = U > 1 ? U / 2 : 1;
  switch (v) {
    case 1: *u_out = H; return ring_cycle_kernel<float, double, CB, 16, H, 3>;
    case 2: *u_out = H; return ring_cycle_kernel<float, double, CB, 16, H, 4>;
    case 3: *u_out = U; return ring_cycle_kernel<float, double, CB, 16, U, 1>;
    default: *u_out = U; return ring_cycle_kernel<float, double, CB, 16, U, 2>;
  }
}

// Co-resident TMA kernel: 32 KB of member data per pipeline stage
// (CB * TV * 16 bytes), 3 stages -> 104 KB of shared memory, two blocks per
// SM (measured best of 3/4/6 stages: 0.918 of measured HBM on BERT C=8).
constexpr int kTmaStages = 3;
constexpr int kTmaStageBytes = 32 * 1024;

template <typename T, typename Acc, int STAGES, int STAGE_BYTES>
KernelFn pick_tma(int c, int *tv_out) {
  if (c <= 2) { *tv_out = STAGE_BYTES / (2 * 16); return ring_tma_kernel<T, Acc, 2, STAGE_BYTES / (2 * 16), STAGES>; }
  if (c <= 4) { *tv_out = STAGE_BYTES / (4 * 16); return ring_tma_kernel<T, Acc, 4, STAGE_BYTES / (4 * 16), STAGES>; }
  if (c <= 8) { *tv_out = STAGE_BYTES / (8 * 16); return ring_tma_kernel<T, Acc, 8, STAGE_BYTES / (8 * 16), STAGES>; }
  *tv_out = STAGE_BYTES / (16 * 16);
  return ring_tma_kernel<T, Acc, 16, STAGE_BYTES / (16 * 16), STAGES>;
}

KernelFn pick_tma_kernel(int mode, int c, int *tv_out, size_t *smem_out) {
  // RAVNEST_B200_TMA_VARIANT (experiments): 1 = 6 stages, 2 = 4 stages (one
  // block per SM), 3 = 8 stages of 16 KB
  const char *ve = getenv("RAVNEST_B200_TMA_VARIANT");
  const int v = ve ? atoi(ve) : 0;
  int stages = kTmaStages;
  KernelFn k;
  if (v > 0 && mode == kF32Acc64) {
    if (v == 1) { stages = 6; k = pick_tma<float, double, 6, kTmaStageBytes>(c, tv_out); }
    else if (v == 2) { stages = 4; k = pick_tma<float, double, 4, kTmaStageBytes>(c, tv_out); }
    else { stages = 8; k = pick_tma<float, double, 8, 16 * 1024>(c, tv_out); }
  } else {
    k = mode == kF32Acc64 ? pick_tma<float, double, kTmaStages, kTmaStageBytes>(c, tv_out)
      : mode == kF32Native ? pick_tma<float, float, kTmaStages, kTmaStageBytes>(c, tv_out)
                           : pick_tma<double, double, kTmaStages, kTmaStageBytes>(c, tv_out);
  }
  const int cb = c <= 2 ? 2 : c <= 4 ? 4 : c <= 8 ? 8 : 16;
  *smem_out = (size_t)stages * cb * (*tv_out) * 16 + 2 * (size_t)(*tv_out) * 16;
  return k;
}

KernelFn pick_kernel(int mode, int c, bool vec, bool push, int *u_out) {
  const char *ve = getenv("RAVNEST_B200_VARIANT");
  const int variant = ve ? atoi(ve) : 0;
  if (variant > 0 && mode == kF32Acc64 && vec && !push) {
    if (c <= 2) return pick_variant<2, 8>(variant, u_out);
    if (c <= 4) return pick_variant<4, 4>(variant, u_out);
    if (c <= 8) return pick_variant<8, 2>(variant, u_out);
    return pick_variant<16, 1>(variant, u_out);
  }
  switch (mode) {
    case kF32Acc64: return vec ? pick_cb<float, double, 16>(c, push, u_out) : pick_cb<float, double, 4>(c, push, u_out);
    case kF32Native: return vec ? pick_cb<float, float, 16>(c, push, u_out) : pick_cb<float, float, 4>(c, push, u_out);
    default: return vec ? pick_cb<double, double, 16>(c, push, u_out) : pick_cb<double, double, 8>(c, push, u_out);
  }
}

// ---------------------------------------------------------------------------
// driver entry point for cuMemGetAddressRange (no link-time libcuda dependency)

typedef int (*PFN_getAddressRange)(unsigned long long *, size_t *, unsigned long long);

int alloc_base(const void *ptr, unsigned long long *base) {
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess || !f) return set_err(RV_E_CUDA, "cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<PFN_getAddressRange>(f);
  }
  size_t size = 0;
  int rc = fn(base, &size, (unsigned long long)(uintptr_t)ptr);
  if (rc != 0) return set_err(RV_E_ARG, "cuMemGetAddressRange(%p) failed (%d)", ptr, rc);
  return RV_OK;
}

struct IpcEntry {
  void *base;
  int refs;
};
std::mutex g_ipc_mu;
std::map<std::pair<int, std::string>, IpcEntry> g_ipc;  // (device, handle bytes) -> mapping

}  // namespace

// ---------------------------------------------------------------------------
// plan

struct rv_plan {
  int device = 0;
  int C = 0, R = 0;
  int64_t total = 0;
  int dtype = RV_DTYPE_F32, acc = RV_ACC_F64;
  int proto = RV_PROTO_PULL;
  std::vector<int64_t> rstart, rlen;
  std::vector<const void *> src;
  std::vector<void *> dst;
  std::vector<char> bound;
  std::vector<int> local;
  int n_lanes = 1;
  int rank = 0, n_ranks = 1;
  std::vector<unsigned long long *> peer_flags;
  unsigned long long *flags = nullptr;  // capacity max(R,1) lanes x RV_MAX_RANKS x 2
  size_t flag_bytes = 0;
  LaneState *states = nullptr;  // max(R,1)
  unsigned int *status = nullptr;
  unsigned long long timeout_ns = 20ull * 1000000000ull;
  int sm_count = 0;
  // push protocol: [unit flags | staging] in one IPC-exportable allocation
  char *push_area = nullptr;
  size_t push_bytes = 0, pflag_bytes = 0;
  int64_t stride_bound = 0, units_max = 0;
  int push_lanes = 0;
  std::vector<char *> peer_push;  // by rank
  unsigned long long *trace = nullptr;  // lanes x 4, when tracing
  std::vector<cudaEvent_t> h2d_done;    // host-buffer pipeline, one per lane
  // built lane tables
  bool dirty = true;       // local positions / lanes / peers / protocol changed
  bool ptrs_dirty = true;  // buffers rebound: rebuild only if the alignment class changed
  int built_vec = -1;
  int64_t built_a0 = -1;
  struct Lane {
    Seg *segs = nullptr;
    int64_t *prefix = nullptr;
    int nseg = 0;
    int64_t n_tiles = 0;
    int64_t elems = 0;
    std::vector<int> rings;
    int grid = 0;
    // push
    int64_t stride = 0, unit_vecs = 0, scatter_umax = 0;
    std::vector<int64_t> ounits;
    std::vector<int> oseg_base;
  };
  std::vector<Lane> lanes;
  KernelFn kernel = nullptr;
  int occ = 0;
  bool use_push = false;
  int block_threads = kThreads;
  size_t smem_bytes = 0;
  int max_blocks = 0;  // 0 = whole device; else cap on resident blocks (SM budget)
};

namespace {

void free_lanes(rv_plan *p) {
  for (auto &l : p->lanes) {
    if (l.segs) cudaFree(l.segs);
    if (l.prefix) cudaFree(l.prefix);
  }
  p->lanes.clear();
}

int elem_size(int dtype) { return dtype == RV_DTYPE_F64 ? 8 : 4; }

// chunk bounds of ring r (multiring.py:134-144)
std::vector<std::pair<int64_t, int64_t>> ring_chunks(const rv_plan *p, int r) {
  std::vector<std::pair<int64_t, int64_t>> b(p->C);
  const int64_t base = p->rlen[r] / p->C, rem = p->rlen[r] % p->C;
  int64_t lo = p->rstart[r];
  for (int k = 0; k < p->C; ++k) {
    const int64_t n = base + (k < rem ? 1 : 0);
    b[k] = {lo, lo + n};
    lo += n;
  }
  return b;
}

// vector body of [lo, hi): element i is 16-byte aligned iff (i + a0) % N == 0
void set_body(Seg &s, int N, int64_t a0) {
  int64_t blo = s.lo + ((N - (s.lo + a0) % N) % N);
  int64_t bhi = s.hi - ((s.hi + a0) % N);
  if (bhi <= blo) blo = bhi = s.hi;  // no aligned vector: all edge elements (< 2N)
  s.body_lo = blo;
  s.body_hi = bhi;
}

bool push_active(const rv_plan *p) { return p->proto == RV_PROTO_PUSH && p->n_ranks > 1; }

// Upper bounds of the push layout, from the schedule alone (before any
// pointer is known): staging elements per writer slot, unit flags per lane.
void push_bounds(const rv_plan *p, int64_t *stride_bound, int64_t *units_max) {
  const int es = elem_size(p->dtype);
  const int64_t nmax = 16 / es, unit_elems = kMinUnitBytes / es;
  int64_t stride = nmax;
  int64_t umax = 1;
  for (int l = 0; l < p->n_lanes; ++l) {
    int64_t u = 0;
    for (int r = l; r < p->R; r += p->n_lanes) {
      const int64_t chunk = (p->rlen[r] + p->C - 1) / p->C;
      u += (chunk + unit_elems - 1) / unit_elems + 1;
    }
    umax = std::max(umax, u);
  }
  for (int r = 0; r < p->R; ++r) stride += (p->rlen[r] + p->C - 1) / p->C + 2 * nmax;
  *stride_bound = (stride + 63) / 64 * 64;  // writer slots stay 256-byte aligned
  *units_max = umax;
}

int upload(rv_plan::Lane &lane, const std::vector<Seg> &segs, const std::vector<int64_t> &prefix) {
  if (segs.empty()) return RV_OK;
  RV_CUDA(cudaMalloc(&lane.segs, sizeof(Seg) * segs.size()));
  RV_CUDA(cudaMemcpy(lane.segs, segs.data(), sizeof(Seg) * segs.size(), cudaMemcpyHostToDevice));
  if (!prefix.empty()) {
    RV_CUDA(cudaMalloc(&lane.prefix, sizeof(int64_t) * prefix.size()));
    RV_CUDA(cudaMemcpy(lane.prefix, prefix.data(), sizeof(int64_t) * prefix.size(), cudaMemcpyHostToDevice));
  }
  return RV_OK;
}

int build_tables(rv_plan *p) {
  for (int i = 0; i < p->C; ++i)
    if (!p->bound[i]) return set_err(RV_E_ARG, "cluster position %d is not bound", i);
  if (p->local.empty()) return set_err(RV_E_ARG, "no local positions set");
  const int es = elem_size(p->dtype);
  // vector path needs every member buffer congruent modulo 16 bytes
  const uintptr_t a = (uintptr_t)p->src[0] % 16;
  bool vec = true;
  for (int i = 0; i < p->C; ++i) {
    if ((uintptr_t)p->src[i] % es || (uintptr_t)p->dst[i] % es)
      return set_err(RV_E_ARG, "buffer of position %d is not %d-byte aligned", i, es);
    if ((uintptr_t)p->src[i] % 16 != a || (uintptr_t)p->dst[i] % 16 != a) vec = false;
  }
  const int N = vec ? 16 / es : 1;
  const int64_t a0 = vec ? (int64_t)(a / es) : 0;
  p->ptrs_dirty = false;
  if (!p->dirty && p->built_vec == (int)vec && p->built_a0 == a0) return RV_OK;
  p->built_vec = (int)vec;
  p->built_a0 = a0;
  const bool push = push_active(p);
  if (push) {
    if (p->n_ranks != p->C || p->local.size() != 1 || p->local[0] != p->rank)
      return set_err(RV_E_CONFIG, "push protocol needs one position per rank with rank == position");
    if (!p->push_area || p->push_lanes != p->n_lanes)
      return set_err(RV_E_ARG, "push area not allocated for %d lanes (call rv_plan_push_area)", p->n_lanes);
    for (int r = 0; r < p->n_ranks; ++r)
      if (!p->peer_push[r]) return set_err(RV_E_ARG, "push area of rank %d missing", r);
  }
  p->use_push = push;
  const int mode = p->dtype == RV_DTYPE_F64 ? kF64 : (p->acc == RV_ACC_NATIVE ? kF32Native : kF32Acc64);
  int U = 1;
  int64_t tile_vecs = 0;
  DeviceGuard g(p->device);
  const char *tma_env = getenv("RAVNEST_B200_TMA");
  const bool tma = vec && p->n_ranks == 1 && !(tma_env && tma_env[0] == '0');
  if (tma) {
    int tv = 0;
    p->kernel = pick_tma_kernel(mode, p->C, &tv, &p->smem_bytes);
    p->block_threads = kTmaConsumers + 32;
    RV_CUDA(cudaFuncSetAttribute(p->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->smem_bytes));
    tile_vecs = tv;
  } else {
    p->kernel = pick_kernel(mode, p->C, vec, push, &U);
    p->block_threads = kThreads;
    p->smem_bytes = 0;
    tile_vecs = (int64_t)kThreads * U;
  }
  RV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->occ, p->kernel, p->block_threads, p->smem_bytes));
  if (p->occ < 1) p->occ = 1;
  // push: unit size adapts so that a cycle has >= ~2 work items per resident
  // block (small shards stay parallel, large ones amortise the unit flags);
  // it depends only on the schedule and the device model, so every rank
  // derives the same layout
  int64_t unit_vecs = kUnitBytes / (N * es);
  if (push) {
    int64_t owner_elems = 0;
    for (int q = 0; q < p->C; ++q) {
      int64_t e = 0;
      for (int r = 0; r < p->R; ++r) {
        const auto b = ring_chunks(p, r);
        e += b[q].second - b[q].first;
      }
      owner_elems = std::max(owner_elems, e);
    }
    const int64_t items = std::max<int64_t>(1, 2LL * p->sm_count * p->occ);
    const int64_t want = (owner_elems / N * (p->C - 1) + items - 1) / items;
    const int64_t lo = kMinUnitBytes / (N * es), hi = kUnitBytes / (N * es);
    unit_vecs = std::min(hi, std::max(lo, (want + kThreads - 1) / kThreads * kThreads));
  }

  free_lanes(p);
  p->lanes.resize(p->n_lanes);
  std::vector<int> loc = p->local;
  std::sort(loc.begin(), loc.end());
  std::vector<int64_t> cursor(p->C, 0);  // push: staging cursor per owner, across lanes
  int64_t all_elems = 0;
  for (int l = 0; l < p->n_lanes; ++l) {
    rv_plan::Lane &lane = p->lanes[l];
    std::vector<Seg> segs;
    std::vector<int64_t> prefix(1, 0);
    for (int r = l; r < p->R; r += p->n_lanes) lane.rings.push_back(r);
    if (!push) {
      for (int r : lane.rings) {
        const auto bounds = ring_chunks(p, r);
        for (int k : loc) {
          Seg s{};
          s.lo = bounds[k].first;
          s.hi = bounds[k].second;
          s.k = k;
          s.ring = r;
          if (s.hi <= s.lo) continue;
          set_body(s, N, a0);
          const int64_t nvec = (s.body_hi - s.body_lo) / N;
          segs.push_back(s);
          prefix.push_back(prefix.back() + std::max<int64_t>(1, (nvec + tile_vecs - 1) / tile_vecs));
          lane.elems += s.hi - s.lo;
        }
      }
      lane.nseg = (int)segs.size();
      lane.n_tiles = prefix.back();
      int rc = upload(lane, segs, prefix);
      if (rc) return rc;
    } else {
      // every owner's chunks (owner-major): writers need the owners' layouts
      lane.ounits.assign(p->C, 0);
      lane.oseg_base.assign(p->C + 1, 0);
      for (int q = 0; q < p->C; ++q) {
        lane.oseg_base[q] = (int)segs.size();
        int64_t u = 0;
        for (int r : lane.rings) {
          const auto bounds = ring_chunks(p, r);
          Seg s{};
          s.lo = bounds[q].first;
          s.hi = bounds[q].second;
          s.k = q;
          s.ring = r;
          if (s.hi <= s.lo) continue;
          set_body(s, N, a0);
          // staging index of element i is stage_off + (i - lo); keep it
          // vector-aligned exactly where the source is
          const int64_t c0 = (cursor[q] + N - 1) / N * N;
          s.stage_off = c0 + ((s.lo + a0) % N);
          cursor[q] = s.stage_off + (s.hi - s.lo);
          s.unit0 = u;
          const int64_t nvec = (s.body_hi - s.body_lo) / N;
          u += std::max<int64_t>(1, (nvec + unit_vecs - 1) / unit_vecs);
          segs.push_back(s);
          if (q == p->rank) lane.elems += s.hi - s.lo;
        }
        lane.ounits[q] = u;
        if (u > p->units_max) return set_err(RV_E_ARG, "push unit bound exceeded (%lld > %lld)",
                                             (long long)u, (long long)p->units_max);
      }
      lane.oseg_base[p->C] = (int)segs.size();
      lane.unit_vecs = unit_vecs;
      lane.scatter_umax = 0;
      for (int q = 0; q < p->C; ++q)
        if (q != p->rank) lane.scatter_umax = std::max(lane.scatter_umax, lane.ounits[q]);
      lane.nseg = (int)segs.size();
      lane.n_tiles = (int64_t)(p->C - 1) * lane.scatter_umax + lane.ounits[p->rank];
      int rc = upload(lane, segs, {});
      if (rc) return rc;
    }
    all_elems += lane.elems;
  }
  if (push) {
    int64_t stride = 0;
    for (int q = 0; q < p->C; ++q) stride = std::max(stride, cursor[q]);
    stride = (stride + 15) / 16 * 16;
    if (stride > p->stride_bound)
      return set_err(RV_E_ARG, "push staging bound exceeded (%lld > %lld)", (long long)stride,
                     (long long)p->stride_bound);
    for (auto &lane : p->lanes) lane.stride = p->stride_bound;
  }
  // persistent grid: all lanes together fit in one wave (no lane can starve
  // another on this device while both wait on peers)
  int64_t capacity = (int64_t)p->sm_count * p->occ;
  if (p->max_blocks > 0) capacity = std::min<int64_t>(capacity, p->max_blocks);
  for (int l = 0; l < p->n_lanes; ++l) {
    rv_plan::Lane &lane = p->lanes[l];
    int64_t share = all_elems > 0 ? capacity * lane.elems / all_elems : 0;
    if (p->n_lanes == 1) share = capacity;
    share = std::max<int64_t>(1, std::min<int64_t>(share, std::max<int64_t>(1, lane.n_tiles)));
    lane.grid = (int)share;
  }
  p->dirty = false;
  return RV_OK;
}

int launch_lane(rv_plan *p, int l, cudaStream_t st) {
  rv_plan::Lane &lane = p->lanes[l];
  CycleParams cp;
  memset(&cp, 0, sizeof(cp));
  for (int i = 0; i < p->C; ++i) {
    cp.src[i] = p->src[i];
    cp.dst[i] = p->dst[i];
  }
  for (int r = 0; r < p->n_ranks && r < RV_MAX_RANKS; ++r) cp.peer_flags[r] = p->peer_flags[r];
  cp.segs = lane.segs;
  cp.tile_prefix = lane.prefix;
  cp.my_flags = p->flags;
  cp.state = p->states + l;
  cp.status = p->status;
  if (p->trace) {
    cp.trace = p->trace + 4 * l;
    RV_CUDA(cudaMemsetAsync(cp.trace, 0xff, sizeof(unsigned long long), st));
    RV_CUDA(cudaMemsetAsync(cp.trace + 1, 0, 3 * sizeof(unsigned long long), st));
  }
  cp.n_tiles = lane.n_tiles;
  cp.timeout_ns = p->timeout_ns;
  cp.C = p->C;
  cp.nseg = lane.nseg;
  cp.rank = p->rank;
  cp.n_ranks = p->n_ranks;
  cp.lane = l;
  cp.me = p->local.empty() ? 0 : p->local[0];
  cp.pow2 = (p->C & (p->C - 1)) == 0;
  cp.inv_c = 1.0 / (double)p->C;
  if (p->use_push) {
    for (int q = 0; q < p->C; ++q) {
      cp.pflags[q] = reinterpret_cast<unsigned long long *>(p->peer_push[q]);
      cp.stage[q] = p->peer_push[q] + p->pflag_bytes;
      cp.ounits[q] = lane.ounits[q];
    }
    for (int q = 0; q <= p->C; ++q) cp.oseg_base[q] = lane.oseg_base[q];
    cp.stride = lane.stride;
    cp.units_max = p->units_max;
    cp.scatter_umax = lane.scatter_umax;
    cp.unit_vecs = lane.unit_vecs;
  }
  if (lane.n_tiles == 0 && p->n_ranks == 1) return RV_OK;  // nothing to fold, nobody to meet
  const int grid = std::max(1, lane.grid);
  p->kernel<<<grid, p->block_threads, p->smem_bytes, st>>>(cp);
  RV_CUDA(cudaGetLastError());
  return RV_OK;
}

}  // namespace

extern "C" {

int rv_version(void) { return RV_ABI_VERSION; }

const char *rv_last_error(void) { return g_err.c_str(); }

const char *rv_status_string(int status) {
  switch (status) {
    case RV_OK: return "ok";
    case RV_E_CONFIG: return "config error";
    case RV_E_LAYOUT: return "layout error";
    case RV_E_CUDA: return "CUDA error";
    case RV_E_PEER_ACCESS: return "peer access unavailable";
    case RV_E_TIMEOUT: return "peer stall (timeout)";
    case RV_E_ARG: return "invalid argument";
    default: return "unknown status";
  }
}

int rv_plan_create(rv_plan **out, int device, int n_clusters, int n_rings, const int64_t *ring_start,
                   const int64_t *ring_len, int64_t total_params, int dtype, int acc_mode) {
  if (!out) return set_err(RV_E_ARG, "out is NULL");
  *out = nullptr;
  if (n_clusters < 2)  // multiring.py:268-269
    return set_err(RV_E_CONFIG, "all-reduce needs at least 2 clusters (got %d)", n_clusters);
  if (n_clusters > RV_MAX_CLUSTERS)
    return set_err(RV_E_CONFIG, "at most %d clusters supported (got %d)", RV_MAX_CLUSTERS, n_clusters);
  if (dtype != RV_DTYPE_F32 && dtype != RV_DTYPE_F64) return set_err(RV_E_CONFIG, "unknown dtype %d", dtype);
  if (acc_mode != RV_ACC_F64 && acc_mode != RV_ACC_NATIVE)
    return set_err(RV_E_CONFIG, "unknown accumulation mode %d", acc_mode);
  if (n_rings < 0 || total_params < 0 || (n_rings > 0 && (!ring_start || !ring_len)))
    return set_err(RV_E_ARG, "bad ring arrays");
  int64_t cursor = 0;  // multiring.py:110-116
  for (int r = 0; r < n_rings; ++r) {
    if (ring_start[r] != cursor || ring_len[r] < 0)
      return set_err(RV_E_LAYOUT, "rings do not tile the parameter space (ring %d)", r);
    cursor += ring_len[r];
  }
  if (cursor != total_params) return set_err(RV_E_LAYOUT, "rings do not cover all parameters");
  int ndev = 0;
  RV_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return set_err(RV_E_ARG, "device %d out of range (%d devices)", device, ndev);

  rv_plan *p = new rv_plan();
  p->device = device;
  p->C = n_clusters;
  p->R = n_rings;
  p->total = total_params;
  p->dtype = dtype;
  p->acc = dtype == RV_DTYPE_F64 ? RV_ACC_F64 : acc_mode;
  p->rstart.assign(ring_start, ring_start + n_rings);
  p->rlen.assign(ring_len, ring_len + n_rings);
  p->src.assign(n_clusters, nullptr);
  p->dst.assign(n_clusters, nullptr);
  p->bound.assign(n_clusters, 0);
  p->peer_flags.assign(RV_MAX_RANKS, nullptr);
  if (const char *t = getenv("RAVNEST_B200_TIMEOUT_S")) {
    const double s = atof(t);
    if (s > 0) p->timeout_ns = (unsigned long long)(s * 1e9);
  }
  {
    DeviceGuard g(device);
    cudaError_t e = cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, device);
    const int lanes_cap = std::max(1, n_rings);
    p->flag_bytes = sizeof(unsigned long long) * flag_index(lanes_cap, 0, 0);
    if (e == cudaSuccess) e = cudaMalloc(&p->flags, p->flag_bytes);
    if (e == cudaSuccess) e = cudaMemset(p->flags, 0, p->flag_bytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->states, sizeof(LaneState) * lanes_cap);
    if (e == cudaSuccess) e = cudaMemset(p->states, 0, sizeof(LaneState) * lanes_cap);
    if (e == cudaSuccess) e = cudaMalloc(&p->status, 4 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(p->status, 0, 4 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      rv_plan_destroy(p);
      return set_err(RV_E_CUDA, "plan allocation failed: %s", cudaGetErrorString(e));
    }
  }
  *out = p;
  return RV_OK;
}

int rv_plan_bind(rv_plan *p, int pos, const void *src, void *dst) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  if (pos < 0 || pos >= p->C) return set_err(RV_E_ARG, "position %d out of range", pos);
  if (!src || !dst) return set_err(RV_E_ARG, "NULL buffer for position %d", pos);
  p->src[pos] = src;
  p->dst[pos] = dst;
  p->bound[pos] = 1;
  p->ptrs_dirty = true;
  return RV_OK;
}

int rv_plan_set_local(rv_plan *p, const int *positions, int n) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  if (n < 0 || (n > 0 && !positions)) return set_err(RV_E_ARG, "bad positions");
  std::vector<char> seen(p->C, 0);
  for (int i = 0; i < n; ++i) {
    if (positions[i] < 0 || positions[i] >= p->C || seen[positions[i]])
      return set_err(RV_E_ARG, "bad or repeated position %d", positions[i]);
    seen[positions[i]] = 1;
  }
  p->local.assign(positions, positions + n);
  p->dirty = true;
  return RV_OK;
}

int rv_plan_set_lanes(rv_plan *p, int n_lanes) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  if (n_lanes < 1 || n_lanes > std::max(1, p->R))
    return set_err(RV_E_ARG, "lanes must be in [1, %d]", std::max(1, p->R));
  p->n_lanes = n_lanes;
  p->dirty = true;
  return RV_OK;
}

int rv_plan_flag_area(rv_plan *p, void **flags, size_t *bytes) {
  if (!p || !flags) return set_err(RV_E_ARG, "NULL argument");
  *flags = p->flags;
  if (bytes) *bytes = p->flag_bytes;
  return RV_OK;
}

int rv_plan_set_peers(rv_plan *p, int rank, int n_ranks, void *const *areas) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  if (n_ranks < 1 || n_ranks > RV_MAX_RANKS || rank < 0 || rank >= n_ranks)
    return set_err(RV_E_ARG, "bad rank %d of %d", rank, n_ranks);
  if (n_ranks > 1 && !areas) return set_err(RV_E_ARG, "peer flag areas missing");
  p->rank = rank;
  p->n_ranks = n_ranks;
  for (int r = 0; r < RV_MAX_RANKS; ++r)
    p->peer_flags[r] = (r < n_ranks && areas) ? static_cast<unsigned long long *>(areas[r]) : nullptr;
  for (int r = 0; r < n_ranks; ++r)
    if (r != rank && !p->peer_flags[r]) return set_err(RV_E_ARG, "flag area of rank %d missing", r);
  p->dirty = true;
  return RV_OK;
}

int rv_plan_set_protocol(rv_plan *p, int proto) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  if (proto != RV_PROTO_PULL && proto != RV_PROTO_PUSH) return set_err(RV_E_CONFIG, "unknown protocol %d", proto);
  p->proto = proto;
  p->dirty = true;
  return RV_OK;
}

int rv_plan_push_area(rv_plan *p, void **area, size_t *bytes) {
  if (!p || !area) return set_err(RV_E_ARG, "NULL argument");
  if (p->push_area && p->push_lanes != p->n_lanes) {
    DeviceGuard g(p->device);
    cudaFree(p->push_area);
    p->push_area = nullptr;
  }
  if (!p->push_area) {
    push_bounds(p, &p->stride_bound, &p->units_max);
    const size_t nflags = (size_t)std::max(1, p->n_lanes) * p->C * p->units_max;
    p->pflag_bytes = (nflags * sizeof(unsigned long long) + 4095) / 4096 * 4096;
    p->push_bytes = p->pflag_bytes + (size_t)p->C * p->stride_bound * elem_size(p->dtype);
    DeviceGuard g(p->device);
    RV_CUDA(cudaMalloc(&p->push_area, p->push_bytes));
    RV_CUDA(cudaMemset(p->push_area, 0, p->pflag_bytes));
    RV_CUDA(cudaDeviceSynchronize());
    p->push_lanes = p->n_lanes;
    p->dirty = true;
  }
  *area = p->push_area;
  if (bytes) *bytes = p->push_bytes;
  return RV_OK;
}

int rv_plan_set_push_peers(rv_plan *p, void *const *areas) {
  if (!p || !areas) return set_err(RV_E_ARG, "NULL argument");
  p->peer_push.assign(RV_MAX_RANKS, nullptr);
  for (int r = 0; r < p->n_ranks; ++r) p->peer_push[r] = static_cast<char *>(areas[r]);
  p->dirty = true;
  return RV_OK;
}

int rv_plan_set_trace(rv_plan *p, int enable) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  DeviceGuard g(p->device);
  if (enable && !p->trace) {
    const size_t n = 4 * (size_t)std::max(1, p->R);
    RV_CUDA(cudaMalloc(&p->trace, n * sizeof(unsigned long long)));
    RV_CUDA(cudaMemset(p->trace, 0, n * sizeof(unsigned long long)));
  } else if (!enable && p->trace) {
    cudaFree(p->trace);
    p->trace = nullptr;
  }
  return RV_OK;
}

int rv_plan_read_trace(rv_plan *p, int lane, uint64_t *out4) {
  if (!p || !out4) return set_err(RV_E_ARG, "NULL argument");
  if (!p->trace) return set_err(RV_E_ARG, "tracing is off");
  if (lane < 0 || lane >= std::max(1, p->R)) return set_err(RV_E_ARG, "bad lane %d", lane);
  DeviceGuard g(p->device);
  RV_CUDA(cudaDeviceSynchronize());
  RV_CUDA(cudaMemcpy(out4, p->trace + 4 * lane, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return RV_OK;
}

int rv_plan_set_max_blocks(rv_plan *p, int max_blocks) {
  if (!p || max_blocks < 0) return set_err(RV_E_ARG, "bad block budget");
  p->max_blocks = max_blocks;
  p->dirty = true;
  return RV_OK;
}

int rv_plan_set_timeout(rv_plan *p, double seconds) {
  if (!p || !(seconds > 0)) return set_err(RV_E_ARG, "bad timeout");
  p->timeout_ns = (unsigned long long)(seconds * 1e9);
  return RV_OK;
}

int rv_allreduce_mean(rv_plan *p, void *const *streams, int n_streams) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  DeviceGuard g(p->device);
  if (p->dirty || p->ptrs_dirty) {
    int rc = build_tables(p);
    if (rc) return rc;
  }
  for (int l = 0; l < p->n_lanes; ++l) {
    cudaStream_t st = (streams && n_streams > 0) ? (cudaStream_t)streams[l % n_streams] : (cudaStream_t)0;
    int rc = launch_lane(p, l, st);
    if (rc) return rc;
  }
  return RV_OK;
}

int rv_allreduce_mean_host(rv_plan *p, const void *const *host_src, void *const *host_dst,
                           void *const *streams, int n_streams) {
  if (!p || !host_src || !host_dst) return set_err(RV_E_ARG, "NULL argument");
  DeviceGuard g(p->device);
  if (p->dirty || p->ptrs_dirty) {
    int rc = build_tables(p);
    if (rc) return rc;
  }
  const int es = elem_size(p->dtype);
  // host->device copies run lane after lane (lane l's kernel starts as soon
  // as its own inputs have landed, while lane l+1's copy streams in and lane
  // l-1's result streams out): a three-stage H2D / average / D2H pipeline
  while ((int)p->h2d_done.size() < p->n_lanes) {
    cudaEvent_t e;
    RV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->h2d_done.push_back(e);
  }
  for (int l = 0; l < p->n_lanes; ++l) {
    cudaStream_t st = (streams && n_streams > 0) ? (cudaStream_t)streams[l % n_streams] : (cudaStream_t)0;
    const auto &rings = p->lanes[l].rings;
    if (l > 0) RV_CUDA(cudaStreamWaitEvent(st, p->h2d_done[l - 1], 0));
    for (size_t i = 0; i < p->local.size(); ++i) {
      const int pos = p->local[i];
      for (int r : rings) {
        if (p->rlen[r] == 0) continue;
        const size_t off = (size_t)p->rstart[r] * es, bytes = (size_t)p->rlen[r] * es;
        RV_CUDA(cudaMemcpyAsync((char *)p->src[pos] + off, (const char *)host_src[i] + off, bytes,
                                cudaMemcpyHostToDevice, st));
      }
    }
    RV_CUDA(cudaEventRecord(p->h2d_done[l], st));
    int rc = launch_lane(p, l, st);
    if (rc) return rc;
    for (size_t i = 0; i < p->local.size(); ++i) {
      const int pos = p->local[i];
      for (int r : rings) {
        if (p->rlen[r] == 0) continue;
        const size_t off = (size_t)p->rstart[r] * es, bytes = (size_t)p->rlen[r] * es;
        RV_CUDA(cudaMemcpyAsync((char *)host_dst[i] + off, (const char *)p->dst[pos] + off, bytes,
                                cudaMemcpyDeviceToHost, st));
      }
    }
  }
  return RV_OK;
}

int rv_plan_status(rv_plan *p, char *diag, size_t diag_len) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  DeviceGuard g(p->device);
  RV_CUDA(cudaDeviceSynchronize());
  unsigned st[4] = {0, 0, 0, 0};
  RV_CUDA(cudaMemcpy(st, p->status, sizeof(st), cudaMemcpyDeviceToHost));
  if (st[0] == 0) {
    if (diag && diag_len) snprintf(diag, diag_len, "no ring is stalled");
    return RV_OK;
  }
  const unsigned phase = st[1] >> 16, lane = (st[1] >> 8) & 0xff, peer = st[1] & 0xff;
  std::string rings;
  if (lane < p->lanes.size())
    for (int r : p->lanes[lane].rings) rings += (rings.empty() ? "" : "|") + std::to_string(r);
  const char *ph = phase == 0 ? "arrive" : phase == 1 ? "depart" : "unit";
  if (diag && diag_len)
    snprintf(diag, diag_len, "waiting on: (ring=%s, phase=%s, rank=%u)", rings.empty() ? "?" : rings.c_str(), ph,
             peer);
  return set_err(RV_E_TIMEOUT, "peer rank %u never reached the %s barrier (lane %u)", peer, ph, lane);
}

int rv_plan_reset_status(rv_plan *p) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  DeviceGuard g(p->device);
  RV_CUDA(cudaMemset(p->status, 0, 4 * sizeof(unsigned)));
  RV_CUDA(cudaDeviceSynchronize());
  return RV_OK;
}

int rv_plan_destroy(rv_plan *p) {
  if (!p) return RV_OK;
  {
    DeviceGuard g(p->device);
    free_lanes(p);
    if (p->push_area) cudaFree(p->push_area);
    if (p->trace) cudaFree(p->trace);
    for (cudaEvent_t e : p->h2d_done) cudaEventDestroy(e);
    if (p->flags) cudaFree(p->flags);
    if (p->states) cudaFree(p->states);
    if (p->status) cudaFree(p->status);
  }
  delete p;
  return RV_OK;
}

int rv_blend(int device, int dtype, void *live, const void *snap, const void *mean, int64_t n, void *stream) {
  if (n < 0 || (n > 0 && (!live || !snap || !mean))) return set_err(RV_E_ARG, "bad blend arguments");
  if (n == 0) return RV_OK;
  DeviceGuard g(device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaStream_t st = (cudaStream_t)stream;
  const bool aligned = ((uintptr_t)live % 16 == 0) && ((uintptr_t)snap % 16 == 0) && ((uintptr_t)mean % 16 == 0);
  const int es = elem_size(dtype);
  const int N = 16 / es;
  if (aligned && n >= N) {
    const int64_t nvec = n / N;
    const int grid = (int)std::min<int64_t>((nvec + kThreads - 1) / kThreads, (int64_t)sms * 8);
    if (dtype == RV_DTYPE_F64)
      blend_kernel_v4<double, unsigned long long><<<grid, kThreads, 0, st>>>(
          (double *)live, (const double *)snap, (const double *)mean, nvec);
    else
      blend_kernel_v4<float, unsigned><<<grid, kThreads, 0, st>>>((float *)live, (const float *)snap,
                                                                 (const float *)mean, nvec);
    RV_CUDA(cudaGetLastError());
    const int64_t done = nvec * N;
    if (done < n) {
      if (dtype == RV_DTYPE_F64)
        blend_kernel<double, unsigned long long><<<1, kThreads, 0, st>>>(
            (double *)live + done, (const double *)snap + done, (const double *)mean + done, n - done);
      else
        blend_kernel<float, unsigned><<<1, kThreads, 0, st>>>((float *)live + done, (const float *)snap + done,
                                                             (const float *)mean + done, n - done);
      RV_CUDA(cudaGetLastError());
    }
    return RV_OK;
  }
  const int grid = (int)std::min<int64_t>((n + kThreads - 1) / kThreads, (int64_t)sms * 8);
  if (dtype == RV_DTYPE_F64)
    blend_kernel<double, unsigned long long><<<grid, kThreads, 0, st>>>((double *)live, (const double *)snap,
                                                                       (const double *)mean, n);
  else
    blend_kernel<float, unsigned><<<grid, kThreads, 0, st>>>((float *)live, (const float *)snap,
                                                            (const float *)mean, n);
  RV_CUDA(cudaGetLastError());
  return RV_OK;
}

int rv_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int rv_ipc_export(const void *dev_ptr, void *handle_out, uint64_t *offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return set_err(RV_E_ARG, "NULL argument");
  cudaPointerAttributes attr;
  RV_CUDA(cudaPointerGetAttributes(&attr, dev_ptr));
  if (attr.type != cudaMemoryTypeDevice) return set_err(RV_E_ARG, "pointer %p is not device memory", dev_ptr);
  DeviceGuard g(attr.device);
  unsigned long long base = 0;
  int rc = alloc_base(dev_ptr, &base);
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  RV_CUDA(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (uint64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  return RV_OK;
}

int rv_ipc_import(int device, const void *handle, uint64_t offset, void **dev_ptr_out) {
  if (!handle || !dev_ptr_out) return set_err(RV_E_ARG, "NULL argument");
  DeviceGuard g(device);
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto key = std::make_pair(device, std::string((const char *)handle, sizeof(cudaIpcMemHandle_t)));
  auto it = g_ipc.find(key);
  void *base = nullptr;
  if (it != g_ipc.end()) {
    base = it->second.base;
    it->second.refs++;
  } else {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return set_err(RV_E_PEER_ACCESS, "cudaIpcOpenMemHandle failed: %s", cudaGetErrorString(e));
    g_ipc[key] = IpcEntry{base, 1};
  }
  *dev_ptr_out = (char *)base + offset;
  return RV_OK;
}

int rv_ipc_close(int device, void *dev_ptr) {
  DeviceGuard g(device);
  unsigned long long base = 0;
  int rc = alloc_base(dev_ptr, &base);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (auto it = g_ipc.begin(); it != g_ipc.end(); ++it) {
    if (it->first.first == device && it->second.base == (void *)(uintptr_t)base) {
      if (--it->second.refs == 0) {
        cudaIpcCloseMemHandle(it->second.base);
        g_ipc.erase(it);
      }
      return RV_OK;
    }
  }
  return set_err(RV_E_ARG, "pointer %p was not imported on device %d", dev_ptr, device);
}

int rv_enable_peer_access(int device, int peer) {
  if (device == peer) return RV_OK;
  int can = 0;
  RV_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return set_err(RV_E_PEER_ACCESS, "device %d cannot access device %d", device, peer);
  DeviceGuard g(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return RV_OK;
  }
  if (e != cudaSuccess)
    return set_err(RV_E_PEER_ACCESS, "cudaDeviceEnablePeerAccess(%d->%d): %s", device, peer, cudaGetErrorString(e));
  return RV_OK;
}

int rv_device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

}  // extern "C"
