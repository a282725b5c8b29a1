// Host error plumbing, device-side types (chunk tables, lane state, kernel
// parameters), PTX helpers and the cross-device flag barriers.
// Part of the single translation unit ravnest_b200.cu (included inside its
// anonymous namespace); see that file for the overview.
#pragma once

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
  unsigned int grab;            // push: work items handed out beyond the first one per block
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
  unsigned int *fail_host;     // host-mapped failure word (rv_plan_failed)
  unsigned long long *trace;   // optional: [start, ready, work done, departed] (globaltimer ns)
  int64_t n_tiles;             // pull
  int64_t stride;              // push: staging elements per writer slot
  int64_t units_max;           // push: unit-flag slots per (lane, writer)
  int64_t scatter_umax;        // push: max units over the other owners
  int64_t umax_all;            // push: max units over every owner (same on every rank)
  int push_dyn;                // push: blocks take work items from a counter (else stride by grid)
  void *live[RV_MAX_CLUSTERS]; // co-resident (TMA), fused blend: every member's live buffer
  void *live_me;               // push, fused blend: this rank's live buffer (else NULL)
  int64_t mflag_off;           // push, fused blend: mean-delivered flags, offset in a push area's flags
  int64_t blend_lag;           // push, fused blend: groups between a fold item and the blends of its unit
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

// Record a stall: the first failing thread sets the device status and its
// diagnostic, and raises the host-visible failure word.
__device__ __forceinline__ void fail(const CycleParams &p, unsigned diag) {
  if (atomicCAS(p.status, 0u, kStatusTimeout) == 0u) {
    p.status[1] = diag;
    if (p.fail_host) *(volatile unsigned *)p.fail_host = 1u;
  }
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
        fail(p, diag);
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

// Next work item of a block: the items go out in position order, each block
// taking a new one when it finishes its last (the first item of block b is
// b).  Uniform across the block.
__device__ __forceinline__ int64_t grab_next(const CycleParams &p, long long *s_next) {
  __syncthreads();
  if (threadIdx.x == 0) *s_next = (long long)gridDim.x + (long long)atomicAdd(&p.state->grab, 1u);
  __syncthreads();
  return *s_next;
}

// Exit barrier: the last block of this launch tells every peer that all of
// this device's stores (local and remote) are done, then waits for theirs,
// so nobody resumes training on a buffer a peer is still writing.
// With `cross` false (push with the fused blend, where every write into this
// rank's buffers is awaited item by item) only the lane bookkeeping remains.
__device__ void depart(const CycleParams &p, unsigned long long epoch, bool cross = true) {
  __syncthreads();
  if (threadIdx.x == 0) {
    trace_max(p, 2);
    __threadfence_system();
    const unsigned prev = atomicAdd(&p.state->done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      if (cross) {
        post_peers(p, 1, epoch);
        if (*(volatile unsigned *)p.status == 0) wait_peers(p, 1, epoch);
      }
      trace_max(p, 3);
      p.state->done = 0u;
      p.state->grab = 0u;
      *(volatile unsigned long long *)&p.state->epoch = epoch;
      __threadfence();
    }
  }
}
