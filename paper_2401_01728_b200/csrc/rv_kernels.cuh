// Kernels: pull/co-resident register path, push transport, co-resident TMA
// path, delayed-update blend.
// Part of the single translation unit ravnest_b200.cu (included inside its
// anonymous namespace); see that file for the overview.
#pragma once

// ---------------------------------------------------------------------------
// pull protocol: the owner of chunk k reads chunk k of every member (local
// HBM or NVLink peer loads) and pushes the mean into every member.  Arrive
// barrier first (peers' inputs final), depart barrier last.

// Segment of tile t for a thread whose tiles increase (t = blockIdx.x +
// i * gridDim.x): one binary search over tile_prefix for the first tile, then
// a forward walk, reloading the chunk record only when the segment changes
// (a binary search per tile cost 1% of HBM bandwidth on the TMA kernel,
// profiles/r01/ab_tma_segwalk_n1.txt).
struct SegWalk {
  int a = -1;
  int64_t next = 0, base = 0;  // tile_prefix[a + 1], tile_prefix[a]
  Seg cur;
  __device__ __forceinline__ const Seg &at(const CycleParams &p, int64_t t, int64_t *local) {
    if (a < 0) {
      int lo = 0, hi = p.nseg - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(p.tile_prefix + mid) <= t) lo = mid; else hi = mid - 1;
      }
      a = lo;
      base = __ldg(p.tile_prefix + a);
      next = __ldg(p.tile_prefix + a + 1);
      cur = p.segs[a];
    } else if (t >= next) {
      int b = a + 1;
      while (__ldg(p.tile_prefix + b + 1) <= t) ++b;
      a = b;
      base = __ldg(p.tile_prefix + a);
      next = __ldg(p.tile_prefix + a + 1);
      cur = p.segs[a];
    }
    *local = t - base;
    return cur;
  }
};

// Two 256-thread blocks per SM (<= 128 registers): measured 1.18 ms vs
// 1.47 ms at one block per SM on the co-resident BERT cycle.
template <typename T, typename Acc, int CB, int VB, int U>
__global__ void __launch_bounds__(kThreads, 2)
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
    SegWalk walk;
    for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
      int64_t local_tile;
      const Seg s = walk.at(p, t, &local_tile);
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
// owner q's staging slot and raises one release flag per unit (16-256 KB).
// Fold: for its own chunk, once every writer's flag for a unit is up, the
// owner folds its own values and the staged ones in ring order and pushes
// the mean into all members.  No arrive barrier is needed: a member's chunk
// reaches the owner only after its kernel started (inputs final), and the
// owner writes a member's buffer only after receiving that member's data for
// the same unit.  The depart barrier closes the cycle; with the fused blend
// the owner also raises a mean-delivered flag per unit on every member, each
// member awaits all of them (its blend items), and no depart barrier is
// needed.

template <typename T>
__device__ __forceinline__ Seg find_unit(const Seg *segs, int nseg, int64_t u) {
  int a = 0, b = nseg - 1;
  while (a < b) {
    const int mid = (a + b + 1) >> 1;
    if (segs[mid].unit0 <= u) a = mid; else b = mid - 1;
  }
  return segs[a];
}

// The fused blend's passes stream two operands per vector through shared
// memory with cp.async (LDGSTS): kBlendStages vectors per thread in flight
// and almost no registers, where a register loop kept one (a blend item is
// local HBM work and was latency-bound at one vector per thread).  Each
// thread reads back only the slots it filled itself, so waiting on its own
// cp.async groups is enough (no block barrier).
// live[j] <- f(a[j], live[j]) for vectors j in [jbeg, jend) of a chunk body
// (pointers already at the body start); ADD: f = a + live (second half, a =
// mean), else f = delta(live, a) (first half, a = snapshot).
template <typename T, int VB, bool ADD>
__device__ __forceinline__ void blend_stream(const T *a, T *live, int64_t jbeg, int64_t jend) {
  constexpr int N = VB / sizeof(T);
  using Raw = typename RawVec<VB>::type;
  extern __shared__ __align__(128) unsigned char smem[];  // kBlendSmem bytes (fused push launches only)
  Raw(*s_buf)[2][kThreads] = reinterpret_cast<Raw(*)[2][kThreads]>(smem);
  const int tid = threadIdx.x;
  const int64_t first = jbeg + tid;
  // prologue: stages 0 .. S-2
#pragma unroll
  for (int k = 0; k < kBlendStages - 1; ++k) {
    const int64_t j = first + (int64_t)k * kThreads;
    const bool ok = j < jend;
    cp_async<VB>(&s_buf[k][0][tid], a + (ok ? j : jbeg) * N, ok);
    cp_async<VB>(&s_buf[k][1][tid], live + (ok ? j : jbeg) * N, ok);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int st = 0;
  for (int64_t j = first; j < jend; j += kThreads) {
    // issue the vector S-1 iterations ahead into the stage freed last round
    const int64_t jn = j + (int64_t)(kBlendStages - 1) * kThreads;
    const int sn = st == 0 ? kBlendStages - 1 : st - 1;
    const bool ok = jn < jend;
    cp_async<VB>(&s_buf[sn][0][tid], a + (ok ? jn : jbeg) * N, ok);
    cp_async<VB>(&s_buf[sn][1][tid], live + (ok ? jn : jbeg) * N, ok);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kBlendStages - 1) : "memory");
    Lanes<T, VB> x, l;
    x.raw = s_buf[st][0][tid];
    l.raw = s_buf[st][1][tid];
#pragma unroll
    for (int e = 0; e < N; ++e) l.v[e] = ADD ? x.v[e] + l.v[e] : blend_delta<T>(l.v[e], x.v[e]);
    __stcs(reinterpret_cast<Raw *>(live + j * N), l.raw);
    st = st + 1 == kBlendStages ? 0 : st + 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Push with the fused blend: unit u of owner q, once q's mean-delivered flag
// for it is set: live <- mean + live over the unit's range of this rank's
// buffers, live holding delta(live, snap) since this rank's scatter item of
// the unit (blend_delta).  That write is ordered before the scatter flag's
// release, the owner's fold acquires it before releasing the mean-delivered
// flag this item acquires: causality carries it here.  False when the cycle
// failed (block must stop).
template <typename T, int VB>
__device__ bool blend_item(const CycleParams &p, int q, int64_t u, unsigned long long epoch, unsigned long long t0,
                           int *s_ok) {
  constexpr int N = VB / sizeof(T);
  using Raw = typename RawVec<VB>::type;
  const int C = p.C, me = p.me;
  if (u < 0 || u >= p.ounits[q]) return true;
  const Seg s = find_unit<T>(p.segs + p.oseg_base[q], p.oseg_base[q + 1] - p.oseg_base[q], u);
  if (threadIdx.x == 0) {
    const unsigned diag = (3u << 16) | ((unsigned)p.lane << 8) | (unsigned)q;
    if (!wait_flag(p, p.pflags[me] + p.mflag_off + pflag_index(p.lane, C, q, p.units_max, u), epoch, t0, diag))
      *s_ok = 0;
  }
  __syncthreads();
  if (!*s_ok) return false;
  const int64_t uu = u - s.unit0;
  const int64_t nvec = (s.body_hi - s.body_lo) / N;
  const int64_t jbeg = uu * p.unit_vecs, jend = min(nvec, jbeg + p.unit_vecs);
  const T *mean = static_cast<const T *>(p.dst[me]);
  T *live = static_cast<T *>(p.live_me);
  blend_stream<T, VB, true>(mean + s.body_lo, live + s.body_lo, jbeg, jend);
  if (uu == 0) {
    const int64_t nhead = s.body_lo - s.lo, ntail = s.hi - s.body_hi;
    if ((int64_t)threadIdx.x < nhead + ntail) {
      const int64_t i = (int64_t)threadIdx.x < nhead ? s.lo + threadIdx.x : s.body_hi + ((int64_t)threadIdx.x - nhead);
      live[i] = __ldcg(mean + i) + live[i];
    }
  }
  return true;
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
  // Work order (identical on every rank): every scatter item (unit-major),
  // then every fold item.  With the fused blend the folds come in groups of
  // C items: group g = fold unit g, then the blend items of unit
  // g - blend_lag of the C - 1 other owners (each waits for that owner's
  // mean-delivered flag, set by a fold item blend_lag groups earlier), so
  // the blend's HBM traffic runs under the NVLink traffic of later folds
  // and finds the means in L2.  Items wait only on items at earlier
  // positions (of other ranks), and blocks take items in position order,
  // so a co-resident grid always drains.
  const int64_t ua = p.umax_all;
  const bool fused = p.live_me != nullptr;
  const int64_t blag = p.blend_lag;
  const int64_t head = ua * (C - 1);
  const int64_t n_work = fused ? head + (ua + blag) * C : ua * C;
  const unsigned long long t0 = globaltimer();
  __shared__ long long s_next;

  for (int64_t w = blockIdx.x; w < n_work; w = p.push_dyn ? grab_next(p, &s_next) : w + gridDim.x) {
    if (!s_ok) break;
    int64_t sidx = -1, fidx = -1;  // scatter item (unit * (C-1) + peer) or fold unit
    if (w < head) {
      sidx = w;
    } else if (!fused) {
      fidx = w - head;
    } else if ((w - head) % C == 0) {
      fidx = (w - head) / C;
    } else {
      // blend item: unit u of owner q, from q's means in this rank's dst
      const int r = (int)((w - head) % C) - 1;
      const int64_t u = (w - head) / C - blag;
      if (!blend_item<T, VB>(p, me + 1 + r < C ? me + 1 + r : me + 1 + r - C, u, epoch, t0, &s_ok)) break;
      continue;
    }
    if (sidx >= 0) {
      const int r = (int)(sidx % (C - 1));
      const int64_t u = sidx / (C - 1);
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
          if (j < jend) v[c] = fused ? __ldcg(reinterpret_cast<const Raw *>(src + s.body_lo + j * N))
                                     : __ldcs(reinterpret_cast<const Raw *>(src + s.body_lo + j * N));
        }
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          const int64_t j = j0 + (int64_t)c * kThreads;
          if (j < jend) __stcs(reinterpret_cast<Raw *>(stg + s.body_lo + j * N), v[c]);
        }
      }
      if (fused) {
        // the blend's first half on this rank's copy of the unit (the
        // snapshot was just read: L2)
        T *live = static_cast<T *>(p.live_me);
        blend_stream<T, VB, false>(src + s.body_lo, live + s.body_lo, jbeg, jend);
      }
      if (uu == 0) {
        const int64_t nhead = s.body_lo - s.lo, ntail = s.hi - s.body_hi;
        if ((int64_t)threadIdx.x < nhead + ntail) {
          const int64_t i = (int64_t)threadIdx.x < nhead ? s.lo + threadIdx.x
                                                          : s.body_hi + ((int64_t)threadIdx.x - nhead);
          stg[i] = src[i];
          if (fused) {
            T *live = static_cast<T *>(p.live_me) + i;
            *live = blend_delta<T>(*live, src[i]);
          }
        }
      }
      __threadfence_system();  // this thread's stores, before the unit flag
      __syncthreads();
      if (threadIdx.x == 0)
        st_release_sys(p.pflags[q] + pflag_index(p.lane, C, me, p.units_max, u), epoch);
    } else {
      const int64_t u = fidx;
      if (u >= p.ounits[me]) continue;
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
      if (fused) {
        // the means of this unit are in every member's dst: tell them
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0)
          for (int m = 0; m < C; ++m)
            if (m != me) st_release_sys(p.pflags[m] + p.mflag_off + pflag_index(p.lane, C, me, p.units_max, u), epoch);
      }
      __syncthreads();  // s_ok is re-armed by thread 0 for the next unit
    }
  }
  depart(p, epoch, !fused);
}

// ---------------------------------------------------------------------------
// LL transport (small fp32 sets; one position per rank, rank == position):
// latency instead of bandwidth.  Every 16-byte store carries two fp32 values
// each paired with the cycle's epoch as a flag ({v0, e, v1, e}); readers poll
// the data itself, so there are no fences, no unit flags and no barriers:
//   scatter  member -> owner q's LL staging slot (chunk q of every ring)
//   fold     owner waits for every member's words, folds in ring order,
//            divides, writes its own buffer and LL words into every
//            member's receive area
//   receive  member waits for the owners' words and writes its buffer.
// All words a rank receives in a cycle are consumed inside that cycle's
// kernel, and a peer can only start cycle e+1 after it received this rank's
// cycle-e means, so the areas are reused without resets (epochs differ).
// Pays twice the bytes on NVLink (8 bytes per value); used below 4 MiB.

constexpr int64_t kLLUnit = 2 * kThreads;  // elements per LL work unit (one pair per thread)

__device__ __forceinline__ void ll_store(unsigned *addr, float v0, float v1, unsigned e) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "r"(__float_as_uint(v0)), "r"(e),
               "r"(__float_as_uint(v1)), "r"(e)
               : "memory");
}

// Spin until both flags of the LL word pair equal e; false on timeout.
__device__ __forceinline__ bool ll_load(const CycleParams &p, const unsigned *addr, unsigned e, float *v0, float *v1,
                                        unsigned diag) {
  unsigned a, b, c, d, spins = 0;
  unsigned long long t0 = 0;
  for (;;) {
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(addr)
                 : "memory");
    if (b == e && d == e) break;
    if ((++spins & 1023u) == 0) {
      if (t0 == 0) t0 = globaltimer();
      if (*(volatile unsigned *)p.status != 0) return false;
      if (globaltimer() - t0 > p.timeout_ns) {
        fail(p, diag);
        return false;
      }
    }
  }
  *v0 = __uint_as_float(a);
  *v1 = __uint_as_float(c);
  return true;
}

template <typename Acc, int CB>
__global__ void __launch_bounds__(kThreads, 2)
ring_ll_kernel(const __grid_constant__ CycleParams p) {
  __shared__ int s_ok;
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) {
    trace_min(p, 0);
    trace_max(p, 1);
    s_epoch = *(volatile unsigned long long *)&p.state->epoch + 1ull;
    s_ok = (*(volatile unsigned *)p.status == 0);
  }
  __syncthreads();
  const unsigned e = (unsigned)s_epoch;
  const int C = p.C, me = p.me;
  const float *src = static_cast<const float *>(p.src[me]);
  float *dst = static_cast<float *>(p.dst[me]);
  const int64_t n_side = (int64_t)(C - 1) * p.scatter_umax;
  const int64_t n_work = 2 * n_side + p.ounits[me];
  bool ok = s_ok;

  for (int64_t w = blockIdx.x; ok && w < n_work; w += gridDim.x) {
    if (w < n_side || w >= n_side + p.ounits[me]) {
      // scatter (first range) or receive (last range): unit u of owner q != me
      const bool scatter = w < n_side;
      const int64_t v = scatter ? w : w - n_side - p.ounits[me];
      const int r = (int)(v % (C - 1));
      const int64_t u = v / (C - 1);
      int q = me + 1 + r;
      if (q >= C) q -= C;
      if (u >= p.ounits[q]) continue;
      const Seg s = find_unit<float>(p.segs + p.oseg_base[q], p.oseg_base[q + 1] - p.oseg_base[q], u);
      const int64_t i0 = s.lo + (u - s.unit0) * kLLUnit + 2 * (int64_t)threadIdx.x;
      if (i0 >= s.hi || i0 >= s.lo + (u - s.unit0 + 1) * kLLUnit) continue;
      const bool two = i0 + 1 < s.hi;
      const int64_t word = s.stage_off + (i0 - s.lo);  // even
      if (scatter) {
        unsigned *stage = static_cast<unsigned *>(p.stage[q]);
        ll_store(stage + 2 * ((int64_t)me * p.stride + word), src[i0], two ? src[i0 + 1] : 0.f, e);
      } else {
        const unsigned *recv = static_cast<const unsigned *>(p.stage[me]) + 2 * (int64_t)C * p.stride;
        float v0, v1;
        const unsigned diag = (3u << 16) | ((unsigned)p.lane << 8) | (unsigned)q;
        if (!ll_load(p, recv + 2 * ((int64_t)q * p.stride + word), e, &v0, &v1, diag)) {
          ok = false;
          continue;
        }
        dst[i0] = v0;
        if (two) dst[i0 + 1] = v1;
      }
    } else {
      // fold: unit u of this rank's own chunk
      const int64_t u = w - n_side;
      const Seg s = find_unit<float>(p.segs + p.oseg_base[me], p.oseg_base[me + 1] - p.oseg_base[me], u);
      const int64_t i0 = s.lo + (u - s.unit0) * kLLUnit + 2 * (int64_t)threadIdx.x;
      if (i0 >= s.hi || i0 >= s.lo + (u - s.unit0 + 1) * kLLUnit) continue;
      const bool two = i0 + 1 < s.hi;
      const int64_t word = s.stage_off + (i0 - s.lo);
      const unsigned *stage = static_cast<const unsigned *>(p.stage[me]);
      Acc a0 = 0, a1 = 0;
      int m = s.k;  // == me: the fold starts at the owner
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        if (j < C) {
          float v0, v1;
          if (m == me) {
            v0 = src[i0];
            v1 = two ? src[i0 + 1] : 0.f;
          } else {
            const unsigned diag = (2u << 16) | ((unsigned)p.lane << 8) | (unsigned)m;
            if (!ll_load(p, stage + 2 * ((int64_t)m * p.stride + word), e, &v0, &v1, diag)) {
              ok = false;
              break;
            }
          }
          if (j == 0) {
            a0 = (Acc)v0;
            a1 = (Acc)v1;
          } else {
            a0 = a0 + (Acc)v0;
            a1 = a1 + (Acc)v1;
          }
          m = (m + 1 == C) ? 0 : m + 1;
        }
      }
      if (!ok) continue;
      const float m0 = finish<float, Acc>(a0, p), m1 = finish<float, Acc>(a1, p);
      dst[i0] = m0;
      if (two) dst[i0 + 1] = m1;
      for (int q = 0; q < C; ++q) {
        if (q == me) continue;
        unsigned *recv = static_cast<unsigned *>(p.stage[q]) + 2 * (int64_t)C * p.stride;
        ll_store(recv + 2 * ((int64_t)me * p.stride + word), m0, m1, e);
      }
    }
  }
  if (!ok && threadIdx.x == 0) s_ok = 0;
  // local bookkeeping only: the last block advances this lane's epoch
  __syncthreads();
  if (threadIdx.x == 0) {
    trace_max(p, 2);
    __threadfence();
    const unsigned prev = atomicAdd(&p.state->done, 1u);
    if (prev == gridDim.x - 1) {
      trace_max(p, 3);
      p.state->done = 0u;
      *(volatile unsigned long long *)&p.state->epoch = s_epoch;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// co-resident TMA path (all C members on this device, 16-byte congruent
// buffers): HBM-bound, so tiles stream through shared memory with bulk async
// copies.  Warp 0 / lane 0 produces: for each tile it loads the tile of all C
// members (cp.async.bulk global->shared, completion on a per-stage mbarrier)
// into a STAGES-deep ring.  The consumer warps (4; 8 with the fused blend)
// fold from shared memory in ring order, write the mean tile to shared
// memory, and one consumer issues C bulk stores (shared->global) of it, from
// rotating output buffers.  No register
// staging of loads, so each SM keeps STAGES * C * TV * 16 bytes in flight.

// Consumer threads per CTA (one producer warp besides).  The plain kernel
// folds with 4 consumer warps, the fused-blend kernel (twice the tiles per
// stage, C blends per vector) with 8.  Alternating A/B builds on one GPU
// (profiles/r02/ab_tma_consumers_n1.txt), BERT / ResNet-50 / GPT-2 config 4:
// 128 consumers 0.995-0.997 / 0.965-0.969 / 0.764, 256: 0.948-0.951 /
// 0.931-0.937 / 0.957-0.958, 384: 0.949-0.952 / 0.934-0.936 / 0.952-0.954,
// 512: 0.948 / 0.929-0.931 / 0.940-0.945 of measured HBM; for the blend
// kernel 192 / 256 / 320 measured alike (ab_tma_bl_consumers_n1.txt).
#ifndef RV_TMA_CONSUMERS  // A/B builds only override these
#define RV_TMA_CONSUMERS 128
#endif
#ifndef RV_TMA_BL_CONSUMERS
#define RV_TMA_BL_CONSUMERS 256
#endif
__host__ __device__ constexpr int tma_consumers(bool bl) { return bl ? RV_TMA_BL_CONSUMERS : RV_TMA_CONSUMERS; }

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

// Output buffers of the TMA kernel (bulk-store groups in flight): 3 for the
// plain kernel; the fused-blend kernel's output tiles are C + 1 times larger,
// so 2.  Three where shared memory allows (CB >= 8, RV_TMA_BL_NOB3 A/B
// builds) measured the same: GPT-2 / BERT C=8 config 4 0.955-0.958 vs
// 0.952-0.963 of HBM (profiles/r02/ab_tma_blend_nob_n1.txt).
__host__ __device__ constexpr int tma_out_buffers(bool bl, int cb) {
#ifdef RV_TMA_BL_NOB3
  return bl ? (cb >= 8 ? 3 : 2) : 3;
#else
  return bl ? 2 : 3;
#endif
}

// BL (fused delayed-update blend): each stage also carries every member's
// live tile; the consumers write the mean tile and C blended live tiles,
// which go out by bulk store to dst and live.
template <typename T, typename Acc, int CB, int TV, int STAGES, bool BL = false>
__global__ void __launch_bounds__(tma_consumers(BL) + 32, tma_consumers(BL) > 256 ? 1 : 2)
ring_tma_kernel(const __grid_constant__ CycleParams p) {
  constexpr int N = 16 / sizeof(T);
  constexpr int SLOTS = BL ? 2 * CB : CB;  // tiles per stage: src (ring order), then live
  constexpr int OUTS = BL ? CB + 1 : 1;    // output tiles: mean, then blended live
  constexpr int NOB = tma_out_buffers(BL, CB);  // output buffers (bulk-store groups in flight)
  constexpr int NC = tma_consumers(BL);          // consumer threads
  extern __shared__ __align__(128) unsigned char smem[];
  uint4 *in = reinterpret_cast<uint4 *>(smem);                       // [STAGES][SLOTS][TV]
  uint4 *out = in + (size_t)STAGES * SLOTS * TV;                       // [NOB][OUTS][TV]
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

  // the tiles this block owns increase (t = blockIdx.x + i * gridDim.x), so
  // each thread walks the segment table forward (SegWalk)
  SegWalk walk;
  auto seg_of = [&](int64_t t, int64_t *local) -> const Seg & { return walk.at(p, t, local); };
  // tiles dealt round-robin (one contiguous run per block measured slower:
  // 0.940 vs 0.947 of HBM, profiles/r02/ab_tma_layouts_n1.txt)
  const int64_t TILE_FIRST = blockIdx.x, TILE_END = p.n_tiles, TILE_STEP = gridDim.x;

  if (tid < 32) {
    if (tid == 0) {  // producer
      int stage = 0;
      unsigned phase = 0;
      int64_t n = 0;
      for (int64_t t = TILE_FIRST; t < TILE_END; t += TILE_STEP, ++n) {
        int64_t lt;
        const Seg s = seg_of(t, &lt);
        const int64_t nvec = (s.body_hi - s.body_lo) / N;
        const int64_t j0 = lt * TV;
        const int cnt = (int)max((int64_t)0, min((int64_t)TV, nvec - j0));
        if (n >= STAGES) mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], (unsigned)(cnt * 16 * C * (BL ? 2 : 1)));
        if (cnt > 0) {
          for (int q = 0; q < C; ++q) {
            int m = s.k + q;
            if (m >= C) m -= C;
            bulk_load(in + ((size_t)stage * SLOTS + q) * TV, static_cast<const T *>(p.src[m]) + s.body_lo + j0 * N,
                      (unsigned)(cnt * 16), &full[stage]);
            if constexpr (BL)
              bulk_load(in + ((size_t)stage * SLOTS + CB + q) * TV,
                        static_cast<const T *>(p.live[m]) + s.body_lo + j0 * N, (unsigned)(cnt * 16), &full[stage]);
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

  // consumers (NC threads)
  const int c = tid - 32;
  int stage = 0;
  unsigned phase = 0;
  int ob = 0;
  for (int64_t t = TILE_FIRST; t < TILE_END; t += TILE_STEP) {
    int64_t lt;
    const Seg s = seg_of(t, &lt);
    const int64_t nvec = (s.body_hi - s.body_lo) / N;
    const int64_t j0 = lt * TV;
    const int cnt = (int)max((int64_t)0, min((int64_t)TV, nvec - j0));
    mbar_wait(&full[stage], phase);
    // consumer 0 finished the previous tile's store bookkeeping (out[ob] free)
    asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
    for (int v = c; v < cnt; v += NC) {
      Lanes<T, 16> x, o;
      Acc acc[N];
      x.raw = in[((size_t)stage * SLOTS + 0) * TV + v];
#pragma unroll
      for (int e = 0; e < N; ++e) acc[e] = (Acc)x.v[e];
#pragma unroll
      for (int q = 1; q < CB; ++q) {
        if (q < C) {
          x.raw = in[((size_t)stage * SLOTS + q) * TV + v];
#pragma unroll
          for (int e = 0; e < N; ++e) acc[e] = acc[e] + (Acc)x.v[e];
        }
      }
#pragma unroll
      for (int e = 0; e < N; ++e) o.v[e] = finish<T, Acc>(acc[e], p);
      out[(size_t)ob * OUTS * TV + v] = o.raw;
      if constexpr (BL) {
#pragma unroll
        for (int q = 0; q < CB; ++q) {
          if (q < C) {
            Lanes<T, 16> sn, l;
            sn.raw = in[((size_t)stage * SLOTS + q) * TV + v];
            l.raw = in[((size_t)stage * SLOTS + CB + q) * TV + v];
#pragma unroll
            for (int e = 0; e < N; ++e) l.v[e] = blend_one<T>(o.v[e], l.v[e], sn.v[e]);
            out[((size_t)ob * OUTS + 1 + q) * TV + v] = l.raw;
          }
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
    if (c == 0) {
      mbar_arrive(&empty[stage]);  // every consumer has read this stage
      if (cnt > 0) {
        const uint4 *mean_tile = out + (size_t)ob * OUTS * TV;
        for (int q = 0; q < C; ++q)
          bulk_store(static_cast<T *>(p.dst[q]) + s.body_lo + j0 * N, mean_tile, (unsigned)(cnt * 16));
        if constexpr (BL)
          for (int q = 0; q < C; ++q) {
            int m = s.k + q;
            if (m >= C) m -= C;
            bulk_store(static_cast<T *>(p.live[m]) + s.body_lo + j0 * N, mean_tile + (size_t)(1 + q) * TV,
                       (unsigned)(cnt * 16));
          }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      // the buffer the next tile writes is free once at most NOB - 1 groups
      // are still reading shared memory
      if constexpr (NOB == 3)
        asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
      else
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    if (lt == 0) {
      const int64_t nhead = s.body_lo - s.lo, ntail = s.hi - s.body_hi;
      if ((int64_t)c < nhead + ntail) {
        const int64_t i = (int64_t)c < nhead ? s.lo + c : s.body_hi + ((int64_t)c - nhead);
        fold_scalar<T, Acc, false>(p, s, i);
        if constexpr (BL)
          for (int m = 0; m < C; ++m) {
            T *l = static_cast<T *>(p.live[m]) + i;
            *l = blend_one<T>(static_cast<const T *>(p.dst[m])[i], *l, static_cast<const T *>(p.src[m])[i]);
          }
      }
    }
    if (++ob == NOB) ob = 0;
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
