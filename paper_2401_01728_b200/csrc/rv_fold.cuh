// The ring-order fold: vector types, the IEEE divide by C, member addressing
// for the pull and push transports, scalar and vector fold passes.
// Part of the single translation unit ravnest_b200.cu (included inside its
// anonymous namespace); see that file for the overview.
#pragma once

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

// Fused push blend: its passes stream operands through shared memory with
// cp.async (see blend_stream, rv_kernels.cuh); the fold also prefetches the
// owner's live vectors this way.
constexpr int kBlendStages = 4;
constexpr int kBlendSmem = kBlendStages * 2 * 256 * 16;  // dynamic shared memory of a fused push launch

template <int VB>
__device__ __forceinline__ void cp_async(void *smem, const void *gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? VB : 0;  // src-size 0: no global read, nothing to wait for
  if constexpr (VB == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(sa), "l"(gmem), "n"(VB), "r"(n)
                 : "memory");
}

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

// Delayed-update blend of one value, live <- mean + (live - snap), two
// roundings in the storage type; where live and snap are the same bits the
// result is mean itself (oracle/ring_oracle.blend, blend_kernel).
template <typename T>
__device__ __forceinline__ T blend_one(T mean, T live, T snap) {
  using U = typename std::conditional<sizeof(T) == 8, unsigned long long, unsigned>::type;
  U lb, sb;
  memcpy(&lb, &live, sizeof(T));
  memcpy(&sb, &snap, sizeof(T));
  return lb == sb ? mean : mean + (live - snap);
}

// The push transport's fused blend of another owner's chunk runs in two
// halves: the scatter item that sends this rank's copy of the chunk also
// turns live into delta(live, snap) (it has the snapshot in hand, and HBM is
// mostly idle while NVLink carries the scatter), and once the owner's means
// land the blend item finishes live <- mean + live.  delta() stores -0.0
// where live and snap are the same bits, and mean + (-0.0) == mean for every
// mean (RN mode, -0.0 included), so the halves are bit for bit
// blend_one(mean, live, snap): one IEEE subtract and one IEEE add.
template <typename T>
__device__ __forceinline__ T blend_delta(T live, T snap) {
  using U = typename std::conditional<sizeof(T) == 8, unsigned long long, unsigned>::type;
  U lb, sb;
  memcpy(&lb, &live, sizeof(T));
  memcpy(&sb, &snap, sizeof(T));
  return lb == sb ? (T)-0.0 : live - snap;
}

// Fold of one element (chunk edges, misaligned buffers): ring order from s.k.
// Push with the fused blend: the owner (s.k == me) also blends its own live
// value, its snapshot being the first member folded.
template <typename T, typename Acc, bool PUSH>
__device__ __forceinline__ void fold_scalar(const CycleParams &p, const Seg &s, int64_t i) {
  int m = s.k;
  const T first = __ldcs(member_elem<T, PUSH>(p, s, m, i));
  Acc acc = (Acc)first;
  for (int q = 1; q < p.C; ++q) {
    m = (m + 1 == p.C) ? 0 : m + 1;
    acc = acc + (Acc)__ldcs(member_elem<T, PUSH>(p, s, m, i));
  }
  const T out = finish<T, Acc>(acc, p);
  for (int q = 0; q < p.C; ++q) __stcs(static_cast<T *>(p.dst[q]) + i, out);
  if (PUSH && p.live_me) {
    T *live = static_cast<T *>(p.live_me) + i;
    *live = blend_one<T>(out, *live, first);
  }
}

// Fold one pass of chunk s: this thread takes vectors j0 + u*kThreads
// (u < U, below jend), loads all C members of each (U*C loads in flight),
// folds in ring order, divides, and stores the mean into all C buffers.
template <typename T, typename Acc, int CB, int VB, int U, bool PUSH>
__device__ __forceinline__ void fold_pass(const CycleParams &p, const Seg &s, int64_t j0, int64_t jend) {
  constexpr int N = VB / sizeof(T);
  using Raw = typename RawVec<VB>::type;
  static_assert(U * 16 * 256 <= kBlendSmem, "live prefetch slots exceed the fused launch's shared memory");
  Lanes<T, VB> x[U][CB];
  extern __shared__ __align__(128) unsigned char smem[];  // fused push launches only (kBlendSmem)
  Raw *lbuf = reinterpret_cast<Raw *>(smem);               // [U][kThreads]: this thread's live prefetch
  // (not for fp64 storage at CB >= 8, whose address registers would spill)
  constexpr bool kPrefetch = PUSH && (sizeof(T) == 4 || CB <= 4);
  if (kPrefetch && p.live_me) {
    // the fused blend of the owner's own copy needs its live vectors after
    // the fold: fetch them now, alongside the members, without registers
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + (int64_t)u * kThreads;
      const bool ok = j < jend;
      cp_async<VB>(&lbuf[u * kThreads + threadIdx.x],
                   static_cast<const T *>(p.live_me) + s.body_lo + (ok ? j : j0) * N, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
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
      if (PUSH && p.live_me) {  // fused blend of the owner's own copy (x[u][0] is its snapshot)
        Lanes<T, VB> l;
        if constexpr (kPrefetch) {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
          l.raw = lbuf[u * kThreads + threadIdx.x];
        } else {
          l.raw = *reinterpret_cast<const Raw *>(static_cast<const T *>(p.live_me) + i);
        }
#pragma unroll
        for (int e = 0; e < N; ++e) l.v[e] = blend_one<T>(out.v[e], l.v[e], x[u][0].v[e]);
        __stcs(reinterpret_cast<Raw *>(static_cast<T *>(p.live_me) + i), l.raw);
      }
    }
  }
}
