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
#include <type_traits>
#include <vector>

#include "../../include/ravnest_b200.h"

namespace {

#include "rv_common.cuh"
#include "rv_fold.cuh"
#include "rv_kernels.cuh"
#include "rv_dispatch.cuh"

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
  std::vector<void *> live;  // delayed-update blend targets (rv_plan_bind_live), NULL = none
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
    int64_t lo = 0, hi = 0;  // element range of this lane
    std::vector<int> rings;  // rings meeting the range
    int grid = 0;
    // push
    int64_t stride = 0, unit_vecs = 0, scatter_umax = 0, umax_all = 0, blend_lag = 0;
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
  // rv_plan_set_option (RV_OPT_*)
  int min_cb = 0;             // member-count bucket floor
  int use_tma = 1;            // co-resident TMA kernel when eligible
  int64_t push_items = 2;     // push: work items per resident block (sizes the units)
  int push_dyn = 1;           // push: work items from a counter (else static grid stride)
  int64_t blend_lag_opt = -1; // push fused blend: lag in groups of C items (-1: two resident grids)
  int layout_sms = 0;         // push: SM count the unit layout assumes (0: this device's)
  unsigned *fail_host = nullptr;  // host-mapped failure word (rv_plan_failed)
  unsigned *fail_dev = nullptr;   // its device alias
  bool blend = false;        // live bound on the local positions: every cycle ends with the blend
  bool fused_blend = false;  // ... inside the push kernel (else blend launches after each lane)
  int64_t mflag_off = 0;     // push: mean-delivered flags after the scatter flags (u64 index)
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

bool push_active(const rv_plan *p) {
  return (p->proto == RV_PROTO_PUSH || p->proto == RV_PROTO_LL) && p->n_ranks > 1;
}
bool ll_active(const rv_plan *p) { return p->proto == RV_PROTO_LL && p->n_ranks > 1; }

// Lane l is the element range [first, second) of the parameter vector that
// one launch (on its own stream) averages.  n_lanes <= R: consecutive whole
// rings per lane (n_lanes == R is one ring per lane); n_lanes > R: every ring
// is cut into equal pieces, more pieces for longer rings.
std::vector<std::pair<int64_t, int64_t>> lane_ranges(const rv_plan *p) {
  const int L = p->n_lanes, R = p->R;
  std::vector<std::pair<int64_t, int64_t>> out;
  if (R == 0) {
    out.assign(L, {0, 0});
    return out;
  }
  if (L <= R) {
    for (int l = 0; l < L; ++l) {
      const int r0 = (int)((int64_t)l * R / L), r1 = (int)((int64_t)(l + 1) * R / L);
      out.push_back({p->rstart[r0], p->rstart[r1 - 1] + p->rlen[r1 - 1]});
    }
    return out;
  }
  std::vector<int> pieces(R, 1);
  int left = L - R;
  const int64_t total = std::max<int64_t>(1, p->total);
  for (int r = 0; r < R && left > 0; ++r) {
    const int extra = (int)std::min<int64_t>(left, (int64_t)(L - R) * p->rlen[r] / total);
    pieces[r] += extra;
    left -= extra;
  }
  for (int r = 0; left > 0; r = (r + 1) % R, --left) pieces[r] += 1;
  for (int r = 0; r < R; ++r)
    for (int k = 0; k < pieces[r]; ++k)
      out.push_back({p->rstart[r] + p->rlen[r] * k / pieces[r], p->rstart[r] + p->rlen[r] * (k + 1) / pieces[r]});
  return out;
}

// chunk k of ring r clipped to a lane; empty when they do not meet
std::pair<int64_t, int64_t> clip(std::pair<int64_t, int64_t> chunk, std::pair<int64_t, int64_t> lane) {
  const int64_t lo = std::max(chunk.first, lane.first), hi = std::min(chunk.second, lane.second);
  return {lo, std::max(lo, hi)};
}

// Upper bounds of the push layout, from the schedule alone (before any
// pointer is known): staging elements per writer slot, unit flags per lane.
void push_bounds(const rv_plan *p, int64_t *stride_bound, int64_t *units_max) {
  const int es = elem_size(p->dtype);
  const bool ll = p->proto == RV_PROTO_LL;
  const int64_t nmax = ll ? 2 : 16 / es, unit_elems = ll ? kLLUnit : kMinUnitBytes / es;
  const auto lanes = lane_ranges(p);
  int64_t stride = nmax;
  int64_t umax = 1;
  for (const auto &ln : lanes) {
    int64_t u = 0;
    for (int r = 0; r < p->R; ++r) {
      const int64_t meet = clip({p->rstart[r], p->rstart[r] + p->rlen[r]}, ln).second -
                           clip({p->rstart[r], p->rstart[r] + p->rlen[r]}, ln).first;
      if (meet <= 0) continue;
      const int64_t piece = std::min(meet, (p->rlen[r] + p->C - 1) / p->C);
      u += (piece + unit_elems - 1) / unit_elems + 1;
      stride += piece + 2 * nmax;  // one piece per owner per (ring, lane), padded for alignment
    }
    umax = std::max(umax, u);
  }
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

// lanes (launches / streams per cycle) a plan can hold beyond one per ring
constexpr int kMaxLanes = 64;

int build_tables(rv_plan *p) {
  for (int i = 0; i < p->C; ++i)
    if (!p->bound[i]) return set_err(RV_E_ARG, "cluster position %d is not bound", i);
  if (p->local.empty()) return set_err(RV_E_ARG, "no local positions set");
  const int es = elem_size(p->dtype);
  // vector path needs every member buffer congruent modulo 16 bytes
  const uintptr_t a = (uintptr_t)p->src[0] % 16;
  bool vec = true;
  for (int i = 0; i < p->C; ++i) {
    if ((uintptr_t)p->src[i] % es || (uintptr_t)p->dst[i] % es || (uintptr_t)p->live[i] % es)
      return set_err(RV_E_ARG, "buffer of position %d is not %d-byte aligned", i, es);
    if ((uintptr_t)p->src[i] % 16 != a || (uintptr_t)p->dst[i] % 16 != a) vec = false;
    if (p->live[i] && (uintptr_t)p->live[i] % 16 != a) vec = false;
  }
  // delayed-update blend: all local positions or none; the means need their
  // own buffer (the blend reads the snapshot = src after the means landed)
  int n_live = 0;
  for (int pos : p->local) n_live += p->live[pos] != nullptr;
  if (n_live != 0 && n_live != (int)p->local.size())
    return set_err(RV_E_ARG, "live buffers bound on %d of %d local positions", n_live, (int)p->local.size());
  p->blend = n_live > 0;
  if (p->blend) {
    // every snapshot, mean and live vector its own buffer (start addresses)
    std::vector<std::pair<uintptr_t, int>> starts;
    for (int i = 0; i < p->C; ++i) {
      starts.push_back({(uintptr_t)p->src[i], i});
      starts.push_back({(uintptr_t)p->dst[i], i});
      if (p->live[i]) starts.push_back({(uintptr_t)p->live[i], i});
    }
    std::sort(starts.begin(), starts.end());
    for (size_t j = 1; j < starts.size(); ++j)
      if (starts[j].first == starts[j - 1].first)
        return set_err(RV_E_ARG, "blend needs distinct snapshot, mean and live buffers (positions %d and %d share one)",
                       starts[j - 1].second, starts[j].second);
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
  p->fused_blend = p->blend && push && p->proto == RV_PROTO_PUSH;  // co-resident TMA: set below
  const bool ll = ll_active(p);
  if (ll && p->dtype != RV_DTYPE_F32) return set_err(RV_E_CONFIG, "the LL transport carries fp32 parameters only");
  const int mode = p->dtype == RV_DTYPE_F64 ? kF64 : (p->acc == RV_ACC_NATIVE ? kF32Native : kF32Acc64);
  int U = 1;
  int64_t tile_vecs = 0;
  DeviceGuard g(p->device);
  const bool tma = vec && p->n_ranks == 1 && p->use_tma;
  const int cb = bucket_c(p->C, p->min_cb);
  if (ll) {
    p->kernel = pick_ll_kernel(mode, cb);
    p->block_threads = kThreads;
    p->smem_bytes = 0;
    tile_vecs = kLLUnit;
  } else if (tma) {
    int tv = 0;
    p->fused_blend = p->blend;
    p->kernel = pick_tma_kernel(mode, cb, p->blend, &tv, &p->smem_bytes);
    p->block_threads = tma_consumers(p->blend) + 32;
    RV_CUDA(cudaFuncSetAttribute(p->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->smem_bytes));
    tile_vecs = tv;
  } else {
    p->kernel = pick_kernel(mode, cb, vec, push, &U);
    p->block_threads = kThreads;
    // the fused push blend streams its operands through shared memory
    p->smem_bytes = p->fused_blend ? (size_t)kBlendSmem : 0;
    tile_vecs = (int64_t)kThreads * U;
  }
  RV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->occ, p->kernel, p->block_threads, p->smem_bytes));
  if (p->occ < 1) p->occ = 1;
  // push: unit size adapts so that a cycle has >= ~2 work items per resident
  // block (small shards stay parallel, large ones amortise the unit flags);
  // it depends only on the schedule and the device model, so every rank
  // derives the same layout
  int64_t unit_vecs = kUnitBytes / (N * es);
  if (push && !ll) {
    int64_t owner_elems = 0;
    for (int q = 0; q < p->C; ++q) {
      int64_t e = 0;
      for (int r = 0; r < p->R; ++r) {
        const auto b = ring_chunks(p, r);
        e += b[q].second - b[q].first;
      }
      owner_elems = std::max(owner_elems, e);
    }
    // target work items (scatter + fold units) per resident block: more
    // shrink the tail when blocks finish unevenly, fewer amortise the flags
    const int64_t sms = p->layout_sms > 0 ? p->layout_sms : p->sm_count;
    const int64_t items = std::max<int64_t>(1, p->push_items * sms * p->occ);
    const int64_t want = (owner_elems / N * (p->C - 1) + items - 1) / items;
    const int64_t lo = kMinUnitBytes / (N * es), hi = kUnitBytes / (N * es);
    unit_vecs = std::min(hi, std::max(lo, (want + kThreads - 1) / kThreads * kThreads));
  }

  free_lanes(p);
  p->lanes.resize(p->n_lanes);
  const auto ranges = lane_ranges(p);
  std::vector<int> loc = p->local;
  std::sort(loc.begin(), loc.end());
  std::vector<int64_t> cursor(p->C, 0);  // push: staging cursor per owner, across lanes
  int64_t all_elems = 0;
  for (int l = 0; l < p->n_lanes; ++l) {
    rv_plan::Lane &lane = p->lanes[l];
    std::vector<Seg> segs;
    std::vector<int64_t> prefix(1, 0);
    lane.lo = ranges[l].first;
    lane.hi = ranges[l].second;
    for (int r = 0; r < p->R; ++r) {
      const auto m = clip({p->rstart[r], p->rstart[r] + p->rlen[r]}, ranges[l]);
      if (m.second > m.first) lane.rings.push_back(r);
    }
    if (!push) {
      for (int r : lane.rings) {
        const auto bounds = ring_chunks(p, r);
        for (int k : loc) {
          Seg s{};
          const auto piece = clip(bounds[k], ranges[l]);
          s.lo = piece.first;
          s.hi = piece.second;
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
          const auto piece = clip(bounds[q], ranges[l]);
          s.lo = piece.first;
          s.hi = piece.second;
          s.k = q;
          s.ring = r;
          if (s.hi <= s.lo) continue;
          set_body(s, N, a0);
          s.unit0 = u;
          if (ll) {
            // LL words pair up elements: even offsets keep each pair in one
            // 16-byte {v0, e, v1, e} store
            s.stage_off = (cursor[q] + 1) / 2 * 2;
            cursor[q] = s.stage_off + (s.hi - s.lo);
            u += (s.hi - s.lo + kLLUnit - 1) / kLLUnit;
          } else {
            // staging index of element i is stage_off + (i - lo); keep it
            // vector-aligned exactly where the source is
            const int64_t c0 = (cursor[q] + N - 1) / N * N;
            s.stage_off = c0 + ((s.lo + a0) % N);
            cursor[q] = s.stage_off + (s.hi - s.lo);
            const int64_t nvec = (s.body_hi - s.body_lo) / N;
            u += std::max<int64_t>(1, (nvec + unit_vecs - 1) / unit_vecs);
          }
          segs.push_back(s);
          // a push / LL rank scatters every other owner's piece of the lane
          // and folds its own: its work is the whole lane, not its own chunk
          // (sizing by the own chunk gave a lane holding another owner's
          // chunk a single block, 36-73 GB/s at lanes > rings)
          lane.elems += s.hi - s.lo;
        }
        lane.ounits[q] = u;
        if (u > p->units_max) return set_err(RV_E_ARG, "push unit bound exceeded (%lld > %lld)",
                                             (long long)u, (long long)p->units_max);
      }
      lane.oseg_base[p->C] = (int)segs.size();
      lane.unit_vecs = unit_vecs;
      lane.scatter_umax = 0;
      lane.umax_all = 0;
      for (int q = 0; q < p->C; ++q) {
        if (q != p->rank) lane.scatter_umax = std::max(lane.scatter_umax, lane.ounits[q]);
        lane.umax_all = std::max(lane.umax_all, lane.ounits[q]);
      }
      // fused blend: a unit's blends trail its fold by about two resident
      // grids of items (RV_OPT_BLEND_LAG: groups of C items; GPT-2 at 4
      // GPUs, 1 / 2 / 4 / 8 / 16 grids: 3.53 / 3.22 / 3.28 / 3.47 / 3.77 ms
      // per cycle + blend).  Every rank must use the same lag.
      lane.blend_lag = p->blend_lag_opt >= 0 ? p->blend_lag_opt
                                             : (2 * (int64_t)p->sm_count * p->occ + p->C - 1) / p->C;
      lane.n_tiles = ll ? (int64_t)(p->C - 1) * lane.scatter_umax * 2 + lane.ounits[p->rank]
                        : (int64_t)(p->fused_blend ? 2 * p->C - 1 : p->C) * lane.umax_all;
      lane.nseg = (int)segs.size();
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
  // Multi-rank lanes spin on their peers, so all lanes of a cycle must be
  // resident together: the budget is split in proportion to lane bytes.  A
  // co-resident plan (no peers) has no such constraint, and its lanes often
  // run one after another (the host-buffer pipeline staggers them behind
  // their copies), so every lane gets the whole budget.
  std::vector<int64_t> share(p->n_lanes);
  int64_t granted = 0;
  for (int l = 0; l < p->n_lanes; ++l) {
    const rv_plan::Lane &lane = p->lanes[l];
    int64_t sh = all_elems > 0 ? capacity * lane.elems / all_elems : 0;
    if (p->n_lanes == 1 || p->n_ranks == 1) sh = capacity;
    share[l] = std::max<int64_t>(1, std::min<int64_t>(sh, std::max<int64_t>(1, lane.n_tiles)));
    granted += share[l];
  }
  // the one-block floor of small lanes must not push the sum past the
  // budget (lanes spin on peers: every block of every lane must be resident)
  while (p->n_ranks > 1 && granted > capacity) {
    int big = 0;
    for (int l = 1; l < p->n_lanes; ++l)
      if (share[l] > share[big]) big = l;
    if (share[big] <= 1) break;  // more lanes than blocks: cannot fit, keep one each
    --share[big];
    --granted;
  }
  for (int l = 0; l < p->n_lanes; ++l) p->lanes[l].grid = (int)share[l];
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
    cp.live[i] = p->live[i];
  }
  for (int r = 0; r < p->n_ranks && r < RV_MAX_RANKS; ++r) cp.peer_flags[r] = p->peer_flags[r];
  cp.segs = lane.segs;
  cp.tile_prefix = lane.prefix;
  cp.my_flags = p->flags;
  cp.state = p->states + l;
  cp.status = p->status;
  cp.fail_host = p->fail_dev;
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
    cp.umax_all = lane.umax_all;
    cp.push_dyn = p->push_dyn;
    cp.live_me = p->fused_blend ? p->live[p->rank] : nullptr;
    cp.mflag_off = p->mflag_off;
    cp.blend_lag = lane.blend_lag;
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
  p->live.assign(n_clusters, nullptr);
  p->bound.assign(n_clusters, 0);
  p->peer_flags.assign(RV_MAX_RANKS, nullptr);
  {
    DeviceGuard g(device);
    cudaError_t e = cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, device);
    const int lanes_cap = std::max(kMaxLanes, n_rings);
    p->flag_bytes = sizeof(unsigned long long) * flag_index(lanes_cap, 0, 0);
    if (e == cudaSuccess) e = cudaMalloc(&p->flags, p->flag_bytes);
    if (e == cudaSuccess) e = cudaMemset(p->flags, 0, p->flag_bytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->states, sizeof(LaneState) * lanes_cap);
    if (e == cudaSuccess) e = cudaMemset(p->states, 0, sizeof(LaneState) * lanes_cap);
    if (e == cudaSuccess) e = cudaMalloc(&p->status, 4 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(p->status, 0, 4 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaHostAlloc(&p->fail_host, sizeof(unsigned), cudaHostAllocMapped | cudaHostAllocPortable);
    if (e == cudaSuccess) {
      *(volatile unsigned *)p->fail_host = 0u;
      e = cudaHostGetDevicePointer(&p->fail_dev, p->fail_host, 0);
    }
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

int rv_plan_bind_live(rv_plan *p, int pos, void *live) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  if (pos < 0 || pos >= p->C) return set_err(RV_E_ARG, "position %d out of range", pos);
  p->live[pos] = live;
  p->ptrs_dirty = true;
  p->dirty = true;
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
  if (n_lanes < 1 || n_lanes > std::max(kMaxLanes, p->R))
    return set_err(RV_E_ARG, "lanes must be in [1, %d]", std::max(kMaxLanes, p->R));
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
  if (proto != RV_PROTO_PULL && proto != RV_PROTO_PUSH && proto != RV_PROTO_LL)
    return set_err(RV_E_CONFIG, "unknown protocol %d", proto);
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
    if (p->proto == RV_PROTO_LL) {
      // [staging: C writer slots | receive: C owner slots], 8 bytes per element
      p->pflag_bytes = 0;
      p->push_bytes = 2 * (size_t)p->C * p->stride_bound * 8;
    } else {
      // [scatter flags | mean-delivered flags (fused blend)], one per (lane, peer, unit) each
      const size_t nflags = (size_t)std::max(1, p->n_lanes) * p->C * p->units_max;
      p->mflag_off = (int64_t)nflags;
      p->pflag_bytes = (2 * nflags * sizeof(unsigned long long) + 4095) / 4096 * 4096;
      p->push_bytes = p->pflag_bytes + (size_t)p->C * p->stride_bound * elem_size(p->dtype);
    }
    DeviceGuard g(p->device);
    RV_CUDA(cudaMalloc(&p->push_area, p->push_bytes));
    RV_CUDA(cudaMemset(p->push_area, 0, p->proto == RV_PROTO_LL ? p->push_bytes : p->pflag_bytes));
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
    const size_t n = 4 * (size_t)std::max(kMaxLanes, p->R);
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
  if (lane < 0 || lane >= std::max(kMaxLanes, p->R)) return set_err(RV_E_ARG, "bad lane %d", lane);
  DeviceGuard g(p->device);
  RV_CUDA(cudaDeviceSynchronize());
  RV_CUDA(cudaMemcpy(out4, p->trace + 4 * lane, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return RV_OK;
}

int rv_lane_ranges(int n_rings, const int64_t *ring_start, const int64_t *ring_len, int n_lanes,
                   int64_t *lane_lo, int64_t *lane_hi) {
  if (n_rings < 0 || n_lanes < 1 || n_lanes > std::max(kMaxLanes, n_rings) || !lane_lo || !lane_hi ||
      (n_rings > 0 && (!ring_start || !ring_len)))
    return set_err(RV_E_ARG, "bad lane-range arguments");
  rv_plan q;  // host-only description; no device state is touched
  q.R = n_rings;
  q.n_lanes = n_lanes;
  q.rstart.assign(ring_start, ring_start + n_rings);
  q.rlen.assign(ring_len, ring_len + n_rings);
  q.total = 0;
  for (int r = 0; r < n_rings; ++r) q.total += ring_len[r];
  const auto ranges = lane_ranges(&q);
  for (int l = 0; l < n_lanes; ++l) {
    lane_lo[l] = ranges[l].first;
    lane_hi[l] = ranges[l].second;
  }
  return RV_OK;
}

int rv_plan_set_max_blocks(rv_plan *p, int max_blocks) {
  if (!p || max_blocks < 0) return set_err(RV_E_ARG, "bad block budget");
  p->max_blocks = max_blocks;
  p->dirty = true;
  return RV_OK;
}

int rv_plan_set_option(rv_plan *p, int option, int64_t value) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  switch (option) {
    case RV_OPT_MIN_CB:
      if (value < 0 || value > RV_MAX_CLUSTERS) return set_err(RV_E_ARG, "min_cb must be in [0, %d]", RV_MAX_CLUSTERS);
      p->min_cb = (int)value;
      break;
    case RV_OPT_TMA: p->use_tma = value != 0; break;
    case RV_OPT_PUSH_ITEMS:
      if (value < 1 || value > 1024) return set_err(RV_E_ARG, "push items per block must be in [1, 1024]");
      p->push_items = value;
      break;
    case RV_OPT_PUSH_DYN: p->push_dyn = value != 0; break;
    case RV_OPT_BLEND_LAG:
      if (value < -1) return set_err(RV_E_ARG, "blend lag must be >= -1");
      p->blend_lag_opt = value;
      break;
    case RV_OPT_LAYOUT_SMS:
      if (value < 0 || value > 4096) return set_err(RV_E_ARG, "layout SM count must be in [0, 4096]");
      p->layout_sms = (int)value;
      break;
    default: return set_err(RV_E_ARG, "unknown option %d", option);
  }
  p->dirty = true;
  return RV_OK;
}

int rv_plan_prepare(rv_plan *p) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  DeviceGuard g(p->device);
  if (p->dirty || p->ptrs_dirty) return build_tables(p);
  return RV_OK;
}

int rv_plan_layout(rv_plan *p, int64_t *out4) {
  if (!p || !out4) return set_err(RV_E_ARG, "NULL argument");
  if (p->dirty || p->lanes.empty()) return set_err(RV_E_ARG, "plan tables not built (call rv_plan_prepare)");
  out4[0] = p->use_push ? p->lanes[0].unit_vecs : 0;
  out4[1] = p->use_push ? p->stride_bound : 0;
  out4[2] = p->use_push ? p->units_max : 0;
  // work items of the push work order (every rank walks the same list); the
  // pull and LL tables hold this rank's own items only
  out4[3] = p->use_push && !ll_active(p) ? p->lanes[0].n_tiles : 0;
  return RV_OK;
}

int rv_plan_failed(rv_plan *p) {
  if (!p || !p->fail_host) return 0;
  return (int)*(volatile unsigned *)p->fail_host;
}

int rv_plan_set_timeout(rv_plan *p, double seconds) {
  if (!p || !(seconds > 0)) return set_err(RV_E_ARG, "bad timeout");
  p->timeout_ns = (unsigned long long)(seconds * 1e9);
  return RV_OK;
}

int rv_allreduce_mean_lanes(rv_plan *p, int first_lane, int n_lanes, void *const *streams, int n_streams) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  DeviceGuard g(p->device);
  if (p->dirty || p->ptrs_dirty) {
    int rc = build_tables(p);
    if (rc) return rc;
  }
  if (first_lane < 0 || n_lanes < 0 || first_lane + n_lanes > p->n_lanes)
    return set_err(RV_E_ARG, "lanes [%d, %d) outside the plan's %d", first_lane, first_lane + n_lanes, p->n_lanes);
  const int es = elem_size(p->dtype);
  for (int l = first_lane; l < first_lane + n_lanes; ++l) {
    cudaStream_t st = (streams && n_streams > 0) ? (cudaStream_t)streams[l % n_streams] : (cudaStream_t)0;
    int rc = launch_lane(p, l, st);
    if (rc) return rc;
    if (p->blend && !p->fused_blend) {
      // transports without the fused blend: the lane's means are final when
      // its kernel ends, so the blend of the lane's range follows on its stream
      const rv_plan::Lane &lane = p->lanes[l];
      const size_t off = (size_t)lane.lo * es;
      for (int pos : p->local) {
        rc = rv_blend(p->device, p->dtype, (char *)p->live[pos] + off, (const char *)p->src[pos] + off,
                      (const char *)p->dst[pos] + off, lane.hi - lane.lo, st);
        if (rc) return rc;
      }
    }
  }
  return RV_OK;
}

int rv_allreduce_mean(rv_plan *p, void *const *streams, int n_streams) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  return rv_allreduce_mean_lanes(p, 0, p->n_lanes, streams, n_streams);
}

int rv_allreduce_mean_host_lanes(rv_plan *p, int first_lane, int n_lanes, const void *const *host_src,
                                 void *const *host_dst, void *const *streams, int n_streams) {
  if (!p || !host_src || !host_dst) return set_err(RV_E_ARG, "NULL argument");
  DeviceGuard g(p->device);
  if (p->dirty || p->ptrs_dirty) {
    int rc = build_tables(p);
    if (rc) return rc;
  }
  if (first_lane < 0 || n_lanes < 0 || first_lane + n_lanes > p->n_lanes)
    return set_err(RV_E_ARG, "lanes [%d, %d) outside the plan's %d", first_lane, first_lane + n_lanes, p->n_lanes);
  if (p->blend) return set_err(RV_E_ARG, "the host-buffer path does not blend (unbind the live buffers)");
  const int es = elem_size(p->dtype);
  // host->device copies run lane after lane (lane l's kernel starts as soon
  // as its own inputs have landed, while lane l+1's copy streams in and lane
  // l-1's result streams out): a three-stage H2D / average / D2H pipeline
  while ((int)p->h2d_done.size() < p->n_lanes) {
    cudaEvent_t e;
    RV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->h2d_done.push_back(e);
  }
  for (int l = first_lane; l < first_lane + n_lanes; ++l) {
    cudaStream_t st = (streams && n_streams > 0) ? (cudaStream_t)streams[l % n_streams] : (cudaStream_t)0;
    const rv_plan::Lane &lane = p->lanes[l];
    const size_t off = (size_t)lane.lo * es, bytes = (size_t)(lane.hi - lane.lo) * es;
    if (l > 0) RV_CUDA(cudaStreamWaitEvent(st, p->h2d_done[l - 1], 0));
    for (size_t i = 0; i < p->local.size() && bytes > 0; ++i) {
      const int pos = p->local[i];
      RV_CUDA(cudaMemcpyAsync((char *)p->src[pos] + off, (const char *)host_src[i] + off, bytes,
                              cudaMemcpyHostToDevice, st));
    }
    RV_CUDA(cudaEventRecord(p->h2d_done[l], st));
    int rc = launch_lane(p, l, st);
    if (rc) return rc;
    for (size_t i = 0; i < p->local.size() && bytes > 0; ++i) {
      const int pos = p->local[i];
      RV_CUDA(cudaMemcpyAsync((char *)host_dst[i] + off, (const char *)p->dst[pos] + off, bytes,
                              cudaMemcpyDeviceToHost, st));
    }
  }
  return RV_OK;
}

int rv_allreduce_mean_host(rv_plan *p, const void *const *host_src, void *const *host_dst,
                           void *const *streams, int n_streams) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  return rv_allreduce_mean_host_lanes(p, 0, p->n_lanes, host_src, host_dst, streams, n_streams);
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
  const char *ph = phase == 0 ? "arrive" : phase == 1 ? "depart" : phase == 2 ? "unit" : "mean-delivered";
  if (diag && diag_len)
    snprintf(diag, diag_len, "waiting on: (ring=%s, phase=%s, rank=%u)", rings.empty() ? "?" : rings.c_str(), ph,
             peer);
  return set_err(RV_E_TIMEOUT, "peer rank %u never reached the %s barrier (lane %u)", peer, ph, lane);
}

int rv_plan_reset_status(rv_plan *p) {
  if (!p) return set_err(RV_E_ARG, "plan is NULL");
  DeviceGuard g(p->device);
  RV_CUDA(cudaDeviceSynchronize());
  RV_CUDA(cudaMemset(p->status, 0, 4 * sizeof(unsigned)));
  // a cycle that ran with the status set advanced its epoch without posting
  // arrive flags: re-align `signaled` so the next cycle posts them again
  const int lanes_cap = std::max(kMaxLanes, p->R);
  std::vector<LaneState> st(lanes_cap);
  RV_CUDA(cudaMemcpy(st.data(), p->states, sizeof(LaneState) * lanes_cap, cudaMemcpyDeviceToHost));
  for (auto &s : st) {
    s.signaled = s.epoch;
    s.done = 0u;
    s.grab = 0u;
  }
  RV_CUDA(cudaMemcpy(p->states, st.data(), sizeof(LaneState) * lanes_cap, cudaMemcpyHostToDevice));
  RV_CUDA(cudaDeviceSynchronize());
  *(volatile unsigned *)p->fail_host = 0u;
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
    if (p->fail_host) cudaFreeHost(p->fail_host);
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
