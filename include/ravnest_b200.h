/*
 * ravnest_b200 -- C ABI of the B200-native Parallel Multi-Ring All-Reduce.
 *
 * Drop-in for the averaging path of Ravnest (arXiv 2401.01728); reference
 * paths below are /root/reference/pkg/src/ravnest/<file>:<line>.
 *
 * Model.  C clusters ("members" of every ring, ascending cluster id =
 * position 0..C-1) each hold a flat parameter vector of total_params
 * elements.  The schedule cuts [0, total_params) into R rings
 * (RingSchedule, multiring.py:31-53, built by build_ring_schedule
 * :56-105).  One cycle leaves every member holding, for chunk k of every ring
 * (chunk_bounds, multiring.py:134-144),
 *
 *     fl( fl(...fl(x_k + x_{k+1}) ... + x_{k+C-1}) / C )      (indices mod C)
 *
 * -- bit for bit what apply_ring_mean (multiring.py:302-333) and
 * AllReduceController (multiring.py:154-247) compute.
 *
 * Execution.  A plan lives on ONE device and folds the chunks of the
 * positions hosted there ("local" positions).  Each chunk k is read from all
 * C member buffers (local HBM or peer memory over NVLink), folded in ring
 * order, divided by C, and written to all C member buffers -- reduce-scatter
 * and all-gather in one kernel.  Devices synchronise through release/acquire
 * flags in each other's memory (no host round trip).  With every position on
 * one device (n_ranks == 1) no flags are used.
 *
 * All calls return an int status (RV_OK or RV_E_*); rv_last_error() gives a
 * thread-local message.  Calls on one plan are not re-entrant.
 */
#ifndef RAVNEST_B200_H
#define RAVNEST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RV_ABI_VERSION 1
#define RV_MAX_CLUSTERS 16
#define RV_MAX_RANKS 16

/* Status codes; the Python shim maps them onto the reference's exception
 * hierarchy (errors.py:4-65). */
#define RV_OK 0
#define RV_E_CONFIG 1      /* ConfigError: C < 2, dtype/mode (multiring.py:268-269)          */
#define RV_E_LAYOUT 2      /* LayoutError: rings do not tile [0,total) (multiring.py:108-116) */
#define RV_E_CUDA 3        /* RavnestError: CUDA runtime failure                              */
#define RV_E_PEER_ACCESS 4 /* RavnestError: peer / IPC mapping unavailable                    */
#define RV_E_TIMEOUT 5     /* StallError: a peer never arrived (multiring.py:296-298)         */
#define RV_E_ARG 6         /* RavnestError: null / unbound / misaligned argument              */

#define RV_DTYPE_F32 0
#define RV_DTYPE_F64 1

/* Accumulation: RV_ACC_F64 folds in float64 and rounds once to the storage
 * dtype -- the reference works in float64 (multiring.py:276,309), so fp32
 * outputs equal float32(reference) bit for bit.  RV_ACC_NATIVE folds in the
 * storage dtype (the fp32 ring order).  For RV_DTYPE_F64 both are the same. */
#define RV_ACC_F64 0
#define RV_ACC_NATIVE 1

/* Transport protocols for multi-device plans.
 * RV_PROTO_PULL: the owner of chunk k loads chunk k of every member over
 *   NVLink, folds, and stores the mean into every member (arrive + depart
 *   barriers).
 * RV_PROTO_PUSH: NVLink carries stores only -- each member stores its copy of
 *   chunk k into owner k's staging slot (one release flag per 256 KB unit),
 *   the owner folds from local memory and stores the mean into every member
 *   (depart barrier only).  Needs one position per rank, rank == position.
 * RV_PROTO_LL: latency transport for small fp32 sets -- every 16-byte store
 *   carries two values each tagged with the cycle's epoch, readers poll the
 *   data itself: no fences, no flags, no barriers; twice the NVLink bytes.
 *   Same placement rule as push; its area comes from rv_plan_push_area. */
#define RV_PROTO_PULL 0
#define RV_PROTO_PUSH 1
#define RV_PROTO_LL 2

typedef struct rv_plan rv_plan;

int rv_version(void);
const char *rv_last_error(void);
const char *rv_status_string(int status);

/* Replaces: consuming RingSchedule (multiring.py:31-53) + the validation of
 * run_allreduce (:267-275) and validate_schedule's tiling check (:108-116).
 * Rings must tile [0, total_params) in order; zero-length rings are legal. */
int rv_plan_create(rv_plan **out, int device, int n_clusters, int n_rings,
                   const int64_t *ring_start, const int64_t *ring_len,
                   int64_t total_params, int dtype, int acc_mode);

/* Member buffers as seen from the plan's device (local, peer-mapped or
 * IPC-imported).  src is read, dst is written; dst == src is in place.
 * Replaces the per-cluster working arrays (multiring.py:276,309). */
int rv_plan_bind(rv_plan *plan, int pos, const void *src, void *dst);

/* Delayed-update blend as part of the cycle (the stale
 * updates of pipeline.py:384-411 landing on the average): with live bound on
 * every local position, each cycle also leaves live <- mean + (live - src)
 * there (exactly mean where live == src bitwise), src being the snapshot that
 * was averaged and dst the mean.  src, dst and live must be distinct.  The
 * push transport blends inside its kernel, unit by unit as the means land
 * (no depart barrier); the others blend each lane's range right after its
 * kernel, on the lane's stream.  live = NULL unbinds. */
int rv_plan_bind_live(rv_plan *plan, int pos, void *live);

/* Positions hosted by this device: their chunks are folded here. */
int rv_plan_set_local(rv_plan *plan, const int *positions, int n_positions);

/* A lane is a contiguous element range averaged by one launch on its own
 * stream (lane l on stream l % n_streams).  1 = one launch for everything;
 * n_rings = one launch per ring (the north-star "one stream per ring");
 * fewer lanes group consecutive rings, more lanes (up to max(64, n_rings))
 * cut rings into equal pieces -- finer host-buffer pipelining. */
int rv_plan_set_lanes(rv_plan *plan, int n_lanes);

/* The lane partition rv_plan_set_lanes uses (host-only, no device needed):
 * lane l covers [lane_lo[l], lane_hi[l]). */
int rv_lane_ranges(int n_rings, const int64_t *ring_start, const int64_t *ring_len, int n_lanes,
                   int64_t *lane_lo, int64_t *lane_hi);

/* This plan's flag area (device memory, cudaMalloc'd: IPC-exportable). */
int rv_plan_flag_area(rv_plan *plan, void **flags, size_t *bytes);

/* Multi-device group: this plan is `rank` of `n_ranks`; peer_flag_areas[r] is
 * rank r's flag area mapped into this device (entry `rank` is ignored). */
int rv_plan_set_peers(rv_plan *plan, int rank, int n_ranks, void *const *peer_flag_areas);

int rv_plan_set_protocol(rv_plan *plan, int proto);

/* Push protocol: this plan's staging + unit-flag area (allocated on first
 * call, sized from the schedule and lane count; IPC-exportable).  Every rank
 * passes all ranks' areas (indexed by rank, mapped into this device). */
int rv_plan_push_area(rv_plan *plan, void **area, size_t *bytes);
int rv_plan_set_push_peers(rv_plan *plan, void *const *areas);

int rv_plan_set_timeout(rv_plan *plan, double seconds);

/* Kernel and layout options.  Kernel choice and the push layout depend only
 * on the schedule, the placement and these calls -- never on the process
 * environment.  Defaults are the measured best (tuning table). */
#define RV_OPT_MIN_CB 1     /* member-count bucket floor (0): run the 8/16-member kernels with fewer members */
#define RV_OPT_TMA 2        /* 1 (default): TMA kernel for co-resident plans with 16 B-congruent buffers; 0: register kernel */
#define RV_OPT_PUSH_ITEMS 3 /* push: work items per resident block that size the units (default 2) */
#define RV_OPT_PUSH_DYN 4   /* push: 1 (default) blocks take work items from a counter; 0: static grid stride */
#define RV_OPT_BLEND_LAG 5  /* push fused blend: groups of C items between a fold and its blends (-1 = two resident grids) */
#define RV_OPT_LAYOUT_SMS 6 /* push: SM count the unit layout assumes (0 = this device's); ranks must agree */
int rv_plan_set_option(rv_plan *plan, int option, int64_t value);

/* Build the device tables now (every position must be bound) instead of at
 * the first cycle, and report the push / LL layout: out[0] vectors per unit,
 * out[1] staging elements per writer slot, out[2] unit-flag slots per (lane,
 * writer), out[3] push work items of lane 0 (all zero for the pull transport,
 * whose tables are per rank; out[3] zero for LL).  Multi-process groups compare it across
 * ranks (it must be identical for push / LL to be correct). */
int rv_plan_prepare(rv_plan *plan);
int rv_plan_layout(rv_plan *plan, int64_t *out4);

/* Non-blocking failure probe: nonzero once a cycle of this plan hit its stall
 * timeout (a host-mapped word the kernels write next to the device status).
 * Reading it after an event that follows the cycle needs no device sync. */
int rv_plan_failed(rv_plan *plan);

/* Cap the blocks a cycle keeps resident (0 = whole device).  An NVLink-bound
 * cycle needs only part of the SMs; the rest stay free for training kernels
 * running concurrently on other streams. */
int rv_plan_set_max_blocks(rv_plan *plan, int max_blocks);

/* Phase tracing (off by default): per lane, the device globaltimer (ns) of
 * [earliest block start, last block ready for data (pull: arrive barrier
 * passed), last block done with data, depart barrier completed] of the most
 * recent launch.  rv_plan_read_trace synchronises the device. */
int rv_plan_set_trace(rv_plan *plan, int enable);
int rv_plan_read_trace(rv_plan *plan, int lane, uint64_t *out4);

/* One averaging cycle, asynchronous on the given CUDA streams (NULL/0 ->
 * the legacy default stream).  Replaces apply_ring_mean / run_allreduce /
 * AllReduceController.kickoff..done (multiring.py:180-232, 254-333). */
int rv_allreduce_mean(rv_plan *plan, void *const *streams, int n_streams);

/* The same for lanes [first_lane, first_lane + n_lanes) only (lane l on
 * streams[l % n_streams]).  Every lane must be run once per cycle.  Lets a
 * process that drives several ranks of one group (loopback, tests) issue the
 * lanes lane-major across its ranks. */
int rv_allreduce_mean_lanes(rv_plan *plan, int first_lane, int n_lanes, void *const *streams, int n_streams);

/* Same cycle with HOST buffers for the local positions: per lane, copy the
 * lane's ring ranges host->device, average, copy device->host, pipelined
 * across lanes.  host_src/host_dst are indexed like rv_plan_set_local's
 * positions (pinned memory for overlap). */
int rv_allreduce_mean_host(rv_plan *plan, const void *const *host_src, void *const *host_dst,
                           void *const *streams, int n_streams);

/* The same for lanes [first_lane, first_lane + n_lanes) only, so a caller can
 * fill lane l+1's host buffers while lane l is in flight (the numpy drop-in
 * path pipelines its float64 copy-in this way).  Every lane must be run once
 * per cycle; lanes are issued in increasing order. */
int rv_allreduce_mean_host_lanes(rv_plan *plan, int first_lane, int n_lanes, const void *const *host_src,
                                 void *const *host_dst, void *const *streams, int n_streams);

/* Blocking: device-side status of the plan (RV_OK or RV_E_TIMEOUT), and a
 * description of the first stall "(ring=r, phase=..., member=m)". */
int rv_plan_status(rv_plan *plan, char *diag, size_t diag_len);
/* Clears the status and re-aligns this plan's own lane bookkeeping (the
 * arrive bookkeeping with its epoch).  It does not re-synchronise epochs
 * across ranks: after a cross-rank stall the ranks may have run different
 * numbers of cycles, so the group must be rebuilt (every rank destroys and
 * recreates its plan, as DistRingGroup.close() + a new group do). */
int rv_plan_reset_status(rv_plan *plan);
int rv_plan_destroy(rv_plan *plan);

/* Delayed-update blend: live <- mean + (live - snap),
 * and exactly mean where live == snap bitwise. */
int rv_blend(int device, int dtype, void *live, const void *snap, const void *mean,
             int64_t n, void *stream);

/* Memory plumbing for multi-process groups (one process per GPU). */
int rv_ipc_handle_size(void);
int rv_ipc_export(const void *dev_ptr, void *handle_out, uint64_t *offset_out);
int rv_ipc_import(int device, const void *handle, uint64_t offset, void **dev_ptr_out);
int rv_ipc_close(int device, void *dev_ptr);
int rv_enable_peer_access(int device, int peer);
int rv_device_sm_count(int device);

#ifdef __cplusplus
}
#endif

#endif /* RAVNEST_B200_H */
