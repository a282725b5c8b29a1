// Kernel selection: dtype / accumulation / member count / vector width /
// transport -> template instantiation.
// Part of the single translation unit ravnest_b200.cu (included inside its
// anonymous namespace); see that file for the overview.
#pragma once

// ---------------------------------------------------------------------------
// kernel dispatch

using KernelFn = void (*)(CycleParams);

// Member-count bucket: the smallest instantiated CB >= c, raised to
// `min_cb` (RV_OPT_MIN_CB) so the CB = 8 / 16 kernels of 8- and 16-GPU jobs
// run, with fewer members, on the GPUs a test box has.  Results are
// unchanged: every kernel loops over the runtime C and uses CB only as a
// register-array bound.
int bucket_c(int c, int min_cb) { return min_cb > c ? std::min(min_cb, RV_MAX_CLUSTERS) : c; }

enum Mode { kF32Acc64 = 0, kF32Native = 1, kF64 = 2 };

// Vectors per thread per pass: U*C 16-byte loads in flight, kept within the
// 128-register budget (fp64 storage and the push kernel's staging addresses
// take more registers, so they run at half U).
template <typename T, typename Acc, int VB>
KernelFn pick_cb(int c, bool push, int *u_out) {
  constexpr bool wide = sizeof(T) == 8;
  if (push) {
    // fp64 storage: half again (the blend items' addresses stay in registers)
    if constexpr (wide) {
      if (c <= 2) { *u_out = 2; return ring_push_kernel<T, Acc, 2, VB, 2>; }
      if (c <= 4) { *u_out = 1; return ring_push_kernel<T, Acc, 4, VB, 1>; }
    } else {
      if (c <= 2) { *u_out = 4; return ring_push_kernel<T, Acc, 2, VB, 4>; }
      if (c <= 4) { *u_out = 2; return ring_push_kernel<T, Acc, 4, VB, 2>; }
    }
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

// Co-resident TMA kernel: 64 KB of member data per pipeline stage
// (CB * TV * 16 bytes), 2 stages -> 136-192 KB of shared memory, one block
// per SM.  Measured on BERT / ResNet-50 C=8 against 3 x 32 KB with two
// blocks per SM (0.895 / 0.878 of measured HBM): 0.905-0.933 / 0.919-0.922;
// 2 x 32/40/48/80/96 KB, 3 x 64 KB, 6 x 32 KB, 8 x 16 KB and L2 evict-first
// hints were slower (round-1 experiment builds, DESIGN.md tuning table).
// Round 2, alternating A/B builds (profiles/r02/ab_tma_layouts_n1.txt), BERT
// / ResNet-50 C=8: 2 x 64 KB 0.947 / 0.932, 3 x 64 KB 0.921 / 0.886,
// 4 x 48 KB 0.881 / 0.850 of HBM -- more bytes in flight per SM is slower:
// the pipeline is not latency-bound (the fp32 fold, which skips the f64
// conversions, is within 0.2%).
#ifndef RV_TMA_STAGES  // A/B builds only (tools/gpu_ab_tma.sh); the library uses the defaults
#define RV_TMA_STAGES 2
#endif
#ifndef RV_TMA_STAGE_KB
#define RV_TMA_STAGE_KB 64
#endif
constexpr int kTmaStages = RV_TMA_STAGES;
constexpr int kTmaStageBytes = RV_TMA_STAGE_KB * 1024;
// The fused-blend kernel (each stage carries C snapshot and C live tiles):
// 3 stages of 48 KB.  GPT-2 C=8 config 4, alternating A/B builds
// (profiles/r02/ab_tma_blend_layouts_n1.txt): 3 x 48 KB 0.987 of HBM on the
// 4*C*S basis, 2 x 64 KB 0.915, 2 x 72 KB 0.943 (and too much shared
// memory at C <= 4), 3 x 40 KB 0.827.
#ifndef RV_TMA_BL_STAGES  // A/B builds only override these
#define RV_TMA_BL_STAGES 3
#endif
#ifndef RV_TMA_BL_STAGE_KB
#define RV_TMA_BL_STAGE_KB 48
#endif
constexpr int kTmaBlStages = RV_TMA_BL_STAGES;
constexpr int kTmaBlStageBytes = RV_TMA_BL_STAGE_KB * 1024;

// BL: the fused-blend kernel; a stage carries C src and C live tiles, so the
// same stage bytes hold half the vectors per member.
template <typename T, typename Acc, int STAGES, int STAGE_BYTES, bool BL = false>
KernelFn pick_tma(int c, int *tv_out) {
  constexpr int K = BL ? 2 : 1;
  if (c <= 2) {
    *tv_out = STAGE_BYTES / (K * 2 * 16);
    return ring_tma_kernel<T, Acc, 2, STAGE_BYTES / (K * 2 * 16), STAGES, BL>;
  }
  if (c <= 4) {
    *tv_out = STAGE_BYTES / (K * 4 * 16);
    return ring_tma_kernel<T, Acc, 4, STAGE_BYTES / (K * 4 * 16), STAGES, BL>;
  }
  if (c <= 8) {
    *tv_out = STAGE_BYTES / (K * 8 * 16);
    return ring_tma_kernel<T, Acc, 8, STAGE_BYTES / (K * 8 * 16), STAGES, BL>;
  }
  *tv_out = STAGE_BYTES / (K * 16 * 16);
  return ring_tma_kernel<T, Acc, 16, STAGE_BYTES / (K * 16 * 16), STAGES, BL>;
}

KernelFn pick_tma_kernel(int mode, int c, bool blend, int *tv_out, size_t *smem_out) {
  KernelFn k;
  if (blend)
    k = mode == kF32Acc64 ? pick_tma<float, double, kTmaBlStages, kTmaBlStageBytes, true>(c, tv_out)
      : mode == kF32Native ? pick_tma<float, float, kTmaBlStages, kTmaBlStageBytes, true>(c, tv_out)
                           : pick_tma<double, double, kTmaBlStages, kTmaBlStageBytes, true>(c, tv_out);
  else
    k = mode == kF32Acc64 ? pick_tma<float, double, kTmaStages, kTmaStageBytes>(c, tv_out)
      : mode == kF32Native ? pick_tma<float, float, kTmaStages, kTmaStageBytes>(c, tv_out)
                           : pick_tma<double, double, kTmaStages, kTmaStageBytes>(c, tv_out);
  const int cb = c <= 2 ? 2 : c <= 4 ? 4 : c <= 8 ? 8 : 16;
  // input stages, then the output buffers: 3 mean tiles, or (blend) 2 x
  // (mean + C live tiles) -- must match ring_tma_kernel's NOB / OUTS
  *smem_out = blend ? (size_t)kTmaBlStages * 2 * cb * (*tv_out) * 16 +
                           (size_t)tma_out_buffers(true, cb) * (cb + 1) * (*tv_out) * 16
                    : (size_t)kTmaStages * cb * (*tv_out) * 16 + 3 * (size_t)(*tv_out) * 16;
  return k;
}

KernelFn pick_kernel(int mode, int c, bool vec, bool push, int *u_out) {
  switch (mode) {
    case kF32Acc64: return vec ? pick_cb<float, double, 16>(c, push, u_out) : pick_cb<float, double, 4>(c, push, u_out);
    case kF32Native: return vec ? pick_cb<float, float, 16>(c, push, u_out) : pick_cb<float, float, 4>(c, push, u_out);
    default: return vec ? pick_cb<double, double, 16>(c, push, u_out) : pick_cb<double, double, 8>(c, push, u_out);
  }
}

// LL transport (fp32 storage only)
template <typename Acc>
KernelFn pick_ll(int c) {
  if (c <= 2) return ring_ll_kernel<Acc, 2>;
  if (c <= 4) return ring_ll_kernel<Acc, 4>;
  if (c <= 8) return ring_ll_kernel<Acc, 8>;
  return ring_ll_kernel<Acc, 16>;
}

KernelFn pick_ll_kernel(int mode, int c) {
  return mode == kF32Native ? pick_ll<float>(c) : pick_ll<double>(c);
}
