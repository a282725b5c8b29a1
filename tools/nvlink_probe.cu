// NVLink traffic-pattern probe (single process, all visible GPUs, peer access).
// Measures what the multi-ring average's traffic patterns can reach on this
// box, per GPU and per direction:
//   read  : GPU g loads chunk g of every peer's buffer (remote loads only)
//   write : GPU g stores its chunk q into peer q's buffer (remote stores only)
//   mixed : GPU g loads chunk g of every member and stores it to every member
//           (the pull protocol's traffic: loads + stores)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_probe tools/nvlink_probe.cu
#include <cuda_runtime.h>

#include <chrono>
#include <string>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e = (x);                                                                \
    if (e != cudaSuccess) {                                                             \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

constexpr int MAXG = 8;
struct Bufs {
  uint4 *b[MAXG];
};

template <int U, int MODE>  // MODE 0 read, 1 write, 2 mixed
__global__ void __launch_bounds__(256) probe(Bufs bufs, int ng, int me, long long chunk_vecs, uint4 *scratch) {
  const long long stride = (long long)gridDim.x * blockDim.x * U;
  for (long long j0 = (long long)blockIdx.x * blockDim.x * U + threadIdx.x; j0 < chunk_vecs; j0 += stride) {
    if (MODE == 0) {
      uint4 acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = make_uint4(0, 0, 0, 0);
      for (int p = 0; p < ng; ++p) {
        if (p == me) continue;
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          long long j = j0 + (long long)u * blockDim.x;
          if (j < chunk_vecs) v[u] = __ldcs(bufs.b[p] + (long long)me * chunk_vecs + j);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u].x ^= v[u].x, acc[u].y ^= v[u].y, acc[u].z ^= v[u].z, acc[u].w ^= v[u].w;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long j = j0 + (long long)u * blockDim.x;
        if (j < chunk_vecs) __stcs(scratch + j, acc[u]);
      }
    } else if (MODE == 1) {
      for (int p = 0; p < ng; ++p) {
        if (p == me) continue;
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          long long j = j0 + (long long)u * blockDim.x;
          if (j < chunk_vecs) v[u] = __ldcs(bufs.b[me] + (long long)p * chunk_vecs + j);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          long long j = j0 + (long long)u * blockDim.x;
          if (j < chunk_vecs) __stcs(bufs.b[p] + (long long)me * chunk_vecs + j + (long long)ng * chunk_vecs, v[u]);
        }
      }
    } else {
      uint4 v[U][MAXG];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long j = j0 + (long long)u * blockDim.x;
        if (j < chunk_vecs)
#pragma unroll
          for (int p = 0; p < MAXG; ++p)
            if (p < ng) v[u][p] = __ldcs(bufs.b[p] + (long long)me * chunk_vecs + j);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long j = j0 + (long long)u * blockDim.x;
        if (j < chunk_vecs) {
          uint4 a = v[u][0];
#pragma unroll
          for (int p = 1; p < MAXG; ++p)
            if (p < ng) a.x += v[u][p].x, a.y += v[u][p].y, a.z += v[u][p].z, a.w += v[u][p].w;
#pragma unroll
          for (int p = 0; p < MAXG; ++p)
            if (p < ng) __stcs(bufs.b[p] + (long long)me * chunk_vecs + j, a);
        }
      }
    }
  }
}

// TMA bulk copies: each block streams 16 KB tiles between peer global memory
// and shared memory with cp.async.bulk (MODE 3: bulk stores smem -> peer,
// MODE 4: bulk loads peer -> smem).  Data content is irrelevant here.
constexpr int kTile = 16384;
constexpr int kStages = 4;

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(128) probe_bulk(Bufs bufs, int ng, int me, long long chunk_bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[kStages];
  const long long tiles = chunk_bytes / kTile;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int stage = 0;
  unsigned phase[kStages] = {0, 0, 0, 0};
  long long issued = 0;
  for (int p = 0; p < ng; ++p) {
    if (p == me) continue;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
      unsigned char *buf = sm + stage * kTile;
      if (MODE == 3) {
        char *dst = (char *)bufs.b[p] + (long long)me * chunk_bytes + t * kTile;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(buf)),
                     "r"(kTile)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kStages - 1));
      } else {
        const char *src = (const char *)bufs.b[p] + (long long)me * chunk_bytes + t * kTile;
        if (issued >= kStages) {
          unsigned ok = 0;
          while (!ok)
            asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }"
                         : "=r"(ok)
                         : "r"(smem_u32(&bar[stage])), "r"(phase[stage]));
          phase[stage] ^= 1;
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[stage])), "r"(kTile));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(buf)),
            "l"(src), "r"(kTile), "r"(smem_u32(&bar[stage]))
            : "memory");
        ++issued;
      }
      stage = (stage + 1) % kStages;
    }
  }
  if (MODE == 3) asm volatile("cp.async.bulk.wait_group 0;");
  else
    for (int s = 0; s < kStages && s < issued; ++s) {
      unsigned ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }"
                     : "=r"(ok)
                     : "r"(smem_u32(&bar[s])), "r"(phase[s]));
    }
}

template <int MODE>
double run_bulk(int ng, Bufs bufs, long long chunk_bytes, int blocks_per_sm, int iters) {
  std::vector<cudaEvent_t> a(ng), b(ng);
  std::vector<cudaStream_t> st(ng);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int smem = kTile * kStages;
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaFuncSetAttribute(probe_bulk<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&a[g]));
    CK(cudaEventCreate(&b[g]));
  }
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    probe_bulk<MODE><<<sms * blocks_per_sm, 128, smem, st[g]>>>(bufs, ng, g, chunk_bytes);
  }
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a[g], st[g]));
  }
  for (int i = 0; i < iters; ++i)
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      probe_bulk<MODE><<<sms * blocks_per_sm, 128, smem, st[g]>>>(bufs, ng, g, chunk_bytes);
    }
  double worst = 0;
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventRecord(b[g], st[g]));
    CK(cudaEventSynchronize(b[g]));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a[g], b[g]));
    worst = ms > worst ? ms : worst;
  }
  const double bytes = (double)(ng - 1) * (chunk_bytes / kTile * kTile);
  return bytes / (worst / iters * 1e-3) / 1e9;
}

// copy engines: every GPU copies its chunk q to peer q on one stream per peer
double run_ce(int ng, Bufs bufs, long long chunk_bytes, int iters) {
  std::vector<std::vector<cudaStream_t>> st(ng, std::vector<cudaStream_t>(ng));
  std::vector<cudaEvent_t> a(ng), b(ng);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < ng; ++p) CK(cudaStreamCreateWithFlags(&st[g][p], cudaStreamNonBlocking));
    CK(cudaEventCreate(&a[g]));
    CK(cudaEventCreate(&b[g]));
  }
  auto once = [&]() {
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      for (int p = 0; p < ng; ++p)
        if (p != g)
          CK(cudaMemcpyPeerAsync((char *)bufs.b[p] + (long long)g * chunk_bytes + (long long)ng * chunk_bytes, p,
                                 (char *)bufs.b[g] + (long long)p * chunk_bytes, g, chunk_bytes, st[g][p]));
    }
  };
  once();
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceSynchronize());
  }
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) once();
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceSynchronize());
  }
  double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return (double)(ng - 1) * chunk_bytes * iters / sec / 1e9;
}

template <int U, int MODE>
double run(int ng, Bufs bufs, std::vector<uint4 *> &scratch, long long chunk_vecs, int blocks_per_sm, int iters) {
  std::vector<cudaEvent_t> a(ng), b(ng);
  std::vector<cudaStream_t> st(ng);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&a[g]));
    CK(cudaEventCreate(&b[g]));
  }
  for (int w = 0; w < 2; ++w)
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      probe<U, MODE><<<sms * blocks_per_sm, 256, 0, st[g]>>>(bufs, ng, g, chunk_vecs, scratch[g]);
    }
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceSynchronize());
  }
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventRecord(a[g], st[g]));
  }
  for (int i = 0; i < iters; ++i)
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      probe<U, MODE><<<sms * blocks_per_sm, 256, 0, st[g]>>>(bufs, ng, g, chunk_vecs, scratch[g]);
    }
  double worst = 0;
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventRecord(b[g], st[g]));
    CK(cudaEventSynchronize(b[g]));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a[g], b[g]));
    worst = ms > worst ? ms : worst;
  }
  // per-GPU bytes per direction per launch: (ng-1) chunks each way for
  // read/write; 2*(ng-1) chunks each way for mixed
  const double chunk_bytes = (double)chunk_vecs * 16;
  const double bytes = (MODE == 2 ? 2.0 : 1.0) * (ng - 1) * chunk_bytes;
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    cudaStreamDestroy(st[g]);
  }
  return bytes / (worst / iters * 1e-3) / 1e9;
}

int main(int argc, char **argv) {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng > MAXG) ng = MAXG;
  const long long total_bytes = argc > 1 ? atoll(argv[1]) : 437928960LL;  // BERT-base fp32
  const long long chunk_vecs = total_bytes / 16 / ng;
  Bufs bufs{};
  std::vector<uint4 *> scratch(ng);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < ng; ++p)
      if (p != g) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(p, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
        cudaGetLastError();
      }
    CK(cudaMalloc(&bufs.b[g], (size_t)chunk_vecs * 16 * ng * 2));
    CK(cudaMemset(bufs.b[g], 1, (size_t)chunk_vecs * 16 * ng * 2));
    CK(cudaMalloc(&scratch[g], (size_t)chunk_vecs * 16));
  }
  printf("GPUs %d, %lld bytes per member, chunk %lld bytes\n", ng, total_bytes, chunk_vecs * 16);
  if (argc > 2) {
    // single pattern, few launches (for ncu: nvlrx/nvltx user vs protocol bytes)
    const std::string m = argv[2];
    double r = 0;
    if (m == "write") r = run<4, 1>(ng, bufs, scratch, chunk_vecs, 2, 2);
    else if (m == "read") r = run<4, 0>(ng, bufs, scratch, chunk_vecs, 2, 2);
    else if (m == "mixed") r = run<4, 2>(ng, bufs, scratch, chunk_vecs, 2, 2);
    else if (m == "bulkstore") r = run_bulk<3>(ng, bufs, chunk_vecs * 16, 2, 2);
    else if (m == "bulkload") r = run_bulk<4>(ng, bufs, chunk_vecs * 16, 2, 2);
    printf("%s %.1f GB/s per GPU per direction\n", m.c_str(), r);
    return 0;
  }
  const int iters = 20;
  for (int bps : {1, 2, 4}) {
    printf("blocks/SM %d: read U4 %.1f  U8 %.1f | write U4 %.1f U8 %.1f | mixed U2 %.1f U4 %.1f GB/s per GPU per direction\n",
           bps, run<4, 0>(ng, bufs, scratch, chunk_vecs, bps, iters), run<8, 0>(ng, bufs, scratch, chunk_vecs, bps, iters),
           run<4, 1>(ng, bufs, scratch, chunk_vecs, bps, iters), run<8, 1>(ng, bufs, scratch, chunk_vecs, bps, iters),
           run<2, 2>(ng, bufs, scratch, chunk_vecs, bps, iters), run<4, 2>(ng, bufs, scratch, chunk_vecs, bps, iters));
  }
  for (int bps : {1, 2}) {
    printf("TMA bulk blocks/SM %d: bulk-store %.1f | bulk-load %.1f GB/s per GPU per direction\n", bps,
           run_bulk<3>(ng, bufs, chunk_vecs * 16, bps, iters), run_bulk<4>(ng, bufs, chunk_vecs * 16, bps, iters));
  }
  printf("copy engines (cudaMemcpyPeerAsync, stream per peer): %.1f GB/s per GPU per direction (host timed)\n",
         run_ce(ng, bufs, chunk_vecs * 16, iters));
  // one pair, one direction: the calibration point for the 770 GB/s figure
  {
    Bufs two = bufs;
    printf("pair 0->1 only: write U4 %.1f\n", run<4, 1>(2, two, scratch, chunk_vecs, 2, iters) * 1.0);
  }
  return 0;
}
