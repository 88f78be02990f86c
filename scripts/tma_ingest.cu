// Micro-benchmark: per-SM bulk-copy (TMA) ingest rate.
// One CTA per SM streams a private region of a large buffer through a ring of
// S shared-memory stages of B bytes (one producer lane, consumers release each
// stage as soon as it lands, optionally after reading it).  Reports total GB/s
// for a given number of CTAs, stage size and depth -- the ceiling a TMA ring
// design can reach with that many streaming SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_ingest scripts/tma_ingest.cu
//   /tmp/tma_ingest
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_ingest(const float* src, size_t per_cta_bytes, int stage_bytes, int S, int read,
                         float* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, warp = tid >> 5, nwc = blockDim.x / 32 - 1;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(nwc));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = reinterpret_cast<const char*>(src) + blockIdx.x * per_cta_bytes;
  const int n = (int)(per_cta_bytes / stage_bytes);
  if (warp == nwc) {
    if ((tid & 31) == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      uint32_t st = 0, ph = 0;
      for (int i = 0; i < n; ++i) {
        asm volatile(
            "{\n.reg .pred P;\nW1_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W1_%=;\n}" ::"r"(
                sa(&empty[st])),
            "r"(ph ^ 1u));
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])),
                     "r"(stage_bytes));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                sa(smem + (size_t)st * stage_bytes)),
            "l"(base + (size_t)i * stage_bytes), "r"(stage_bytes), "r"(sa(&full[st])), "l"(pol)
            : "memory");
        if (++st == (uint32_t)S) { st = 0; ph ^= 1u; }
      }
    }
  } else {
    uint32_t st = 0, ph = 0;
    float acc = 0.f;
    for (int i = 0; i < n; ++i) {
      asm volatile(
          "{\n.reg .pred P;\nW2_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W2_%=;\n}" ::"r"(
              sa(&full[st])),
          "r"(ph)
          : "memory");
      if (read) {
        const float* x = reinterpret_cast<const float*>(smem + (size_t)st * stage_bytes);
        for (int k = tid; k < stage_bytes / 4; k += nwc * 32) acc += x[k];
      }
      __syncwarp();
      if ((tid & 31) == 0)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
      if (++st == (uint32_t)S) { st = 0; ph ^= 1u; }
    }
    if (acc == 123.f) sink[0] = acc;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)8 << 30;  // 8 GB: far larger than L2
  float* buf;
  if (cudaMalloc(&buf, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 0, total);
  float* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int ctas_list[] = {16, 112, 148};
  const int stage_list[] = {4096, 8192, 17280, 32768};
  const int ring_list[] = {64 * 1024, 128 * 1024, 200 * 1024};
  printf("ctas stage_B ring_KB read  GB/s  GB/s/SM\n");
  for (int ctas : ctas_list) {
    if (ctas > sms) continue;
    for (int sb : stage_list)
      for (int ring : ring_list)
        for (int read = 0; read < 2; ++read) {
          const int S = ring / sb;
          if (S < 2) continue;
          const size_t smem = (size_t)S * sb + 2 * S * 8;
          cudaFuncSetAttribute(k_ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          size_t per = (total / ctas) / sb * sb;
          per = per > ((size_t)48 << 20) ? ((size_t)48 << 20) / sb * sb : per;
          k_ingest<<<ctas, 512, smem>>>(buf, per, sb, S, read, sink);
          cudaEventRecord(a);
          k_ingest<<<ctas, 512, smem>>>(buf, per, sb, S, read, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms = 0;
          cudaEventElapsedTime(&ms, a, b);
          const double gbs = (double)per * ctas / (ms * 1e-3) / 1e9;
          printf("%4d %7d %7d %4d %7.0f %7.1f\n", ctas, sb, ring / 1024, read, gbs, gbs / ctas);
        }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
