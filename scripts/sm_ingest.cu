// Micro-benchmark: per-SM ingest rate under config 3's access pattern.
// G CTAs (one per SM) each stream their row slice (SLICE bytes) of N columns
// of a column-major matrix (column stride LDA bytes, columns in a seeded
// random order) through an S-stage TMA ring -- k_grid_epoch's data path with
// no grid synchronisation.  Every CTA records its SM id and the %globaltimer
// when it has consumed 1/4, 1/2 and all of its columns, so a per-SM spread of
// ingest rates (the grid kernel runs at its slowest CTA's pace) shows up
// directly.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sm_ingest scripts/sm_ingest.cu
//   /tmp/sm_ingest [G] [slice_bytes] [stages]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_slices(const char* A, long long lda_bytes, const int* order, int n, int slice,
                         int S, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * slice);
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
  const long long off = (long long)blockIdx.x * slice;
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
                     "r"(slice));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                sa(smem + (size_t)st * slice)),
            "l"(A + (long long)order[i] * lda_bytes + off), "r"(slice), "r"(sa(&full[st])), "l"(pol)
            : "memory");
        if (++st == (uint32_t)S) { st = 0; ph ^= 1u; }
      }
    }
  } else {
    uint32_t st = 0, ph = 0;
    float acc = 0.f;
    unsigned long long* o = out + (size_t)blockIdx.x * 8;
    if (tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      o[0] = smid;
      o[1] = gt();
    }
    for (int i = 0; i < n; ++i) {
      asm volatile(
          "{\n.reg .pred P;\nW2_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W2_%=;\n}" ::"r"(
              sa(&full[st])),
          "r"(ph)
          : "memory");
      // 16-byte reads, four independent sums: the consumers must not be
      // what limits the ring
      const float4* x = reinterpret_cast<const float4*>(smem + (size_t)st * slice);
      float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
      for (int k = tid; k < slice / 16; k += nwc * 32) {
        const float4 v = x[k];
        s4.x += v.x; s4.y += v.y; s4.z += v.z; s4.w += v.w;
      }
      acc += s4.x + s4.y + s4.z + s4.w;
      __syncwarp();
      if ((tid & 31) == 0)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
      if (++st == (uint32_t)S) { st = 0; ph ^= 1u; }
      if (tid == 0 && (i + 1 == n / 4 || i + 1 == n / 2 || i + 1 == n)) o[2 + (i + 1 == n / 4 ? 0 : i + 1 == n / 2 ? 1 : 2)] = gt();
    }
    if (acc == 123.f) o[7] = 1;
  }
}

int main(int argc, char** argv) {
  const int G = argc > 1 ? atoi(argv[1]) : 145;
  const int slice = argc > 2 ? atoi(argv[2]) : 27648;
  const int S = argc > 3 ? atoi(argv[3]) : 8;
  const long long lda = 4000000;  // config 3: d = 1M fp32 rows
  const int n = 8000;
  char* A;
  if (cudaMalloc(&A, (size_t)lda * n) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(A, 0, (size_t)lda * n);
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  srand(1);
  for (int i = n - 1; i > 0; --i) std::swap(order[i], order[rand() % (i + 1)]);
  int* dorder;
  cudaMalloc(&dorder, n * 4);
  cudaMemcpy(dorder, order.data(), n * 4, cudaMemcpyHostToDevice);
  unsigned long long* out;
  cudaMalloc(&out, (size_t)G * 8 * 8);
  const size_t smem = (size_t)S * slice + 2 * S * 8;
  cudaFuncSetAttribute(k_slices, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_slices<<<G, 256, smem>>>(A, lda, dorder, n, slice, S, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> h((size_t)G * 8);
    cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < G; ++c) t0 = std::min(t0, h[c * 8 + 1]);
    printf("rep %d: %.3f ms, %.0f GB/s (G=%d slice=%d S=%d)\n", rep, ms,
           (double)G * slice * n / (ms * 1e-3) / 1e9, G, slice, S);
    if (rep == 2) {
      printf("cta smid t_quarter_us t_half_us t_end_us\n");
      for (int c = 0; c < G; ++c)
        printf("%d %llu %.2f %.2f %.2f\n", c, h[c * 8], (h[c * 8 + 2] - t0) * 1e-3,
               (h[c * 8 + 3] - t0) * 1e-3, (h[c * 8 + 4] - t0) * 1e-3);
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
