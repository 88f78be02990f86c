// Counter-based synthetic data for the BASELINE workloads.
//
// No reference counterpart: the reference generates its synthetic data with
// numpy on the host (dataset.py:262-273).  Here every value is a pure function
// of (seed, stream tag, column id, row), computed by Philox4x32-10, so a rank
// generates exactly the columns of its own shard in HBM (column-block keys,
// SURVEY 8(d)) and a sharded job holds the same matrix as a one-GPU job.
//
//   syscd_gen_normal_cols  N(0,1) float32 columns into an (n_cols, lda) store
//   syscd_gen_ids          one N(0,1) or U(0,1) float64 value per id
//   syscd_gen_zipf_onehot  nnz distinct Zipf rows per column (inverse CDF),
//                          sorted ascending (config 4's one-hot samples)
#include "common.cuh"

namespace syscd {
namespace {

struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ U4 draw(uint64_t seed, uint32_t tag, uint64_t col, uint32_t ctr) {
  return philox10(U4{ctr, (uint32_t)col, (uint32_t)(col >> 32), tag}, (uint32_t)seed,
                  (uint32_t)(seed >> 32));
}

__device__ __forceinline__ float u24(uint32_t x) {  // (0, 1)
  return ((float)(x >> 8) + 0.5f) * (1.0f / 16777216.0f);
}

__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {  // (0, 1)
  uint64_t m = (((uint64_t)hi << 32) | lo) >> 11;
  return ((double)m + 0.5) * (1.0 / 9007199254740992.0);
}

// four N(0,1) rows 4m..4m+3 of column col
__global__ void k_gen_normal_cols(uint64_t seed, uint32_t tag, const int64_t* __restrict__ cols,
                                  int64_t n_cols, int64_t d, int64_t lda, float* __restrict__ out) {
  const int64_t groups = lda / 4;
  const int64_t total = n_cols * groups;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / groups, m = t - s * groups;
    const uint64_t col = cols ? (uint64_t)cols[s] : (uint64_t)s;
    U4 r = draw(seed, tag, col, (uint32_t)m);
    float rad0 = sqrtf(-2.0f * logf(u24(r.x))), rad1 = sqrtf(-2.0f * logf(u24(r.z)));
    float s0, c0, s1, c1;
    sincospif(2.0f * u24(r.y), &s0, &c0);
    sincospif(2.0f * u24(r.w), &s1, &c1);
    float4 v = make_float4(rad0 * c0, rad0 * s0, rad1 * c1, rad1 * s1);
    const int64_t i = 4 * m;
    if (i + 4 > d) {  // zero padding rows d..lda-1
      if (i + 0 >= d) v.x = 0.f;
      if (i + 1 >= d) v.y = 0.f;
      if (i + 2 >= d) v.z = 0.f;
      if (i + 3 >= d) v.w = 0.f;
    }
    reinterpret_cast<float4*>(out + s * lda)[m] = v;
  }
}

// id streams live in a column range no data column uses
constexpr uint64_t kIdColumn = 0xFFFFFFFF00000000ull;

__global__ void k_gen_ids(uint64_t seed, uint32_t tag, const int64_t* __restrict__ ids, int64_t n,
                          int32_t uniform, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t id = ids ? (uint64_t)ids[t] : (uint64_t)t;
    U4 r = draw(seed, tag, kIdColumn | (id >> 32), (uint32_t)id);
    double u0 = u53(r.x, r.y);
    if (uniform) {
      out[t] = u0;
    } else {
      double u1 = u53(r.z, r.w);
      out[t] = sqrt(-2.0 * log(u0)) * cospi(2.0 * u1);
    }
  }
}

constexpr int kMaxOnehot = 64;

// one thread per column: inverse-CDF Zipf draws until nnz distinct rows,
// in draw order, then sorted (the first-nnz-distinct rule of configs.py)
__global__ void k_gen_zipf_onehot(uint64_t seed, uint32_t tag, const int64_t* __restrict__ cols,
                                  int64_t n_cols, int64_t d, int32_t nnz,
                                  const double* __restrict__ cdf, int32_t* __restrict__ rows,
                                  int32_t* __restrict__ failed) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_cols;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t col = cols ? (uint64_t)cols[s] : (uint64_t)s;
    int32_t got[kMaxOnehot];
    int k = 0;
    for (uint32_t ctr = 0; k < nnz && ctr < (1u << 20); ++ctr) {
      U4 r = draw(seed, tag, col, ctr);
      double us[2] = {u53(r.x, r.y), u53(r.z, r.w)};
      for (int h = 0; h < 2 && k < nnz; ++h) {
        int64_t lo = 0, hi = d - 1;  // first index with cdf >= u
        while (lo < hi) {
          int64_t mid = (lo + hi) >> 1;
          if (cdf[mid] >= us[h])
            hi = mid;
          else
            lo = mid + 1;
        }
        int32_t f = (int32_t)lo;
        bool dup = false;
        for (int q = 0; q < k; ++q) dup |= got[q] == f;
        if (!dup) got[k++] = f;
      }
    }
    if (k < nnz) {
      atomicExch(failed, 1);
      for (; k < nnz; ++k) got[k] = 0;
    }
    for (int a = 1; a < nnz; ++a) {  // insertion sort
      int32_t x = got[a];
      int b = a - 1;
      while (b >= 0 && got[b] > x) {
        got[b + 1] = got[b];
        --b;
      }
      got[b + 1] = x;
    }
    for (int q = 0; q < nnz; ++q) rows[s * nnz + q] = got[q];
  }
}

int grid_of(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  return (int)(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

}  // namespace
}  // namespace syscd

using namespace syscd;

extern "C" int syscd_gen_normal_cols(uint64_t seed, uint32_t tag, const int64_t* cols,
                                     int64_t n_cols, int64_t d, int64_t lda, float* out,
                                     void* stream) {
  if (n_cols < 0 || d < 1 || lda < d || (lda % 4) != 0 || (n_cols > 0 && !out)) {
    set_error("syscd_gen_normal_cols: invalid arguments");
    return SYSCD_EINVAL;
  }
  if (n_cols == 0) return SYSCD_OK;
  k_gen_normal_cols<<<grid_of(n_cols * (lda / 4), 256), 256, 0, (cudaStream_t)stream>>>(
      seed, tag, cols, n_cols, d, lda, out);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_gen_ids(uint64_t seed, uint32_t tag, const int64_t* ids, int64_t n,
                             int32_t uniform, double* out, void* stream) {
  if (n < 0 || (n > 0 && !out)) {
    set_error("syscd_gen_ids: invalid arguments");
    return SYSCD_EINVAL;
  }
  if (n == 0) return SYSCD_OK;
  k_gen_ids<<<grid_of(n, 256), 256, 0, (cudaStream_t)stream>>>(seed, tag, ids, n, uniform, out);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_gen_zipf_onehot(uint64_t seed, uint32_t tag, const int64_t* cols,
                                     int64_t n_cols, int64_t d, int32_t nnz, const double* cdf,
                                     int32_t* rows, int32_t* failed, void* stream) {
  if (n_cols < 0 || d < 1 || nnz < 1 || nnz > kMaxOnehot || nnz > d || !cdf || !failed ||
      (n_cols > 0 && !rows)) {
    set_error("syscd_gen_zipf_onehot: invalid arguments");
    return SYSCD_EINVAL;
  }
  if (n_cols == 0) return SYSCD_OK;
  k_gen_zipf_onehot<<<grid_of(n_cols, 128), 128, 0, (cudaStream_t)stream>>>(
      seed, tag, cols, n_cols, d, nnz, cdf, rows, failed);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}
