// Replica reduction + gradient epilogue, and the metrics passes (fresh A alpha,
// A^T w, objective and duality-gap terms) with fp64 accumulation.
//
// Reductions are deterministic: fixed grid, fixed per-block order, then one
// block folds the block partials in index order (reduce_replicas' ascending
// order, solvers.py:122-125).
#include "common.cuh"

namespace syscd {

constexpr int kRedBlocks = 296;  // 2 x 148 SMs
constexpr int kRedThreads = 256;

__device__ __forceinline__ double grad_of(int kind, double v, double y, double lam, double n) {
  switch (kind) {
    case SYSCD_RIDGE:
    case SYSCD_LASSO:
      return v - y;  // objective.py:40-41
    case SYSCD_LOGISTIC: {
      double z = -y * v;  // -y * expit(-y v), objective.py:42
      double s = z >= 0 ? 1.0 / (1.0 + exp(-z)) : exp(z) / (1.0 + exp(z));
      return -y * s;
    }
    default:
      return v / (lam * n * n);
  }
}

__global__ void k_reduce_partials(const float* __restrict__ partials, int64_t ld, int nw, int64_t d,
                                  float* __restrict__ dv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += (double)partials[(int64_t)w * ld + i];
    dv[i] = (float)s;
  }
}

__global__ void k_apply_dv(int kind, int64_t d, const float* __restrict__ dv, double* __restrict__ v,
                           const double* __restrict__ y, double lam, double n, float* __restrict__ u) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double nv = v[i] + (double)dv[i];
    v[i] = nv;
    if (u) u[i] = (float)grad_of(kind, nv, y ? y[i] : 0.0, lam, n);
  }
}

__global__ void k_grad(int kind, int64_t d, const double* __restrict__ v, const double* __restrict__ y,
                       double lam, double n, const double* __restrict__ v_node, double drift,
                       float* __restrict__ u) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x) {
    double gval = grad_of(kind, v[i], y ? y[i] : 0.0, lam, n);
    if (v_node) gval += drift * (v_node[i] - v[i]);
    u[i] = (float)gval;
  }
}

// T2 > 1 node bookkeeping (solvers.py:393,423): acc (+)= v_node - v, v += acc
__global__ void k_node_delta(int64_t d, const double* __restrict__ v_node,
                             const double* __restrict__ v, double* __restrict__ acc, int first) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double dv = v_node[i] - v[i];
    acc[i] = first ? dv : acc[i] + dv;
  }
}

__global__ void k_vec_add(int64_t d, double* __restrict__ v, const double* __restrict__ acc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] += acc[i];
}

__global__ void k_dual_point(int kind, int64_t d, const double* __restrict__ v,
                             const double* __restrict__ y, double lam, double n,
                             double* __restrict__ w) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (kind == SYSCD_SVM_DUAL || kind == SYSCD_LOGISTIC_DUAL) {
      w[i] = v[i] / (lam * n);
    } else {
      w[i] = grad_of(kind, v[i], y ? y[i] : 0.0, lam, n);
    }
  }
}

// out = A x, rows on threads, column chunks on blockIdx.y, fp64 accumulation.
__global__ void k_dense_matvec(int64_t d, int64_t n, int64_t lda, const float* __restrict__ A,
                               const float* __restrict__ x, int64_t chunk, double* __restrict__ dst,
                               int64_t dst_ld) {
  __shared__ float xs[256];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * chunk;
  const int64_t j1 = min(n, j0 + chunk);
  double acc = 0.0;
  for (int64_t jb = j0; jb < j1; jb += 256) {
    const int64_t m = min((int64_t)256, j1 - jb);
    __syncthreads();
    for (int t = threadIdx.x; t < m; t += blockDim.x) xs[t] = x[jb + t];
    __syncthreads();
    if (i < d) {
      const float* col = A + jb * lda + i;
      for (int t = 0; t < m; ++t) {
        const float xv = xs[t];
        if (xv != 0.f) acc += (double)col[(int64_t)t * lda] * (double)xv;
      }
    }
  }
  if (i < d) dst[(int64_t)blockIdx.y * dst_ld + i] = acc;
}

__global__ void k_sum_rows(int64_t d, int nchunks, const double* __restrict__ work, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += work[(int64_t)c * d + i];
    out[i] = s;
  }
}

// out[j] = x_j . w, one warp per column.
__global__ void k_dense_rmatvec(int64_t d, int64_t n, int64_t lda, const float* __restrict__ A,
                                const double* __restrict__ w, double* __restrict__ out) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    const float* col = A + j * lda;
    double acc = 0.0;
    for (int64_t i = lane; i < d; i += 32) acc += (double)col[i] * w[i];
    acc = warp_sum_d(acc);
    if (lane == 0) out[j] = acc;
  }
}

__global__ void k_dense_sqnorm(int64_t d, int64_t n, int64_t lda, const float* __restrict__ A,
                               float* __restrict__ out) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    const float* col = A + j * lda;
    double acc = 0.0;
    for (int64_t i = lane; i < d; i += 32) acc += (double)col[i] * (double)col[i];
    acc = warp_sum_d(acc);
    if (lane == 0) out[j] = (float)acc;
  }
}

// Tall columns (d >= kColBlockMinD): one 256-thread block per column, 16-byte
// loads, four fp64 accumulators per thread and a fixed-order block reduction
// (deterministic).  Optional w (nullptr: squared norm).
constexpr int kColBlockThreads = 256;
constexpr int64_t kColBlockMinD = 4096;

__global__ void __launch_bounds__(kColBlockThreads)
    k_dense_coldot_block(int64_t d, int64_t n, int64_t lda, const float* __restrict__ A,
                         const double* __restrict__ w, double* __restrict__ out_d,
                         float* __restrict__ out_f) {
  __shared__ double red[kColBlockThreads / 32];
  const int tid = threadIdx.x;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const float* col = A + j * lda;  // lda % 4 == 0, 16-byte aligned columns
    const int64_t d4 = d >> 2;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const float4* c4 = reinterpret_cast<const float4*>(col);
    for (int64_t q = tid; q < d4; q += kColBlockThreads) {
      const float4 x = __ldg(c4 + q);
      if (w) {
        const double2 w0 = __ldg(reinterpret_cast<const double2*>(w) + 2 * q);
        const double2 w1 = __ldg(reinterpret_cast<const double2*>(w) + 2 * q + 1);
        a0 = fma((double)x.x, w0.x, a0);
        a1 = fma((double)x.y, w0.y, a1);
        a2 = fma((double)x.z, w1.x, a2);
        a3 = fma((double)x.w, w1.y, a3);
      } else {
        a0 = fma((double)x.x, (double)x.x, a0);
        a1 = fma((double)x.y, (double)x.y, a1);
        a2 = fma((double)x.z, (double)x.z, a2);
        a3 = fma((double)x.w, (double)x.w, a3);
      }
    }
    for (int64_t i = 4 * d4 + tid; i < d; i += kColBlockThreads)
      a0 = fma((double)col[i], w ? w[i] : (double)col[i], a0);
    double acc = warp_sum_d((a0 + a1) + (a2 + a3));
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int k = 0; k < kColBlockThreads / 32; ++k) t += red[k];
      if (out_d) out_d[j] = t;
      if (out_f) out_f[j] = (float)t;
    }
    __syncthreads();
  }
}

__global__ void k_sparse_matvec(int64_t n, const int64_t* __restrict__ cp, const int32_t* __restrict__ ri,
                                const float* __restrict__ vals, const float* __restrict__ x,
                                double* __restrict__ out) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    const float xv = x[j];
    if (xv == 0.f) continue;
    for (int64_t e = cp[j] + lane; e < cp[j + 1]; e += 32)
      atomicAdd(out + ri[e], (double)vals[e] * (double)xv);
  }
}

__global__ void k_sparse_rmatvec(int64_t n, const int64_t* __restrict__ cp, const int32_t* __restrict__ ri,
                                 const float* __restrict__ vals, const double* __restrict__ w,
                                 double* __restrict__ out) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    double acc = 0.0;
    for (int64_t e = cp[j] + lane; e < cp[j + 1]; e += 32) acc += (double)vals[e] * w[ri[e]];
    acc = warp_sum_d(acc);
    if (lane == 0) out[j] = acc;
  }
}

__global__ void k_sparse_sqnorm(int64_t n, const int64_t* __restrict__ cp, const float* __restrict__ vals,
                                float* __restrict__ out) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    double acc = 0.0;
    for (int64_t e = cp[j] + lane; e < cp[j + 1]; e += 32) acc += (double)vals[e] * (double)vals[e];
    acc = warp_sum_d(acc);
    if (lane == 0) out[j] = (float)acc;
  }
}

// ---------------------------------------------------------------------------
// deterministic multi-term reductions: NT terms, sum or max per term
// ---------------------------------------------------------------------------
template <int NT>
struct Terms {
  double v[NT];
};

__device__ __forceinline__ double xlogx(double t) { return t > 0.0 ? t * log(t) : 0.0; }
__device__ __forceinline__ double log1pexp(double z) {  // log(1 + e^z)
  return z > 0 ? z + log1p(exp(-z)) : log1p(exp(z));
}

// mode 0: objective terms. term 0 over rows (f), term 1 over columns (g).
// mode 1: gap terms (see syscd_gap_terms).
struct TermArgs {
  int mode, kind;
  int64_t d, n;
  const double* v;
  const double* y;
  const float* alpha;
  const double* atw;
  double lam, ncoord, scale;
};

__device__ void row_terms(const TermArgs& a, int64_t i, double* t) {
  const double v = a.v[i];
  const double y = a.y ? a.y[i] : 0.0;
  if (a.mode == 0) {
    if (a.kind == SYSCD_RIDGE || a.kind == SYSCD_LASSO) {
      t[0] += 0.5 * (v - y) * (v - y);
    } else if (a.kind == SYSCD_LOGISTIC) {
      t[0] += log1pexp(-y * v);
    } else {
      t[0] += v * v;
    }
    return;
  }
  if (a.kind == SYSCD_RIDGE || a.kind == SYSCD_LASSO) {
    const double w = v - y;
    t[0] += w * w;
    t[1] += w * y;
  } else if (a.kind == SYSCD_LOGISTIC) {
    const double z = -y * v;
    const double s = z >= 0 ? 1.0 / (1.0 + exp(-z)) : exp(z) / (1.0 + exp(z));
    t[0] += xlogx(s) + xlogx(1.0 - s);
  } else {
    const double w = v / (a.lam * a.ncoord);
    t[0] += w * w;
  }
}

__device__ void col_terms(const TermArgs& a, int64_t j, double* t) {
  if (a.mode == 0) {
    const double al = (double)a.alpha[j];
    switch (a.kind) {
      case SYSCD_RIDGE:
      case SYSCD_LOGISTIC:
        t[1] += al * al;
        break;
      case SYSCD_LASSO:
        t[1] += fabs(al);
        break;
      case SYSCD_SVM_DUAL:
        t[1] += al;
        break;
      default:
        t[1] += xlogx(al) + xlogx(1.0 - al);
    }
    return;
  }
  const double m = a.atw[j];
  if (a.kind == SYSCD_RIDGE || a.kind == SYSCD_LOGISTIC) {
    t[2] += m * m;
  } else if (a.kind == SYSCD_LASSO) {
    t[3] = fmax(t[3], fabs(m));
  } else if (a.kind == SYSCD_SVM_DUAL) {
    t[2] += fmax(0.0, 1.0 - m);
  } else {
    t[2] += log1pexp(-m);
  }
}

__global__ void k_terms_partial(TermArgs a, double* __restrict__ work) {
  __shared__ double sh[kRedThreads / 32][4];
  double t[4] = {0, 0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.d; i += stride)
    row_terms(a, i, t);
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.n; j += stride)
    col_terms(a, j, t);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double v = t[q];
    if (q == 3) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    } else {
      v = warp_sum_d(v);
    }
    if (lane == 0) sh[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    const int q = threadIdx.x;
    double v = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) v = q == 3 ? fmax(v, sh[w][q]) : v + sh[w][q];
    work[blockIdx.x * 4 + q] = v;
  }
}

__global__ void k_terms_final(int nblocks, const double* __restrict__ work, double* __restrict__ out) {
  if (threadIdx.x < 4) {
    const int q = threadIdx.x;
    double v = 0.0;
    for (int b = 0; b < nblocks; ++b) v = q == 3 ? fmax(v, work[b * 4 + q]) : v + work[b * 4 + q];
    out[q] = v;
  }
}

static int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace syscd

using namespace syscd;

extern "C" int syscd_reduce_partials(const float* partials, int64_t part_ld, int32_t n_workers,
                                     int64_t d, float* dv, void* stream) {
  if (!partials || !dv || n_workers < 1 || d < 1 || part_ld < d) {
    set_error("syscd_reduce_partials: invalid arguments");
    return SYSCD_EINVAL;
  }
  k_reduce_partials<<<grid_for(d, 256), 256, 0, (cudaStream_t)stream>>>(partials, part_ld,
                                                                          n_workers, d, dv);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_apply_dv(int32_t kind, int64_t d, const float* dv, double* v, const double* y,
                              double lam, double n_coords, float* u, void* stream) {
  if (!dv || !v || d < 1) {
    set_error("syscd_apply_dv: invalid arguments");
    return SYSCD_EINVAL;
  }
  k_apply_dv<<<grid_for(d, 256), 256, 0, (cudaStream_t)stream>>>(kind, d, dv, v, y, lam, n_coords,
                                                                   u);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_grad(int32_t kind, int64_t d, const double* v, const double* y, double lam,
                          double n_coords, const double* v_node, double drift, float* u,
                          void* stream) {
  if (!v || !u || d < 1) {
    set_error("syscd_grad: invalid arguments");
    return SYSCD_EINVAL;
  }
  k_grad<<<grid_for(d, 256), 256, 0, (cudaStream_t)stream>>>(kind, d, v, y, lam, n_coords, v_node,
                                                              drift, u);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_node_delta(int64_t d, const double* v_node, const double* v, double* acc,
                                int32_t first, void* stream) {
  if (!v_node || !v || !acc || d < 1) {
    set_error("syscd_node_delta: invalid arguments");
    return SYSCD_EINVAL;
  }
  k_node_delta<<<grid_for(d, 256), 256, 0, (cudaStream_t)stream>>>(d, v_node, v, acc, first);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_vec_add(int64_t d, double* v, const double* acc, void* stream) {
  if (!v || !acc || d < 1) {
    set_error("syscd_vec_add: invalid arguments");
    return SYSCD_EINVAL;
  }
  k_vec_add<<<grid_for(d, 256), 256, 0, (cudaStream_t)stream>>>(d, v, acc);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_dual_point(int32_t kind, int64_t d, const double* v, const double* y,
                                double lam, double n_coords, double* w, void* stream) {
  if (!v || !w || d < 1) {
    set_error("syscd_dual_point: invalid arguments");
    return SYSCD_EINVAL;
  }
  k_dual_point<<<grid_for(d, 256), 256, 0, (cudaStream_t)stream>>>(kind, d, v, y, lam, n_coords,
                                                                    w);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_dense_matvec(int64_t d, int64_t n, int64_t lda, const float* A, const float* x,
                                  double* out, double* work, int64_t work_bytes, void* stream) {
  if (d < 1 || n < 1 || !A || !x || !out || lda < d) {
    set_error("syscd_dense_matvec: invalid arguments");
    return SYSCD_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int threads = d >= 256 ? 256 : (int)((d + 31) / 32 * 32);
  const int64_t tiles = (d + threads - 1) / threads;
  int64_t nch = (2 * 148 * 8 + tiles - 1) / tiles;
  if (nch > n) nch = n;
  if (nch > 4096) nch = 4096;
  if (work == nullptr || work_bytes < (int64_t)(nch * d * 8)) nch = work ? work_bytes / (d * 8) : 1;
  if (nch < 1) nch = 1;
  const int64_t chunk = (n + nch - 1) / nch;
  nch = (n + chunk - 1) / chunk;
  if (nch == 1) {
    k_dense_matvec<<<dim3((unsigned)tiles, 1), threads, 0, s>>>(d, n, lda, A, x, chunk, out, d);
  } else {
    k_dense_matvec<<<dim3((unsigned)tiles, (unsigned)nch), threads, 0, s>>>(d, n, lda, A, x, chunk,
                                                                           work, d);
    SYSCD_CUDA_TRY(cudaGetLastError());
    k_sum_rows<<<grid_for(d, 256), 256, 0, s>>>(d, (int)nch, work, out);
  }
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_dense_rmatvec(int64_t d, int64_t n, int64_t lda, const float* A,
                                   const double* w, double* out, void* stream) {
  if (d < 1 || n < 1 || !A || !w || !out || lda < d) {
    set_error("syscd_dense_rmatvec: invalid arguments");
    return SYSCD_EINVAL;
  }
  if (d >= kColBlockMinD && ((uintptr_t)w & 15) == 0 && (lda % 4) == 0)
    k_dense_coldot_block<<<(int)(n < 148 * 16 ? n : 148 * 16), kColBlockThreads, 0,
                           (cudaStream_t)stream>>>(d, n, lda, A, w, out, nullptr);
  else
    k_dense_rmatvec<<<grid_for(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(d, n, lda, A, w, out);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_dense_col_sq_norms(int64_t d, int64_t n, int64_t lda, const float* A,
                                        float* out, void* stream) {
  if (d < 1 || n < 1 || !A || !out || lda < d) {
    set_error("syscd_dense_col_sq_norms: invalid arguments");
    return SYSCD_EINVAL;
  }
  if (d >= kColBlockMinD && (lda % 4) == 0)
    k_dense_coldot_block<<<(int)(n < 148 * 16 ? n : 148 * 16), kColBlockThreads, 0,
                           (cudaStream_t)stream>>>(d, n, lda, A, nullptr, nullptr, out);
  else
    k_dense_sqnorm<<<grid_for(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(d, n, lda, A, out);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_sparse_matvec(int64_t d, int64_t n, const int64_t* col_ptr,
                                   const int32_t* row_idx, const float* vals, const float* x,
                                   double* out, void* stream) {
  if (d < 1 || n < 1 || !col_ptr || !row_idx || !vals || !x || !out) {
    set_error("syscd_sparse_matvec: invalid arguments");
    return SYSCD_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  SYSCD_CUDA_TRY(cudaMemsetAsync(out, 0, d * sizeof(double), s));
  k_sparse_matvec<<<grid_for(n * 32, 256), 256, 0, s>>>(n, col_ptr, row_idx, vals, x, out);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_sparse_rmatvec(int64_t n, const int64_t* col_ptr, const int32_t* row_idx,
                                    const float* vals, const double* w, double* out, void* stream) {
  if (n < 1 || !col_ptr || !row_idx || !vals || !w || !out) {
    set_error("syscd_sparse_rmatvec: invalid arguments");
    return SYSCD_EINVAL;
  }
  k_sparse_rmatvec<<<grid_for(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(n, col_ptr, row_idx,
                                                                            vals, w, out);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

extern "C" int syscd_sparse_col_sq_norms(int64_t n, const int64_t* col_ptr, const float* vals,
                                         float* out, void* stream) {
  if (n < 1 || !col_ptr || !vals || !out) {
    set_error("syscd_sparse_col_sq_norms: invalid arguments");
    return SYSCD_EINVAL;
  }
  k_sparse_sqnorm<<<grid_for(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(n, col_ptr, vals, out);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

static int run_terms(const TermArgs& a, double* out, double* work, cudaStream_t s) {
  if (!out || !work) {
    set_error("terms: missing buffers");
    return SYSCD_EINVAL;
  }
  k_terms_partial<<<kRedBlocks, kRedThreads, 0, s>>>(a, work);
  SYSCD_CUDA_TRY(cudaGetLastError());
  k_terms_final<<<1, 32, 0, s>>>(kRedBlocks, work, out);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

// out[0] = sum_rows f-term, out[1] = sum_cols g-term  (callers scale: ridge/logistic g
// is lam/2 * out[1]; lasso lam*out[1]; svm -out[1]/n; logistic-dual out[1]/n;
// dual f = out[0] / (2 lam n^2)).  work: >= 296*4 doubles.
extern "C" int syscd_objective_terms(int32_t kind, int64_t d, int64_t n, const double* v,
                                     const double* y, const float* alpha, double lam,
                                     double n_coords, double* out, double* work, void* stream) {
  if (!v || !alpha || d < 1 || n < 1) {
    set_error("syscd_objective_terms: invalid arguments");
    return SYSCD_EINVAL;
  }
  TermArgs a = {0, kind, d, n, v, y, alpha, nullptr, lam, n_coords, 1.0};
  return run_terms(a, out, work, (cudaStream_t)stream);
}

// Gap terms given atw = A^T w (w from syscd_dual_point):
//  ridge/lasso: out[0]=|w|^2, out[1]=w.y, out[2]=|atw|^2 (ridge), out[3]=max|atw| (lasso)
//  logistic:    out[0]=sum entropy(s), out[2]=|atw|^2
//  svm/logdual: out[0]=|w|^2 (w = v/(lam n)), out[2]=sum hinge / log-loss of margins atw
extern "C" int syscd_gap_terms(int32_t kind, int64_t d, int64_t n, const double* v, const double* y,
                               const double* atw, double lam, double n_coords, double scale,
                               double* out, double* work, void* stream) {
  if (!v || !atw || d < 1 || n < 1) {
    set_error("syscd_gap_terms: invalid arguments");
    return SYSCD_EINVAL;
  }
  TermArgs a = {1, kind, d, n, v, y, nullptr, atw, lam, n_coords, scale};
  return run_terms(a, out, work, (cudaStream_t)stream);
}
