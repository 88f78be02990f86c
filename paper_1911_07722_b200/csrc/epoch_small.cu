// SySCD round for short columns (d <= 32, e.g. BASELINE config 1: the SVM
// dual with 28 features and 2M coordinates).
//
// Semantics: _surrogate_thread_round (solvers.py:289-334) -- per coordinate
// lin = x_j . (u + a dv), alpha_j <- step, dv += delta x_j -- on a private
// replica per partition.
//
// For tiny d the chain is latency-bound, so the kernel rewrites it exactly
// (in real arithmetic) over chunks of up to 32 consecutive updates of a
// partition:  with w = u + a dv at the chunk start,
//     c_t  = x_t . w                       (all t in parallel)
//     G_ts = x_t . x_s                     (all s < t in parallel)
//     lin_t = c_t + a * sum_{s<t} delta_s G_ts
// so the sequential part is one step evaluation, one shuffle and one FMA per
// update; afterwards w += a * sum_t delta_t x_t.  One warp is one worker:
// lane t holds column t of the chunk (chain order) in registers; the chunk
// tile and w live in shared memory.  Workers take contiguous update-balanced
// ranges of partitions and fold (w-u)/a into their own partials row at each
// partition end (fixed order: deterministic).
#include <algorithm>

#include "common.cuh"

namespace syscd {

struct SmallArgs {
  const float* A;
  int64_t lda;
  int d;
  const float* sq;
  float* alpha;
  const float* u;
  const int32_t* seq;
  const int64_t* wp;
  int32_t n_parts;
  float a;
  float lam_f, inv_n_f;
  double a_d, lam, n_coords;
  int32_t kind;
  int32_t iid;
  float* partials;
  int64_t part_ld;
  int32_t* status;
};

constexpr int kSmallWarps = 1;  // one worker (partition chain) per block: one SM each

// step for one coordinate given its linear term (kind fixed at compile time)
template <int KIND>
__device__ __forceinline__ float small_step(float r, float alpha, float q, float a, float inv_aq,
                                            float lam, float inv_n, const SmallArgs& A) {
  if (KIND == SYSCD_RIDGE || KIND == SYSCD_LOGISTIC) {
    return alpha - __fdiv_rn(r + lam * alpha, a * q + lam);
  } else if (KIND == SYSCD_LASSO) {
    const float z = alpha - r * inv_aq;
    const float mm = fabsf(z) - lam * inv_aq;
    return q > 0.f ? (mm > 0.f ? copysignf(mm, z) : 0.f) : 0.f;
  } else if (KIND == SYSCD_SVM_DUAL) {
    const float z = alpha - (r - inv_n) * inv_aq;
    return q > 0.f ? fminf(fmaxf(z, 0.f), 1.f) : 1.f;
  } else {
    return (float)logistic_dual_solve((double)r, A.a_d * (double)q, (double)alpha, A.n_coords);
  }
}

__device__ __forceinline__ int64_t lb_small(const int64_t* a, int n, int64_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) {
      lo = mid + 1;
    } else {
      hi = mid;
    }
  }
  return lo;
}

template <int D, int KIND>
__global__ void __launch_bounds__(32 * kSmallWarps) k_small_epoch(SmallArgs A, int W) {
  constexpr int DP = D + 4;  // padded row: 16-byte aligned, conflict-free 16-byte reads
  __shared__ __align__(16) float s_tile[kSmallWarps][32][DP];  // [chunk column][row]
  __shared__ float s_w[kSmallWarps][32];
  __shared__ float s_delta[kSmallWarps][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int g = blockIdx.x * kSmallWarps + wib;
  if (g >= W) return;
  float(*tile)[DP] = s_tile[wib];
  float* wsh = s_w[wib];
  float* dsh = s_delta[wib];
  const int d = A.d;
  const float a = A.a;
  const float inv_a = (float)(1.0 / A.a_d);

  const int64_t total = A.wp[A.n_parts];
  const int64_t t_lo = (int64_t)((__int128)total * g / W);
  const int64_t t_hi = (int64_t)((__int128)total * (g + 1) / W);
  const int64_t p_lo = g == 0 ? 0 : lb_small(A.wp, A.n_parts + 1, t_lo);
  const int64_t p_hi = g == W - 1 ? A.n_parts : lb_small(A.wp, A.n_parts + 1, t_hi);
  float* out = A.partials + (int64_t)g * A.part_ld;
  const float u_l = lane < d ? A.u[lane] : 0.f;
  bool flushed = false;

  for (int64_t p = p_lo; p < p_hi; ++p) {
    const int64_t s0 = A.wp[p], s1 = A.wp[p + 1];
    if (s1 == s0) continue;
    wsh[lane] = u_l;  // w = u at the partition start
    __syncwarp();
    // prefetch registers for the next chunk (columns + scalars)
    int j_n = 0;
    float x_n[D];
    float q_n = 0.f, a_n = 0.f;
    {
      const int m0 = (int)min((int64_t)32, s1 - s0);
      if (lane < m0) {
        j_n = A.seq[s0 + lane];
        const float* col = A.A + (int64_t)j_n * A.lda;
#pragma unroll
        for (int i = 0; i < D; ++i) x_n[i] = i < d ? __ldg(col + i) : 0.f;
        q_n = __ldg(A.sq + j_n);
        a_n = A.alpha[j_n];
      } else {
#pragma unroll
        for (int i = 0; i < D; ++i) x_n[i] = 0.f;
      }
    }
    for (int64_t c0 = s0; c0 < s1; c0 += 32) {
      const int m = (int)min((int64_t)32, s1 - c0);
      // ---- stage: lane t holds column j_t (chain order) and its scalars
      const int j = j_n;
      float x[D];
#pragma unroll
      for (int i = 0; i < D; ++i) x[i] = x_n[i];
      const float q_t = q_n;
      // iid rounds may revisit a coordinate of an earlier chunk: reload
      float alpha_t = A.iid ? (lane < m ? *(volatile float*)(A.alpha + j) : 0.f) : a_n;
      {
        const int64_t c1 = c0 + 32;
        const int m1 = (int)min((int64_t)32, s1 - c1);
        if (lane < m1) {
          j_n = A.seq[c1 + lane];
          const float* col = A.A + (int64_t)j_n * A.lda;
#pragma unroll
          for (int i = 0; i < D; ++i) x_n[i] = i < d ? __ldg(col + i) : 0.f;
          q_n = __ldg(A.sq + j_n);
          if (!A.iid) a_n = A.alpha[j_n];
        }
      }
      const float inv_aq = q_t > 0.f ? __fdiv_rn(1.f, a * q_t) : 0.f;
#pragma unroll
      for (int i = 0; i < D; ++i) tile[lane][i] = x[i];
      __syncwarp();
      // ---- c_t = x_t . w and the strictly-lower Gram row G_t[s], s < t
      float r = 0.f;
#pragma unroll
      for (int i = 0; i < D; ++i) r = fmaf(x[i], wsh[i], r);
      // branch-free: every lane computes the full row, entries s >= t unused
      float G[32];
#pragma unroll
      for (int s = 0; s < 32; ++s) {
        const float4* ts = reinterpret_cast<const float4*>(tile[s]);
        float acc = 0.f;
#pragma unroll
        for (int i4 = 0; i4 < D / 4; ++i4) {
          const float4 v = ts[i4];
          acc = fmaf(x[4 * i4], v.x, acc);
          acc = fmaf(x[4 * i4 + 1], v.y, acc);
          acc = fmaf(x[4 * i4 + 2], v.z, acc);
          acc = fmaf(x[4 * i4 + 3], v.w, acc);
        }
        G[s] = acc;
      }
      // ---- sequential chain: lane s finalises lin_s, broadcasts delta_s
      float my_delta = 0.f;
#pragma unroll
      for (int s = 0; s < 32; ++s) {
        if (s < m) {
          float cand;
          if (KIND == SYSCD_LOGISTIC_DUAL) {
            // Newton solve on the owning lane only (keeps the loop body small)
            cand = 0.f;
            if (lane == s)
              cand = small_step<KIND>(r, alpha_t, q_t, a, inv_aq, A.lam_f, A.inv_n_f, A);
          } else {
            cand = small_step<KIND>(r, alpha_t, q_t, a, inv_aq, A.lam_f, A.inv_n_f, A);
          }
          float dl = cand - alpha_t;
          if (!isfinite(cand)) dl = 0.f;
          const float delta = __shfl_sync(0xffffffffu, dl, s);
          const int js = __shfl_sync(0xffffffffu, j, s);
          if (lane == s) {
            my_delta = delta;
            if (!isfinite(cand)) atomicOr(A.status, SYSCD_ENONFINITE);
          }
          r = fmaf(a * delta, G[s], r);
          // a coordinate drawn twice in one chunk (iid) sees its new value
          if (A.iid && lane > s && j == js) alpha_t += delta;
        }
      }
      {
        // a repeated coordinate (iid) is written once, by its last occurrence
        const unsigned act = __ballot_sync(0xffffffffu, lane < m);
        const unsigned same = __match_any_sync(0xffffffffu, lane < m ? j : -1 - lane) & act;
        if (lane < m && (31 - __clz(same)) == lane) A.alpha[j] = alpha_t + my_delta;
      }
      dsh[lane] = lane < m ? my_delta : 0.f;
      __syncwarp();
      // ---- w += a * sum_t delta_t x_t   (lane = row)
      if (lane < d) {
        float acc = 0.f;
        for (int t = 0; t < m; ++t) acc = fmaf(dsh[t], tile[t][lane], acc);
        wsh[lane] = fmaf(a, acc, wsh[lane]);
      }
      __syncwarp();
    }
    // ---- partition end: fold (w - u)/a into this worker's partial row
    if (lane < d) {
      const float dv = (wsh[lane] - u_l) * inv_a;
      out[lane] = flushed ? out[lane] + dv : dv;
    }
    flushed = true;
    __syncwarp();
  }
  if (!flushed && lane < d) out[lane] = 0.f;
}

int small_workers(int32_t n_parts) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, std::min((int)n_parts, sms * 8));
}

int small_launch(const syscd_dense_epoch_args* e, cudaStream_t stream) {
  SmallArgs A;
  A.A = e->A;
  A.lda = e->lda;
  A.d = (int)e->d;
  A.sq = e->sq;
  A.alpha = e->alpha;
  A.u = e->u;
  A.seq = e->seq;
  A.wp = e->work_prefix;
  A.n_parts = e->n_parts;
  A.a = (float)e->a;
  A.lam_f = (float)e->lam;
  A.inv_n_f = (float)(1.0 / e->n_coords);
  A.a_d = e->a;
  A.lam = e->lam;
  A.n_coords = e->n_coords;
  A.kind = e->kind;
  A.iid = e->iid;
  A.partials = e->partials;
  A.part_ld = e->part_ld;
  A.status = e->status;
  const int W = small_workers(e->n_parts);
  const int blocks = (W + kSmallWarps - 1) / kSmallWarps;
  const int Dsel = e->d <= 8 ? 8 : (e->d <= 16 ? 16 : 32);
  void (*fn)(SmallArgs, int) = nullptr;
#define SYSCD_SMALL_CASE(DD, KK) \
  if (Dsel == DD && kind_sel == KK) fn = &k_small_epoch<DD, KK>;
  const int kind_sel = e->kind == SYSCD_LOGISTIC ? SYSCD_RIDGE : e->kind;
  SYSCD_SMALL_CASE(8, SYSCD_RIDGE) SYSCD_SMALL_CASE(8, SYSCD_LASSO)
  SYSCD_SMALL_CASE(8, SYSCD_SVM_DUAL) SYSCD_SMALL_CASE(8, SYSCD_LOGISTIC_DUAL)
  SYSCD_SMALL_CASE(16, SYSCD_RIDGE) SYSCD_SMALL_CASE(16, SYSCD_LASSO)
  SYSCD_SMALL_CASE(16, SYSCD_SVM_DUAL) SYSCD_SMALL_CASE(16, SYSCD_LOGISTIC_DUAL)
  SYSCD_SMALL_CASE(32, SYSCD_RIDGE) SYSCD_SMALL_CASE(32, SYSCD_LASSO)
  SYSCD_SMALL_CASE(32, SYSCD_SVM_DUAL) SYSCD_SMALL_CASE(32, SYSCD_LOGISTIC_DUAL)
#undef SYSCD_SMALL_CASE
  if (!fn) {
    set_error("small epoch: unsupported objective");
    return SYSCD_EINVAL;
  }
  fn<<<blocks, 32 * kSmallWarps, 0, stream>>>(A, W);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

}  // namespace syscd
