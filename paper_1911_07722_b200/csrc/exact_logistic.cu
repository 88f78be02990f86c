// K = P = 1 primal logistic regression: exact coordinate updates on the live
// shared vector (solvers.py:403-410 -> _exact_worker_pass :140-171 ->
// exact_coordinate_update / _logistic_newton, objective.py:113-184).
//
// For quadratic losses the exact update equals the surrogate step with
// a = gamma and runs in the epoch kernels; the logistic loss needs the
// reference's safeguarded 1-D Newton on
//     phi'(d)  = -sum_i x_i y_i sigma(-y_i (v_i + d x_i)) + lam (alpha_j + d)
//     phi''(d) =  sum_i x_i^2 s_i (1 - s_i) + lam
// with the same bracket (rad = 10/sqrt(q_j) + |alpha_j|, doubling up to 60 /
// 120 times), the same 20-iteration Newton with bisection fallback and the
// same 1e-12 step tolerance.  Every phi'/phi'' evaluation is a reduction over
// the column; one cooperative CTA-cluster-free kernel (a single CTA of 1024
// threads, fp64 accumulation, fixed-order block reduction) walks the round's
// coordinates and applies v += delta x_j in place.  This path only serves the
// degenerate configuration (one worker), so a single CTA is the right size.
#include "common.cuh"

namespace syscd {

struct ExactArgs {
  int64_t d;
  int64_t lda;
  const float* A;              // dense store (nullptr for CSC)
  const int64_t* cp;           // CSC store
  const int32_t* ri;
  const float* vals;
  const float* sq;
  float* alpha;
  double* v;                   // live shared vector (fp64), updated in place
  const double* y;
  double lam;
  const int32_t* seq;
  const int64_t* wp;           // one partition: updates wp[0] .. wp[1]
  int32_t* status;
};

constexpr int kExactThreads = 1024;

__device__ __forceinline__ double block_sum2(double a, double b, double* sh, double* out_b) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum_d(a);
  b = warp_sum_d(b);
  __syncthreads();
  if (lane == 0) {
    sh[warp] = a;
    sh[32 + warp] = b;
  }
  __syncthreads();
  double ra = 0.0, rb = 0.0;
  for (int w = 0; w < kExactThreads / 32; ++w) {
    ra += sh[w];
    rb += sh[32 + w];
  }
  *out_b = rb;
  return ra;
}

__device__ __forceinline__ double sig(double z) {
  return z >= 0 ? 1.0 / (1.0 + exp(-z)) : exp(z) / (1.0 + exp(z));
}

__global__ void __launch_bounds__(kExactThreads, 1) k_exact_logistic(ExactArgs A) {
  __shared__ double sh[64];
  const int tid = threadIdx.x;
  const bool dense = A.A != nullptr;
  for (int64_t s = A.wp[0]; s < A.wp[1]; ++s) {
    const int j = A.seq[s];
    const double alpha_j = (double)A.alpha[j];
    const double q = (double)A.sq[j];
    const float* col = dense ? A.A + (int64_t)j * A.lda : nullptr;
    const int64_t e0 = dense ? 0 : A.cp[j];
    const int64_t e1 = dense ? A.d : A.cp[j + 1];
    // phi'(dd), phi''(dd) over the column
    auto dphi = [&](double dd, double* h) -> double {
      double g = 0.0, hh = 0.0;
      for (int64_t e = e0 + tid; e < e1; e += kExactThreads) {
        const int64_t i = dense ? e : A.ri[e];
        const double x = dense ? (double)col[e] : (double)A.vals[e];
        if (x == 0.0) continue;
        const double yi = A.y[i];
        const double sv = sig(-yi * (A.v[i] + dd * x));
        g += x * yi * sv;
        hh += x * x * sv * (1.0 - sv);
      }
      double hsum;
      const double gsum = block_sum2(g, hh, sh, &hsum);
      *h = hsum + A.lam;
      return -gsum + A.lam * (alpha_j + dd);
    };
    double h;
    const double rad = 10.0 / fmax(sqrt(q), 1e-30) + fabs(alpha_j);
    double lo = -rad, hi = rad;
    double glo = dphi(lo, &h);
    double ghi = dphi(hi, &h);
    int widen = 0;
    while (glo > 0.0 && widen < 60) {
      lo *= 2.0;
      glo = dphi(lo, &h);
      ++widen;
    }
    while (ghi < 0.0 && widen < 120) {
      hi *= 2.0;
      ghi = dphi(hi, &h);
      ++widen;
    }
    double dd = 0.0;
    for (int it = 0; it < 20; ++it) {
      const double g = dphi(dd, &h);
      if (g > 0.0) {
        hi = dd;
      } else if (g < 0.0) {
        lo = dd;
      } else {
        break;
      }
      double step = -g / h;
      double nd = dd + step;
      if (!(lo < nd && nd < hi) || !isfinite(nd)) {
        nd = 0.5 * (lo + hi);
        step = nd - dd;
      }
      dd = nd;
      if (fabs(step) < 1e-12) break;
    }
    if (!isfinite(dd)) {
      if (tid == 0) atomicOr(A.status, SYSCD_ENONFINITE);
      dd = 0.0;
    }
    // alpha_j += delta (stored fp32); v += delta_eff x_j so v stays A alpha
    const float an = (float)(alpha_j + dd);
    const double de = (double)an - alpha_j;
    __syncthreads();
    if (tid == 0) A.alpha[j] = an;
    for (int64_t e = e0 + tid; e < e1; e += kExactThreads) {
      const int64_t i = dense ? e : A.ri[e];
      const double x = dense ? (double)col[e] : (double)A.vals[e];
      A.v[i] += de * x;
    }
    __syncthreads();
  }
}

}  // namespace syscd

using namespace syscd;

extern "C" int syscd_exact_logistic_round(const syscd_exact_args* e, void* stream) {
  if (!e || !e->sq || !e->alpha || !e->v || !e->y || !e->seq || !e->work_prefix || !e->status ||
      e->d < 1 || !(e->lam > 0.0) || (!e->A && (!e->col_ptr || !e->row_idx || !e->vals))) {
    set_error("syscd_exact_logistic_round: invalid arguments");
    return SYSCD_EINVAL;
  }
  ExactArgs A;
  A.d = e->d;
  A.lda = e->lda;
  A.A = e->A;
  A.cp = e->col_ptr;
  A.ri = e->row_idx;
  A.vals = e->vals;
  A.sq = e->sq;
  A.alpha = e->alpha;
  A.v = e->v;
  A.y = e->y;
  A.lam = e->lam;
  A.seq = e->seq;
  A.wp = e->work_prefix;
  A.status = e->status;
  k_exact_logistic<<<1, kExactThreads, 0, (cudaStream_t)stream>>>(A);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}
