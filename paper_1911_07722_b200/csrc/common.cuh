// Shared device helpers: status codes, objective kinds, per-coordinate steps,
// and the sm_100a PTX wrappers (mbarrier, 1-D bulk TMA, DSMEM st.async).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/syscd_b200.h"

namespace syscd {

// ---------------------------------------------------------------------------
// per-coordinate step: argmin_delta lin*delta + (a q/2) delta^2 + g_j(alpha+delta)
// Ridge/primal-logistic row = reference surrogate_delta (objective.py:213-215);
// the others are SURVEY Appendix A.  Computed in fp64 on every thread of the
// worker (uniform), returns the new coordinate value.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double sigmoid_d(double s) {
  if (s >= 0.0) return 1.0 / (1.0 + exp(-s));
  double e = exp(s);
  return e / (1.0 + e);
}

// fp32 logistic with SFU exp (relative error ~1e-7, below alpha's fp32 storage)
__device__ __forceinline__ double sigmoid_fast(double s) {
  const float e = __expf(-fabsf((float)s));
  const float r = __fdividef(1.f, 1.f + e);
  return (double)(s >= 0.0 ? r : e * r);
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Fast path of the logistic-dual coordinate solve (see logistic_dual_solve).
// Mirror the root into the left half: with C = aq alpha - lin the root of h
// solves aq sigma(s) = C - s/n; if C > aq/2 substitute s' = -s, which turns it
// into aq sigma(s') = (aq - C) - s'/n.  So always solve aq sigma(s) = Cl - s/n
// with Cl <= aq/2 (the root then sits at sigma <= 1/2, where the log form is
// well conditioned):
//   * tail (n aq sigma(n Cl) small): the sigmoid term is a small perturbation
//     of the linear one and the contraction s <- n (Cl - aq sigma(s)) starting
//     at s = n Cl converges in a few steps;
//   * otherwise Newton on G(s) = log sigma(s) - log(Cl - s/n) + log aq, which
//     is monotone and close to linear near the root; ~3 steps from
//     s0 = logit(Cl / aq).
// Both iterations run in fp32 with SFU exp / log / rcp (they only have to
// land within ~1e-5 of the root).
// One fp64 Newton step on h itself then polishes the root to the accuracy of
// the fp32 sigmoid.  Returns false (caller falls back to the bracketed loop)
// when 8 steps do not converge or the residual of h is not small.
#ifdef SYSCD_NEWTON_HIST
// experiment: [tail][iterations] counts and fallbacks of the fast path
__device__ unsigned long long g_newton_hist[2][12];
#endif
__device__ __forceinline__ bool logistic_dual_fast(double lin, double aq, double alpha, double n,
                                                   double inv_n, double* s_out, double* alpha_out) {
  const double C = aq * alpha - lin;
  const bool left = 0.5 * aq - C > 0.0;
  const double Cl = left ? C : aq - C;
  // the iteration runs in fp32 (the fp64 polish below restores accuracy)
  const float aqf = (float)aq, nf = (float)n, inv_nf = (float)inv_n;
  const float Clf = (float)Cl, nClf = (float)(n * Cl);
  const float e0 = __expf(-fabsf(nClf));
  const float sig0 = nClf >= 0.f ? rcp_approx(1.f + e0) : e0 * rcp_approx(1.f + e0);
  const bool tail = nf * aqf * sig0 < 0.25f;
  const float cap = nClf - 1e-6f * fmaxf(1.f, fabsf(nClf));
  float sp;
  if (tail) {
    sp = nClf;
  } else {
    const float r = Clf * rcp_approx(aqf);
    sp = r > 0.f ? __logf(r) - __logf(1.f - fminf(r, 0.5f)) : nClf - 1.f;
    sp = fminf(sp, nClf - 1e-3f * fmaxf(1.f, fabsf(nClf)));
  }
  const float log_aq = __logf(aqf);
  bool conv = false;
#ifdef SYSCD_NEWTON_HIST
  int its = 0;
#endif
#pragma unroll 1
  for (int it = 0; it < 8; ++it) {
#ifdef SYSCD_NEWTON_HIST
    ++its;
#endif
    const float e = __expf(-fabsf(sp));
    const float w = rcp_approx(1.f + e);
    float ns;
    if (tail) {
#ifndef SYSCD_TAIL_CONTRACTION
      // Newton on F(s) = s - n (Cl - aq sigma(s)): F' = 1 + n aq sigma (1 -
      // sigma) >= 1 and F is convex in the tail, so from s0 = n Cl (F > 0)
      // the iterates decrease monotonically onto the root, quadratically
      const float sig = sp >= 0.f ? w : e * w;
      const float F = sp - nf * (Clf - aqf * sig);
      const float dF = fmaf(nf * aqf * sig, 1.f - sig, 1.f);
      ns = sp - F * rcp_approx(dF);
#else
      ns = nf * (Clf - aqf * (sp >= 0.f ? w : e * w));
#endif
    } else {
      const float R = Clf - sp * inv_nf;
      if (R > 0.f) {
        const float G = fminf(sp, 0.f) - __logf(1.f + e) - __logf(R) + log_aq;
        const float dG = (sp >= 0.f ? e * w : w) + inv_nf * rcp_approx(R);
        ns = fminf(sp - G * rcp_approx(dG), cap);
      } else {
        ns = 0.5f * (sp + nClf);
      }
    }
    const float step = ns - sp;
    sp = ns;
    // Newton on G converges quadratically with |G''/2G'| <= ~1/4 once the
    // root is in the left half, so a step of 4e-3 leaves an error of ~4e-6
    // (and the fp64 polish squares it again; its residual check guards the
    // rest): exit one iteration earlier than waiting for a 1e-5 step.  The
    // tail contraction converges linearly and keeps the 1e-5 test.
#ifndef SYSCD_NEWTON_EXIT
#define SYSCD_NEWTON_EXIT 4e-3f
#endif
#ifndef SYSCD_TAIL_CONTRACTION
    if (fabsf(step) <= SYSCD_NEWTON_EXIT * fmaxf(1.f, fabsf(sp))) {
#else
    if (fabsf(step) <= (tail ? 1e-5f : 4e-3f) * fmaxf(1.f, fabsf(sp))) {
#endif
      conv = true;
      break;
    }
  }
#ifdef SYSCD_NEWTON_HIST
  atomicAdd(&g_newton_hist[tail ? 1 : 0][conv ? its : 9], 1ull);
#endif
  const double s = left ? (double)sp : -(double)sp;
  if (!conv || !isfinite(s)) return false;
  const double t = sigmoid_fast(s);
  const double h = lin + aq * (t - alpha) + s * inv_n;
  const double dh = aq * t * (1.0 - t) + inv_n;
  if (!(fabs(h) <= 1e-4 * dh * fmax(1.0, fabs(s)))) {
#ifdef SYSCD_NEWTON_HIST
    atomicAdd(&g_newton_hist[tail ? 1 : 0][10], 1ull);
#endif
    return false;
  }
  const double ds = -h * (double)rcp_approx((float)dh);
  *s_out = s + ds;
  // sigma(s + ds) to first order: the polish step is ~1e-5 (the fp32 loop's
  // exit), so the dropped t (1-t)(1-2t) ds^2 / 2 is below fp32 resolution,
  // and no second sigmoid evaluation sits on the chain
  *alpha_out = t + t * (1.0 - t) * ds;
  return true;
}

// Root of h(s) = lin + aq (sigma(s) - alpha) + s/n in log-odds s (the oracle's
// logistic_dual_newton, oracle/objectives.py).  logistic_dual_fast handles
// the common case in ~3 steps; anything it does not certify goes through a
// bracketed Newton + bisection in fp64 from logit(alpha), with the sigmoid /
// logit evaluated by fp32 SFU intrinsics.  The result is stored as fp32
// alpha = sigma(s) and sigma' <= 1/4, so the iteration stops at
// |ds| <= 1e-9 max(1,|s|) (the oracle uses 1e-13 with fp64 transcendentals).
// inv_n = 1/n precomputed by the caller (a loop-invariant fp64 division the
// chain should not carry)
__device__ __forceinline__ double logistic_dual_solve(double lin, double aq, double alpha,
                                                      double n, double inv_n) {
  double s = 0.0, an = 0.0;
  if (aq > 0.0 && logistic_dual_fast(lin, aq, alpha, n, inv_n, &s, &an)) return an;
  double lo = -n * (lin + aq * (1.0 - alpha)) - 1.0;
  double hi = n * (aq * alpha - lin) + 1.0;
  s = 0.0;
  if (alpha > 0.0 && alpha < 1.0) {
    const float af = (float)alpha;
    s = (double)(__logf(af) - __logf(1.f - af));
  }
  s = fmin(fmax(s, lo), hi);
  for (int it = 0; it < 100; ++it) {
    const double t = sigmoid_fast(s);
    const double h = lin + aq * (t - alpha) + s * inv_n;
    if (h > 0.0) {
      hi = s;
    } else if (h < 0.0) {
      lo = s;
    } else {
      break;
    }
    const double dh = aq * t * (1.0 - t) + inv_n;
    double ns = s - h / dh;
    if (!(lo < ns && ns < hi)) ns = 0.5 * (lo + hi);
    const double step = ns - s;
    s = ns;
    if (fabs(step) <= 1e-9 * fmax(1.0, fabs(s))) break;
  }
  return sigmoid_fast(s);
}

__device__ __forceinline__ double coord_step(int kind, double lin, double a, double q, double lam,
                                             double alpha, double n) {
  switch (kind) {
    case SYSCD_RIDGE:
    case SYSCD_LOGISTIC:
      return alpha - (lin + lam * alpha) / (a * q + lam);
    case SYSCD_LASSO: {
      double aq = a * q;
      if (aq <= 0.0) return 0.0;
      double z = alpha - lin / aq;
      double m = fabs(z) - lam / aq;
      return m > 0.0 ? copysign(m, z) : 0.0;
    }
    case SYSCD_SVM_DUAL: {
      double aq = a * q;
      if (aq <= 0.0) return 1.0;
      double z = alpha - (lin - 1.0 / n) / aq;
      return fmin(fmax(z, 0.0), 1.0);
    }
    default:  // SYSCD_LOGISTIC_DUAL
      return logistic_dual_solve(lin, a * q, alpha, n, 1.0 / n);
  }
}

// fp32 closed-form steps (ridge / primal-logistic surrogate / lasso / svm):
// the inputs are fp32, so IEEE fp32 division keeps the step within an ulp of
// the fp64 evaluation while staying off the fp64 pipe.
__device__ __forceinline__ float coord_step_f(int kind, float lin, float a, float q, float lam,
                                             float alpha, float inv_n) {
  const float aq = a * q;
  switch (kind) {
    case SYSCD_RIDGE:
    case SYSCD_LOGISTIC:
      return alpha - (lin + lam * alpha) * __frcp_rn(aq + lam);
    case SYSCD_LASSO: {
      if (aq <= 0.f) return 0.f;
      const float r = __frcp_rn(aq);
      const float z = fmaf(-lin, r, alpha);
      const float m = fmaf(-lam, r, fabsf(z));
      return m > 0.f ? copysignf(m, z) : 0.f;
    }
    default: {  // SVM dual
      if (aq <= 0.f) return 1.f;
      const float z = fmaf(-(lin - inv_n), __frcp_rn(aq), alpha);
      return fminf(fmaxf(z, 0.f), 1.f);
    }
  }
}

// The same steps with the column's reciprocal precomputed off the chain
// (step_inv): bitwise equal to coord_step_f.  inv < 0 marks aq <= 0 for the
// Lasso / SVM rows.
__device__ __forceinline__ float step_inv(int kind, float a, float q, float lam) {
  const float aq = a * q;
  if (kind == SYSCD_RIDGE || kind == SYSCD_LOGISTIC) return __frcp_rn(aq + lam);
  return aq > 0.f ? __frcp_rn(aq) : -1.f;
}

__device__ __forceinline__ float coord_step_fr(int kind, float lin, float inv, float lam,
                                               float alpha, float inv_n) {
  switch (kind) {
    case SYSCD_RIDGE:
    case SYSCD_LOGISTIC:
      return alpha - (lin + lam * alpha) * inv;
    case SYSCD_LASSO: {
      if (inv < 0.f) return 0.f;
      const float z = fmaf(-lin, inv, alpha);
      const float m = fmaf(-lam, inv, fabsf(z));
      return m > 0.f ? copysignf(m, z) : 0.f;
    }
    default: {  // SVM dual
      if (inv < 0.f) return 1.f;
      const float z = fmaf(-(lin - inv_n), inv, alpha);
      return fminf(fmaxf(z, 0.f), 1.f);
    }
  }
}

// fire-and-forget fp32 add; no "memory" clobber so independent loads (e.g.
// read-only u in the partition flush) may be scheduled across it
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v));
}

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef SYSCD_WAIT_HINT
  // suspend-time hint: the warp sleeps in the barrier instead of re-issuing
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity), "r"((uint32_t)SYSCD_WAIT_HINT)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
#endif
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAITC_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> this CTA's shared memory, completion on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t cluster_map(uint32_t local_smem_addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(local_smem_addr), "r"(rank));
  return out;
}

// Remote 4-byte store into a peer CTA's shared memory, signalling the peer's
// mbarrier with complete_tx(4).
__device__ __forceinline__ void st_async_f32(uint32_t remote_addr, float v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                   remote_addr),
               "r"(__float_as_uint(v)), "r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Worker g of G takes partitions [p_lo, p_hi): contiguous ranges whose
// boundaries are the partition starts nearest to g*total/G updates, so equal
// partitions split evenly and no worker is left idle while another holds two.
__device__ __forceinline__ int64_t nearest_part_start(const int64_t* wp, int n_parts, int64_t t) {
  int lo = 0, hi = n_parts + 1;  // first index with wp[idx] >= t
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (wp[mid] < t) {
      lo = mid + 1;
    } else {
      hi = mid;
    }
  }
  if (lo > n_parts) lo = n_parts;
  if (lo > 0 && t - wp[lo - 1] < wp[lo] - t) --lo;
  return lo;
}

// The same split on a cost that also charges each partition a fixed amount
// (its replica flush): cost(p) = 100 wp[p] + fc100 p, with fc100 the flush
// cost in hundredths of an update.  Still a static function of the plan, so
// the partition -> worker assignment (and the summation order) is
// deterministic.
__device__ __forceinline__ int64_t nearest_cost_start(const int64_t* wp, int n_parts, int fc100,
                                                      int64_t t) {
  auto cost = [&](int i) { return 100 * wp[i] + (int64_t)fc100 * i; };
  int lo = 0, hi = n_parts + 1;  // first index with cost >= t
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cost(mid) < t) {
      lo = mid + 1;
    } else {
      hi = mid;
    }
  }
  if (lo > n_parts) lo = n_parts;
  if (lo > 0 && t - cost(lo - 1) < cost(lo) - t) --lo;
  return lo;
}

__device__ __forceinline__ void worker_parts_cost(const int64_t* wp, int n_parts, int G, int g,
                                                  int fc100, int64_t* p_lo, int64_t* p_hi) {
  const int64_t total = 100 * wp[n_parts] + (int64_t)fc100 * n_parts;
  *p_lo = g == 0 ? 0 : nearest_cost_start(wp, n_parts, fc100, (int64_t)((__int128)total * g / G));
  *p_hi = g == G - 1 ? n_parts
                     : nearest_cost_start(wp, n_parts, fc100,
                                          (int64_t)((__int128)total * (g + 1) / G));
}

__device__ __forceinline__ void worker_parts(const int64_t* wp, int n_parts, int G, int g,
                                             int64_t* p_lo, int64_t* p_hi) {
  const int64_t total = wp[n_parts];
  *p_lo = g == 0 ? 0 : nearest_part_start(wp, n_parts, (int64_t)((__int128)total * g / G));
  *p_hi = g == G - 1 ? n_parts
                     : nearest_part_start(wp, n_parts, (int64_t)((__int128)total * (g + 1) / G));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace syscd

#define SYSCD_CUDA_TRY(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) {                                   \
      syscd::set_error("%s: %s", #expr, cudaGetErrorString(_e)); \
      return SYSCD_ECUDA;                                      \
    }                                                          \
  } while (0)

namespace syscd {
void set_error(const char* fmt, ...);
}
