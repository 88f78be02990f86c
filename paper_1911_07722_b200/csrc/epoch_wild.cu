// Asynchronous ("wild") parallel SCD epoch: run_wild_parallel_scd
// (pkg/src/syscd/solvers.py:214-286).  P workers share one model alpha and one
// shared vector; worker w walks chunk w of np.array_split(perm, P) (:252-253)
// doing exact coordinate updates (exact_coordinate_update, objective.py:113-125)
// on the LIVE shared state and writes its axpy without synchronisation.
//
// B200 mapping.  The shared vector is v = v0 + dv: v0 (fp64) and u = grad f(v0)
// are fixed for the epoch, dv (fp32) is the live change that every worker reads
// through L2 (ld.global.cg: other SMs update it) and adds to with fire-and-forget
// red.global.add.  For the quadratic f of ridge / lasso / svm-dual /
// logistic-dual, grad f(v) = u + gamma dv exactly, so
//     lin_j = x_j . (u + gamma dv)
// and the exact update is the closed-form step with a = gamma.  (Primal
// logistic needs Newton on whole-column reductions; the host runs it through
// the exact-logistic kernel, chunks back to back, which is one valid
// interleaving of the wild schedule.)  Staleness is whatever the hardware
// interleaving gives, as in the reference's threads.
//
// Worker granularity: a CTA of 256 threads per worker for long dense columns,
// a warp per worker for short dense columns and for CSC columns.
#include "common.cuh"

namespace syscd {

struct WildArgs {
  int kind;
  int64_t d, lda;
  const float* A;
  const int64_t* cp;
  const int32_t* ri;
  const float* vals;
  const float* sq;
  float* alpha;
  const float* u;
  float* dv;
  const int32_t* perm;
  int64_t n;
  int32_t P;
  double gamma, lam, n_coords;
  int32_t* status;
};

constexpr int kWildCta = 256;
constexpr int kWildWarpsPerBlock = 4;
constexpr int64_t kWildWarpMaxD = 2048;

// np.array_split: the first n % P chunks hold one extra element
__device__ __forceinline__ void chunk_of(int64_t n, int P, int w, int64_t* lo, int64_t* hi) {
  const int64_t base = n / P, rem = n % P;
  *lo = (int64_t)w * base + (w < rem ? w : rem);
  *hi = *lo + base + (w < rem ? 1 : 0);
}

__device__ __forceinline__ bool wild_step(const WildArgs& W, int j, double lin, float* delta) {
  const float aj = W.alpha[j];
  const double an =
      coord_step(W.kind, lin, W.gamma, (double)__ldg(W.sq + j), W.lam, (double)aj, W.n_coords);
  const float anf = (float)an;
  if (!isfinite(anf)) return false;
  W.alpha[j] = anf;
  *delta = anf - aj;
  return true;
}

__global__ void __launch_bounds__(kWildCta) k_wild_dense_cta(WildArgs W) {
  __shared__ float red[kWildCta / 32];
  __shared__ float s_delta;
  __shared__ int s_ok;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t lo, hi;
  chunk_of(W.n, W.P, blockIdx.x, &lo, &hi);
  const float g = (float)W.gamma;
  for (int64_t s = lo; s < hi; ++s) {
    const int j = W.perm[s];
    const float* x = W.A + (int64_t)j * W.lda;
    float acc = 0.f;
    for (int64_t i = tid; i < W.d; i += kWildCta)
      acc = fmaf(__ldg(x + i), fmaf(g, __ldcg(W.dv + i), __ldg(W.u + i)), acc);
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      float lin = 0.f;
      for (int k = 0; k < kWildCta / 32; ++k) lin += red[k];
      float delta = 0.f;
      s_ok = wild_step(W, j, (double)lin, &delta);
      if (!s_ok) atomicOr(W.status, SYSCD_ENONFINITE);
      s_delta = delta;
    }
    __syncthreads();
    if (!s_ok) return;  // the reference's worker stops at NonFiniteUpdateError
    const float delta = s_delta;
    if (delta != 0.f)
      for (int64_t i = tid; i < W.d; i += kWildCta) red_add_f32(W.dv + i, delta * __ldg(x + i));
  }
}

__global__ void __launch_bounds__(32 * kWildWarpsPerBlock) k_wild_warp(WildArgs W) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * kWildWarpsPerBlock + (threadIdx.x >> 5);
  if (w >= W.P) return;
  int64_t lo, hi;
  chunk_of(W.n, W.P, w, &lo, &hi);
  const float g = (float)W.gamma;
  const bool dense = W.A != nullptr;
  for (int64_t s = lo; s < hi; ++s) {
    const int j = W.perm[s];
    const int64_t e0 = dense ? (int64_t)j * W.lda : W.cp[j];
    const int64_t e1 = dense ? e0 + W.d : W.cp[j + 1];
    float acc = 0.f;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int64_t i = dense ? e - e0 : (int64_t)__ldg(W.ri + e);
      const float xv = dense ? __ldg(W.A + e) : __ldg(W.vals + e);
      acc = fmaf(xv, fmaf(g, __ldcg(W.dv + i), __ldg(W.u + i)), acc);
    }
    const float lin = warp_sum(acc);
    float delta = 0.f;
    int ok = 1;
    if (lane == 0) {
      ok = wild_step(W, j, (double)lin, &delta);
      if (!ok) atomicOr(W.status, SYSCD_ENONFINITE);
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (!ok) return;
    delta = __shfl_sync(0xffffffffu, delta, 0);
    if (delta != 0.f) {
      for (int64_t e = e0 + lane; e < e1; e += 32) {
        const int64_t i = dense ? e - e0 : (int64_t)__ldg(W.ri + e);
        const float xv = dense ? __ldg(W.A + e) : __ldg(W.vals + e);
        red_add_f32(W.dv + i, delta * xv);
      }
    }
  }
}

}  // namespace syscd

using namespace syscd;

extern "C" int syscd_wild_epoch(const syscd_wild_epoch_args* e, void* stream) {
  if (!e || e->d < 1 || e->n < 0 || e->P < 1 || !e->sq || !e->alpha || !e->u || !e->dv ||
      !e->status || (e->n > 0 && !e->perm) ||
      (!e->A && (!e->col_ptr || !e->row_idx || !e->vals)) || !(e->gamma > 0.0) ||
      !(e->lam > 0.0) || e->kind == SYSCD_LOGISTIC || e->kind < 0 || e->kind > 4) {
    set_error("syscd_wild_epoch: invalid arguments");
    return SYSCD_EINVAL;
  }
  if (e->n == 0) return SYSCD_OK;
  WildArgs W;
  W.kind = e->kind;
  W.d = e->d;
  W.lda = e->lda;
  W.A = e->A;
  W.cp = e->col_ptr;
  W.ri = e->row_idx;
  W.vals = e->vals;
  W.sq = e->sq;
  W.alpha = e->alpha;
  W.u = e->u;
  W.dv = e->dv;
  W.perm = e->perm;
  W.n = e->n;
  W.P = e->P;
  W.gamma = e->gamma;
  W.lam = e->lam;
  W.n_coords = e->n_coords;
  W.status = e->status;
  cudaStream_t s = (cudaStream_t)stream;
  if (e->A && e->d > kWildWarpMaxD) {
    k_wild_dense_cta<<<e->P, kWildCta, 0, s>>>(W);
  } else {
    const int blocks = (e->P + kWildWarpsPerBlock - 1) / kWildWarpsPerBlock;
    k_wild_warp<<<blocks, 32 * kWildWarpsPerBlock, 0, s>>>(W);
  }
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}
