// Sparse (CSC) SySCD round: the reference's sparse col_dot / col_axpy
// (dataset.py:77-78, 90-91) inside _surrogate_thread_round
// (solvers.py:289-334).
//
// B200 mapping: one warp is one worker; a worker runs whole partitions in
// sequence (contiguous, update-balanced ranges like the dense kernel).  The
// private replica dv of the running partition is a dense fp32 d-vector in
// HBM/L2 that is all-zero between partitions: only the rows the partition's
// columns touch are ever non-zero, and the flush re-walks those columns,
// zeroes it again; every update also adds delta*x_j into the node sum
// `delta_v` with a fire-and-forget red.global.add.  Work and traffic are therefore proportional to nnz,
// never to workers x d.  Per update, lanes own nonzeros: gather u[i] and
// dv[i], warp-reduce x.(u + a dv), fp64 step, scatter dv[i] += delta x_i
// (rows of one column are distinct, so the scatter is conflict-free).
//
// The replica sum uses fp32 atomics, so the summation order across workers is
// not fixed: unlike the dense path this kernel is deterministic only up to
// fp32 rounding of that sum (documented in DESIGN.md).
#include <algorithm>

#include "common.cuh"

namespace syscd {

struct SparseArgs {
  int64_t d;
  const int64_t* cp;
  const int32_t* ri;
  const float* vals;
  const float* sq;
  float* alpha;
  const float* u;
  const int32_t* seq;
  const int64_t* wp;
  int32_t n_parts;
  float a;
  float lam_f, inv_n_f;
  double a_d, lam, n_coords;
  int32_t kind, iid;
  float* dv_work;
  float* delta_v;
  int32_t* status;
};

__device__ __forceinline__ int64_t lb_i64(const int64_t* a, int n, int64_t key) {
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

__global__ void __launch_bounds__(256) k_sparse_epoch(SparseArgs A) {
  const int lane = threadIdx.x & 31;
  const int W = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  const int g = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int64_t total = A.wp[A.n_parts];
  const int64_t t_lo = (int64_t)((__int128)total * g / W);
  const int64_t t_hi = (int64_t)((__int128)total * (g + 1) / W);
  const int64_t p_lo = g == 0 ? 0 : lb_i64(A.wp, A.n_parts + 1, t_lo);
  const int64_t p_hi = g == W - 1 ? A.n_parts : lb_i64(A.wp, A.n_parts + 1, t_hi);
  float* dv = A.dv_work + (int64_t)g * A.d;
  for (int64_t p = p_lo; p < p_hi; ++p) {
    const int64_t s0 = A.wp[p], s1 = A.wp[p + 1];
    if (s1 == s0) continue;
    // software pipeline: the next update's column (<= 32 nonzeros per lane
    // pass) and scalars are loaded while the current one is processed
    int jn = A.seq[s0];
    int64_t en0 = A.cp[jn], en1 = A.cp[jn + 1];
    int rn = en0 + lane < en1 ? A.ri[en0 + lane] : 0;
    float vn = en0 + lane < en1 ? A.vals[en0 + lane] : 0.f;
    float an = A.iid ? 0.f : A.alpha[jn];
    float qn = __ldg(A.sq + jn);
    for (int64_t s = s0; s < s1; ++s) {
      const int j = jn;
      const int64_t e0 = en0, e1 = en1;
      const int r_first = rn;
      const float v_first = vn;
      float aj = an;
      const float qj = qn;
      if (s + 1 < s1) {
        jn = A.seq[s + 1];
        en0 = A.cp[jn];
        en1 = A.cp[jn + 1];
        rn = en0 + lane < en1 ? A.ri[en0 + lane] : 0;
        vn = en0 + lane < en1 ? A.vals[en0 + lane] : 0.f;
        if (!A.iid) an = A.alpha[jn];
        qn = __ldg(A.sq + jn);
      }
      float acc = 0.f;
      if (e0 + lane < e1) acc = v_first * fmaf(A.a, dv[r_first], A.u[r_first]);
      for (int64_t e = e0 + 32 + lane; e < e1; e += 32) {
        const int i = A.ri[e];
        acc = fmaf(A.vals[e], fmaf(A.a, dv[i], A.u[i]), acc);
      }
      acc = warp_sum(acc);
      if (A.iid) aj = *(volatile float*)(A.alpha + j);
      float anew;
      if (A.kind == SYSCD_LOGISTIC_DUAL) {
        anew = (float)coord_step(A.kind, (double)acc, A.a_d, (double)qj, A.lam, (double)aj,
                                 A.n_coords);
      } else {
        anew = coord_step_f(A.kind, acc, A.a, qj, A.lam_f, aj, A.inv_n_f);
      }
      float delta = 0.f;
      if (isfinite(anew)) {
        delta = anew - aj;
        if (lane == 0) A.alpha[j] = anew;
      } else if (lane == 0) {
        atomicOr(A.status, SYSCD_ENONFINITE);
      }
      // private replica for the partition's own dots, plus a fire-and-forget
      // contribution to the node sum (no end-of-partition gather pass)
      if (delta != 0.f) {
        if (e0 + lane < e1) {
          const float c = delta * v_first;
          dv[r_first] += c;
          red_add_f32(A.delta_v + r_first, c);
        }
        for (int64_t e = e0 + 32 + lane; e < e1; e += 32) {
          const int i = A.ri[e];
          const float c = delta * A.vals[e];
          dv[i] += c;
          red_add_f32(A.delta_v + i, c);
        }
      }
      __syncwarp();
    }
    // restore the all-zero replica: lanes walk different columns in parallel
    // (a row shared by two columns is simply zeroed twice)
    for (int64_t s = s0 + lane; s < s1; s += 32) {
      const int j = A.seq[s];
      const int64_t c0 = A.cp[j], c1 = A.cp[j + 1];
      for (int64_t e = c0; e < c1; ++e) dv[A.ri[e]] = 0.f;
    }
    __syncwarp();
  }
}

static int sparse_workers(int32_t n_parts) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int w = std::max(1, std::min((int)n_parts, sms * 16));
  return w > 8 ? w / 8 * 8 : w;
}

}  // namespace syscd

using namespace syscd;

extern "C" int syscd_sparse_epoch_workers(int64_t d, int32_t n_parts, int32_t* n_workers) {
  if (d < 1 || n_parts < 1 || !n_workers) {
    set_error("syscd_sparse_epoch_workers: invalid arguments");
    return SYSCD_EINVAL;
  }
  *n_workers = sparse_workers(n_parts);
  return SYSCD_OK;
}

extern "C" int syscd_sparse_epoch(const syscd_sparse_epoch_args* e, void* stream) {
  if (!e || !e->col_ptr || !e->row_idx || !e->vals || !e->sq || !e->alpha || !e->u || !e->seq ||
      !e->work_prefix || !e->dv_work || !e->delta_v || !e->status || e->d < 1 ||
      e->n_parts < 1 || e->n_workers < 1 || !(e->a > 0.0) || !(e->lam > 0.0)) {
    set_error("syscd_sparse_epoch: invalid arguments");
    return SYSCD_EINVAL;
  }
  const int W = e->n_workers;
  SparseArgs A;
  A.d = e->d;
  A.cp = e->col_ptr;
  A.ri = e->row_idx;
  A.vals = e->vals;
  A.sq = e->sq;
  A.alpha = e->alpha;
  A.u = e->u;
  A.seq = e->seq;
  A.wp = e->work_prefix;
  A.n_parts = e->n_parts;
  A.a = (float)e->a;
  A.a_d = e->a;
  A.lam_f = (float)e->lam;
  A.inv_n_f = (float)(1.0 / e->n_coords);
  A.lam = e->lam;
  A.n_coords = e->n_coords;
  A.kind = e->kind;
  A.iid = e->iid;
  A.dv_work = e->dv_work;
  A.delta_v = e->delta_v;
  A.status = e->status;
  cudaStream_t s = (cudaStream_t)stream;
  SYSCD_CUDA_TRY(cudaMemsetAsync(e->delta_v, 0, e->d * sizeof(float), s));
  // exactly W warps: blocks of 32*W threads when W is small, else 256-thread blocks
  if (W <= 8) {
    k_sparse_epoch<<<1, 32 * W, 0, s>>>(A);
  } else {
    if (W % 8 != 0) {
      set_error("syscd_sparse_epoch: n_workers must be <= 8 or a multiple of 8");
      return SYSCD_EINVAL;
    }
    k_sparse_epoch<<<W / 8, 256, 0, s>>>(A);
  }
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}
