// Sparse (CSC) SySCD round: the reference's sparse col_dot / col_axpy
// (dataset.py:77-78, 90-91) inside _surrogate_thread_round
// (solvers.py:289-334).
//
// B200 mapping.  One warp is one worker; a worker runs whole partitions in
// sequence (contiguous, update-balanced ranges like the dense kernels).  The
// private replica dv of the running partition is a dense fp32 d-vector in HBM
// that is all-zero between partitions.
//
// The chain is processed in chunks of up to 32 consecutive updates holding at
// most kChunkNnz nonzeros.  The chunk's rows are hashed into a shared-memory
// table (one slot per distinct row) that holds b = u + a dv for that row and
// the chunk's accumulated replica change; every update then runs entirely in
// shared memory:
//     lin_t = sum_{e in col t} val_e * b[slot_e]        (lanes over nonzeros)
//     alpha_t <- step(lin_t)                             (fp64 for logistic dual)
//     b[slot_e] += a delta_t val_e ; acc[slot_e] += delta_t val_e
// which is exactly the reference's per-coordinate chain (rows shared by two
// columns of the chunk see each other's updates through the shared slot).  At
// the chunk end every distinct row is written back once: dv = dv_old + acc in
// the private replica and acc into the node sum (red.global.add).  Global
// round trips drop from ~3 per update to ~3 per chunk.  A column longer than
// the chunk capacity is processed on its own with lanes streaming it.
// At a partition end the replica's touched rows are re-zeroed (lanes walk
// different columns in parallel).
//
// The node sum uses fp32 atomics across workers, so this kernel is
// deterministic only up to that summation order (documented in DESIGN.md).
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

constexpr int kChunkNnz = 1024;  // nonzeros per chunk
constexpr int kTable = 2048;     // hash slots (>= 2 x kChunkNnz)
constexpr int kSparseWarps = 4;  // workers per block
constexpr int kEmpty = -1;

struct SparseWarpSmem {
  int key[kTable];
  float b[kTable];
  float acc[kTable];
  float dvold[kTable];
  short slot[kChunkNnz];
  float val[kChunkNnz];
  int row[kChunkNnz];
  float alpha_c[32];
  int col_j[32];
  int col_pre[33];
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

__device__ __forceinline__ unsigned hash_row(int r) {
  return ((unsigned)r * 2654435761u) >> (32 - 11);  // 11 bits = kTable
}

__device__ __forceinline__ float sparse_step(const SparseArgs& A, float lin, float aj, float qj) {
  if (A.kind == SYSCD_LOGISTIC_DUAL)
    return (float)coord_step(A.kind, (double)lin, A.a_d, (double)qj, A.lam, (double)aj,
                             A.n_coords);
  return coord_step_f(A.kind, lin, A.a, qj, A.lam_f, aj, A.inv_n_f);
}

__global__ void __launch_bounds__(32 * kSparseWarps) k_sparse_epoch(SparseArgs A, int W) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int g = blockIdx.x * kSparseWarps + wib;
  if (g >= W) return;
  SparseWarpSmem& S = reinterpret_cast<SparseWarpSmem*>(smem_raw)[wib];
  const int64_t total = A.wp[A.n_parts];
  const int64_t t_lo = (int64_t)((__int128)total * g / W);
  const int64_t t_hi = (int64_t)((__int128)total * (g + 1) / W);
  const int64_t p_lo = g == 0 ? 0 : lb_i64(A.wp, A.n_parts + 1, t_lo);
  const int64_t p_hi = g == W - 1 ? A.n_parts : lb_i64(A.wp, A.n_parts + 1, t_hi);
  float* dv = A.dv_work + (int64_t)g * A.d;
  const float a = A.a;
  for (int k = lane; k < kTable; k += 32) S.key[k] = kEmpty;
  __syncwarp();

  for (int64_t p = p_lo; p < p_hi; ++p) {
    const int64_t s0 = A.wp[p], s1 = A.wp[p + 1];
    int64_t c0 = s0;
    while (c0 < s1) {
      // ---- form the chunk: up to 32 columns with <= kChunkNnz nonzeros
      const int64_t sl = c0 + lane;
      int j = 0;
      int nnz = 0;
      int64_t e0 = 0;
      if (sl < s1) {
        j = A.seq[sl];
        e0 = A.cp[j];
        nnz = (int)(A.cp[j + 1] - e0);
      }
      int pre = nnz;  // inclusive scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += v;
      }
      const unsigned fits = __ballot_sync(0xffffffffu, sl < s1 && pre <= kChunkNnz);
      const int m = __popc(fits);  // fits is a prefix of lanes
      if (m == 0) {
        // ---- a single long column: lanes stream it (no table)
        const int jj = __shfl_sync(0xffffffffu, j, 0);
        const int64_t a0 = A.cp[jj], a1 = A.cp[jj + 1];
        float part = 0.f;
        for (int64_t e = a0 + lane; e < a1; e += 32) {
          const int i = A.ri[e];
          part = fmaf(A.vals[e], fmaf(a, dv[i], A.u[i]), part);
        }
        part = warp_sum(part);
        const float aj = A.iid ? *(volatile float*)(A.alpha + jj) : A.alpha[jj];
        const float an = sparse_step(A, part, aj, __ldg(A.sq + jj));
        float delta = 0.f;
        if (isfinite(an)) {
          delta = an - aj;
          if (lane == 0) A.alpha[jj] = an;
        } else if (lane == 0) {
          atomicOr(A.status, SYSCD_ENONFINITE);
        }
        if (delta != 0.f) {
          for (int64_t e = a0 + lane; e < a1; e += 32) {
            const int i = A.ri[e];
            const float c = delta * A.vals[e];
            dv[i] += c;
            red_add_f32(A.delta_v + i, c);
          }
        }
        __syncwarp();
        c0 += 1;
        continue;
      }
      // ---- stage the chunk's nonzeros and hash their rows (the table is
      // empty here: cleared once at start, used slots reset at writeback)
      if (lane < m) {
        S.col_j[lane] = j;
        S.col_pre[lane + 1] = pre;
        S.alpha_c[lane] = A.iid ? *(volatile float*)(A.alpha + j) : A.alpha[j];
      }
      if (lane == 0) S.col_pre[0] = 0;
      __syncwarp();
      const int nz = S.col_pre[m];
      // copy the chunk's nonzeros: all lanes on one column, 8 columns' loads
      // in flight before their shared-memory stores
      for (int t0 = 0; t0 < m; t0 += 8) {
        int rr[8][2];
        float vv[8][2];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int t = t0 + q;
          const int jt = __shfl_sync(0xffffffffu, j, t & 31);
          const int64_t et = __shfl_sync(0xffffffffu, e0, t & 31);
          const int nt = __shfl_sync(0xffffffffu, nnz, t & 31);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int k = lane + 32 * h2;
            if (t < m && k < nt) {
              rr[q][h2] = A.ri[et + k];
              vv[q][h2] = A.vals[et + k];
            }
          }
          (void)jt;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int t = t0 + q;
          const int nt = __shfl_sync(0xffffffffu, nnz, t & 31);
          const int bt = __shfl_sync(0xffffffffu, pre - nnz, t & 31);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int k = lane + 32 * h2;
            if (t < m && k < nt) {
              S.row[bt + k] = rr[q][h2];
              S.val[bt + k] = vv[q][h2];
            }
          }
        }
        // columns longer than 64 nonzeros: the rest, plainly
#pragma unroll 1
        for (int q = 0; q < 8; ++q) {
          const int t = t0 + q;
          const int nt = __shfl_sync(0xffffffffu, nnz, t & 31);
          const int64_t et = __shfl_sync(0xffffffffu, e0, t & 31);
          const int bt = __shfl_sync(0xffffffffu, pre - nnz, t & 31);
          if (t < m && nt > 64) {
            for (int k = 64 + lane; k < nt; k += 32) {
              S.row[bt + k] = A.ri[et + k];
              S.val[bt + k] = A.vals[et + k];
            }
          }
        }
      }
      __syncwarp();
      // insert rows (each lane owns entries lane + 32k); owners of new slots
      // then gather b = u + a dv, 8 loads in flight per batch
      unsigned own = 0;
      for (int k = 0; k < 32; ++k) {
        const int e = lane + 32 * k;
        if (e >= nz) break;
        const int r = S.row[e];
        unsigned h = hash_row(r);
        while (true) {
          const int prev = atomicCAS(&S.key[h], kEmpty, r);
          if (prev == kEmpty) {
            own |= 1u << k;
            break;
          }
          if (prev == r) break;
          h = (h + 1) & (kTable - 1);
        }
        S.slot[e] = (short)h;
      }
      for (int k0 = 0; k0 < 32 && 32 * k0 < nz; k0 += 8) {
        float uu[8], dd[8];
        int hh[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int k = k0 + q;
          hh[q] = -1;
          if ((own >> k) & 1u) {
            const int e = lane + 32 * k;
            const int r = S.row[e];
            hh[q] = S.slot[e];
            uu[q] = A.u[r];
            dd[q] = dv[r];
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (hh[q] >= 0) {
            S.dvold[hh[q]] = dd[q];
            S.b[hh[q]] = fmaf(a, dd[q], uu[q]);
            S.acc[hh[q]] = 0.f;
          }
        }
      }
      __syncwarp();
      // ---- the chain, entirely in shared memory
      for (int t = 0; t < m; ++t) {
        const int b0 = S.col_pre[t], b1 = S.col_pre[t + 1];
        float part = 0.f;
        for (int e = b0 + lane; e < b1; e += 32) part = fmaf(S.val[e], S.b[S.slot[e]], part);
        const float lin = warp_sum(part);
        const int jt = S.col_j[t];
        const float aj = S.alpha_c[t];
        const float an = sparse_step(A, lin, aj, __ldg(A.sq + jt));
        float delta = 0.f;
        if (isfinite(an)) {
          delta = an - aj;
        } else if (lane == 0) {
          atomicOr(A.status, SYSCD_ENONFINITE);
        }
        if (delta != 0.f) {
          for (int e = b0 + lane; e < b1; e += 32) {
            const int h = S.slot[e];
            const float c = delta * S.val[e];
            S.b[h] = fmaf(a, c, S.b[h]);
            S.acc[h] += c;
          }
        }
        // later occurrences of the same coordinate (iid) see its new value
        if (lane < m && lane > t && S.col_j[lane] == jt) S.alpha_c[lane] = aj + delta;
        // the last occurrence's value is the one that survives
        if (lane == 0 && isfinite(an)) A.alpha[jt] = aj + delta;
        __syncwarp();
      }
      // ---- write back every distinct row once (by the lane that inserted
      // it) and release its slot
      for (unsigned o = own; o; o &= o - 1) {
        const int e = lane + 32 * (__ffs(o) - 1);
        const int h = S.slot[e];
        const int r = S.row[e];
        const float c = S.acc[h];
        if (c != 0.f) {
          dv[r] = S.dvold[h] + c;
          red_add_f32(A.delta_v + r, c);
        }
        S.key[h] = kEmpty;
      }
      __syncwarp();
      c0 += m;
    }
    // restore the all-zero replica: lanes walk different columns in parallel
    // (a row shared by two columns is simply zeroed twice)
    for (int64_t s = s0 + lane; s < s1; s += 32) {
      const int jj = A.seq[s];
      const int64_t q0 = A.cp[jj], q1 = A.cp[jj + 1];
      for (int64_t e = q0; e < q1; ++e) dv[A.ri[e]] = 0.f;
    }
    __syncwarp();
  }
}

static int sparse_workers(int32_t n_parts) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, std::min((int)n_parts, sms * 16));
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
  const size_t smem = sizeof(SparseWarpSmem) * kSparseWarps;
  SYSCD_CUDA_TRY(
      cudaFuncSetAttribute(k_sparse_epoch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int blocks = (W + kSparseWarps - 1) / kSparseWarps;
  k_sparse_epoch<<<blocks, 32 * kSparseWarps, smem, s>>>(A, W);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}
