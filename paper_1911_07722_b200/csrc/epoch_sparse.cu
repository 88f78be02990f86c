// Sparse (CSC) SySCD round: the reference's sparse col_dot / col_axpy
// (dataset.py:77-78, 90-91) inside _surrogate_thread_round
// (solvers.py:289-334).
//
// B200 mapping.  One warp is one worker; a worker runs whole partitions in
// sequence (contiguous, update-balanced ranges like the dense kernels).  The
// private replica dv of the running partition is a d-vector of tagged 64-bit
// words in HBM, (tag << 32 | fp32): a word whose tag is not the running
// partition's reads as zero, so a new partition starts from an all-zero
// replica without any re-zeroing pass.
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
  unsigned long long* dv_work;  // tagged replicas (see syscd_b200.h)
  float* delta_v;
  int32_t* status;
  uint32_t tag0;
  unsigned long long* prof;  // debug: per-worker phase cycles (nullptr = off)
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
  float q_c[32];
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

// tagged replica word: (tag << 32) | fp32 bits; other tags read as zero
__device__ __forceinline__ float rep_load(const unsigned long long* dv, int64_t r, uint32_t tag) {
  const unsigned long long x = dv[r];
  return (uint32_t)(x >> 32) == tag ? __uint_as_float((uint32_t)x) : 0.f;
}

__device__ __forceinline__ void rep_store(unsigned long long* dv, int64_t r, uint32_t tag, float v) {
  dv[r] = ((unsigned long long)tag << 32) | __float_as_uint(v);
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
  unsigned long long* dv = A.dv_work + (int64_t)g * A.d;
  const float a = A.a;
  for (int k = lane; k < kTable; k += 32) S.key[k] = kEmpty;
  __syncwarp();
  unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
#define SPARSE_PHASE(i)                   \
  if (A.prof) {                           \
    const long long tn = clock64();       \
    ph[i] += (unsigned long long)(tn - tq); \
    tq = tn;                              \
  }

  for (int64_t p = p_lo; p < p_hi; ++p) {
    const int64_t s0 = A.wp[p], s1 = A.wp[p + 1];
    const uint32_t tag = A.tag0 + (uint32_t)p;
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
      SPARSE_PHASE(0);
      if (m == 0) {
        // ---- a single long column: lanes stream it (no table)
        const int jj = __shfl_sync(0xffffffffu, j, 0);
        const int64_t a0 = A.cp[jj], a1 = A.cp[jj + 1];
        float part = 0.f;
        for (int64_t e = a0 + lane; e < a1; e += 32) {
          const int i = A.ri[e];
          part = fmaf(A.vals[e], fmaf(a, rep_load(dv, i, tag), A.u[i]), part);
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
            rep_store(dv, i, tag, rep_load(dv, i, tag) + c);
            red_add_f32(A.delta_v + i, c);
          }
        }
        __syncwarp();
        c0 += 1;
        SPARSE_PHASE(7);
        continue;
      }
      // ---- stage the chunk's nonzeros and hash their rows (the table is
      // empty here: cleared once at start, used slots reset at writeback)
      if (lane < m) {
        S.col_j[lane] = j;
        S.col_pre[lane + 1] = pre;
        S.alpha_c[lane] = A.iid ? *(volatile float*)(A.alpha + j) : A.alpha[j];
        S.q_c[lane] = __ldg(A.sq + j);
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
      SPARSE_PHASE(1);
      // insert rows (each lane owns entries lane + 32k); owners of new slots
      // then gather b = u + a dv, 8 loads in flight per batch
      // 8 first-probe CASes in flight per lane, collisions then probe on
      unsigned own = 0;
      for (int k0 = 0; k0 < 32 && 32 * k0 < nz; k0 += 8) {
        int rq[8], pq[8];
        unsigned hq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = lane + 32 * (k0 + q);
          rq[q] = e < nz ? S.row[e] : kEmpty;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          hq[q] = hash_row(rq[q]);
          pq[q] = rq[q] != kEmpty ? atomicCAS(&S.key[hq[q]], kEmpty, rq[q]) : kEmpty;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = lane + 32 * (k0 + q);
          if (rq[q] == kEmpty) continue;
          unsigned h = hq[q];
          int prev = pq[q];
          while (prev != kEmpty && prev != rq[q]) {
            h = (h + 1) & (kTable - 1);
            prev = atomicCAS(&S.key[h], kEmpty, rq[q]);
          }
          if (prev == kEmpty) own |= 1u << (k0 + q);
          S.slot[e] = (short)h;
        }
      }
      SPARSE_PHASE(2);
      for (int k0 = 0; k0 < 32 && 32 * k0 < nz; k0 += 8) {
        float uu[8];
        unsigned long long dw[8];  // raw tagged words: decoded after all loads issue
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
            dw[q] = dv[r];
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (hh[q] >= 0) {
            const float dd = (uint32_t)(dw[q] >> 32) == tag ? __uint_as_float((uint32_t)dw[q]) : 0.f;
            S.dvold[hh[q]] = dd;
            S.b[hh[q]] = fmaf(a, dd, uu[q]);
            S.acc[hh[q]] = 0.f;
          }
        }
      }
      __syncwarp();
      SPARSE_PHASE(3);
      // ---- the chain, entirely in shared memory
      for (int t = 0; t < m; ++t) {
        const int b0 = S.col_pre[t], b1 = S.col_pre[t + 1];
        float part = 0.f;
        for (int e = b0 + lane; e < b1; e += 32) part = fmaf(S.val[e], S.b[S.slot[e]], part);
        const float lin = warp_sum(part);
        const int jt = S.col_j[t];
        const float aj = S.alpha_c[t];
        const float an = sparse_step(A, lin, aj, S.q_c[t]);
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
      SPARSE_PHASE(4);
      // ---- write back every distinct row once (by the lane that inserted
      // it) and release its slot
      for (unsigned o = own; o; o &= o - 1) {
        const int e = lane + 32 * (__ffs(o) - 1);
        const int h = S.slot[e];
        const int r = S.row[e];
        const float cv = S.acc[h];
        if (cv != 0.f) {
          rep_store(dv, r, tag, S.dvold[h] + cv);
          red_add_f32(A.delta_v + r, cv);
        }
        S.key[h] = kEmpty;
      }
      __syncwarp();
      c0 += m;
      SPARSE_PHASE(5);
    }
    SPARSE_PHASE(6);
  }
#undef SPARSE_PHASE
  if (A.prof && lane == 0)
    for (int i = 0; i < 8; ++i) A.prof[(int64_t)g * 8 + i] = ph[i];
}

static unsigned long long* g_sparse_prof = nullptr;

static int sparse_workers(int32_t n_parts) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, std::min((int)n_parts, sms * 16));
}

}  // namespace syscd

using namespace syscd;

// Debug hook (not part of the C-ABI contract): with a device buffer of
// n_workers * 8 uint64, the next sparse epochs record per-worker cycles spent
// in: chunk formation, column copy, hash insert, gather, chain, writeback,
// partition-end zeroing, long-column path.
extern "C" void syscd_debug_set_sparse_profile(void* device_buffer) {
  g_sparse_prof = (unsigned long long*)device_buffer;
}

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
  A.dv_work = (unsigned long long*)e->dv_work;
  A.tag0 = e->replica_tag;
  A.delta_v = e->delta_v;
  A.status = e->status;
  A.prof = g_sparse_prof;
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
