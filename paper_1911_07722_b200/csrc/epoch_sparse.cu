// Sparse (CSC) SySCD round: the reference's sparse col_dot / col_axpy
// (dataset.py:77-78, 90-91) inside _surrogate_thread_round
// (solvers.py:289-334).
//
// B200 mapping.  A worker (one 64-thread block = a consumer warp and a
// producer warp) runs whole partitions in sequence (contiguous,
// update-balanced ranges like the dense kernels).  The private replica dv of
// the running partition is a d-vector of tagged 64-bit words in HBM,
// (tag << 32 | fp32): a word whose tag is not the running partition's reads as
// zero, so a new partition starts from an all-zero replica without any
// re-zeroing pass.
//
// The chain is cut into chunks of up to 32 consecutive updates holding at most
// kPcNnz nonzeros.  The producer stages a chunk into one of two shared-memory
// buffers: the columns' rows and values, a hash table with one slot per
// distinct row (linear probing, the inserting lane owns the slot), and per
// slot b = u + a dv gathered once.  The consumer then runs the chain entirely
// in shared memory:
//     lin_t = sum_{e in col t} val_e * b[slot_e]        (lanes over nonzeros)
//     alpha_t <- step(lin_t)
//     b[slot_e] += a delta_t val_e ; acc[slot_e] += delta_t val_e
// which is exactly the reference's per-coordinate chain (rows shared by two
// columns of the chunk see each other's updates through the shared slot).
// While chunk k's chain runs, the producer writes back chunk k-1's buffer
// (dv = dv_old + acc per distinct row, acc into the node sum with
// red.global.add) and stages chunk k+1.  Chunk k+1 was gathered before chunk
// k's updates reached memory, so after its chain the consumer patches chunk
// k+1's copy of every row chunk k changed (a hash probe; both tables use the
// same hash, so most probes hit the first slot).  A column longer than the
// chunk capacity is streamed by the consumer on its own.
//
// Node sum.  When every partition has its own worker (n_parts <= resident
// workers, e.g. config 4: 512 partitions), worker g runs exactly partition g
// and its tagged replica words ARE that partition's dv at the end of the
// round; k_sparse_node_sum then adds them in ascending partition order
// (fixed order, bitwise reproducible; the reference's reduce_replicas,
// solvers.py:112-125,393).  With more partitions than workers a worker's
// replica region is reused, so the node sum falls back to fp32 atomics
// (deterministic only up to their order).
#include <stdlib.h>

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
  double a_d, lam, n_coords, inv_n_d;
  int32_t kind, iid;
  unsigned long long* dv_work;  // tagged replicas (see syscd_b200.h)
  float* delta_v;
  int32_t* status;
  uint32_t tag0;
  int32_t one_part;  // worker g runs partition g; node sum reduced after the kernel
  int32_t hot;       // rows [0, hot) of the replica stay in shared memory (0: none)
  unsigned long long* prof;  // debug: per-worker phase cycles (nullptr = off)
};

constexpr int kEmpty = -1;

// tagged replica word: (tag << 32) | fp32 bits; other tags read as zero
__device__ __forceinline__ float rep_load(const unsigned long long* dv, int64_t r, uint32_t tag) {
  const unsigned long long x = dv[r];
  return (uint32_t)(x >> 32) == tag ? __uint_as_float((uint32_t)x) : 0.f;
}

__device__ __forceinline__ float rep_load_cg(const unsigned long long* dv, int64_t r, uint32_t tag) {
  const unsigned long long x = __ldcg(dv + r);
  return (uint32_t)(x >> 32) == tag ? __uint_as_float((uint32_t)x) : 0.f;
}

__device__ __forceinline__ void rep_store(unsigned long long* dv, int64_t r, uint32_t tag, float v) {
  dv[r] = ((unsigned long long)tag << 32) | __float_as_uint(v);
}

// KIND is the kernel instance's step (SYSCD_RIDGE also serves the primal
// logistic surrogate): no runtime switch and no fp64 Newton code in the
// closed-form instances' chain.
template <int KIND>
__device__ __forceinline__ float sparse_step(const SparseArgs& A, float lin, float aj, float qj) {
  if (KIND == SYSCD_LOGISTIC_DUAL)
    return (float)logistic_dual_solve((double)lin, A.a_d * (double)qj, (double)aj, A.n_coords,
                                      A.inv_n_d);
  return coord_step_f(KIND, lin, A.a, qj, A.lam_f, aj, A.inv_n_f);
}

constexpr int kPcNnz = 512;
constexpr int kPcTable = 1024;
constexpr int kPcFilterWords = 128;  // 4096-bit membership filter of a chunk's rows

struct PcBuf {
  int key[kPcTable];
  float b[kPcTable];
  float acc[kPcTable];
  float dvold[kPcTable];
  short slot[kPcNnz];
  short uniq[kPcNnz];  // the chunk's distinct slots
  unsigned filt[kPcFilterWords];  // one bit per row hash: which rows this chunk holds
  float val[kPcNnz];
  int row[kPcNnz];
  float alpha_c[32];
  float q_c[32];
  int col_j[32];
  int col_pre[33];
  int m;  // columns; 0 = one long column (col_j[0]); -1 = end of the worker's work
  int n_uniq;
  uint32_t tag;
};

struct PcSmem {
  PcBuf buf[2];
  uint64_t full[2];
  uint64_t empty[2];
};

__device__ __forceinline__ unsigned pc_hash(int r) {
  return ((unsigned)r * 2654435761u) >> (32 - 10);  // 10 bits = kPcTable
}

__device__ __forceinline__ unsigned pc_fhash(int r) {
  return ((unsigned)r * 0x85ebca6bu) >> (32 - 12);  // 12 bits = 32 * kPcFilterWords
}

__device__ __forceinline__ int pc_find(const PcBuf& T, int r) {
  unsigned h = pc_hash(r);
  int k;
  while ((k = T.key[h]) != kEmpty) {
    if (k == r) return (int)h;
    h = (h + 1) & (kPcTable - 1);
  }
  return -1;
}

// Stage the chunk starting at c0 of the partition into B.
// Slots: a nonzero's slot is its row r when r < H (the worker's resident
// hot rows, shared by both buffers) and H + h for hash slot h otherwise.
__device__ __forceinline__ void pc_produce(const SparseArgs& A, PcBuf& B, int lane, int64_t c0,
                                           int64_t s1, uint32_t tag,
                                           const unsigned long long* dv, int* m_out) {
  const int H = A.hot;
  const float a = A.a;
  const int64_t sl = c0 + lane;
  int j = 0, nnz = 0;
  int64_t e0 = 0;
  if (sl < s1) {
    j = A.seq[sl];
    e0 = A.cp[j];
    nnz = (int)(A.cp[j + 1] - e0);
  }
  int pre = nnz;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre += v;
  }
  const unsigned fits = __ballot_sync(0xffffffffu, sl < s1 && pre <= kPcNnz);
  const int m = __popc(fits);
  *m_out = m;
  if (lane == 0) B.tag = tag;
  if (m == 0) {  // one long column: the consumer streams it from global memory
    if (lane == 0) {
      B.m = 0;
      B.col_j[0] = j;
    }
    return;
  }
  if (lane < m) {
    B.col_j[lane] = j;
    B.col_pre[lane + 1] = pre;
    if (!A.iid) B.alpha_c[lane] = A.alpha[j];
    B.q_c[lane] = __ldg(A.sq + j);
  }
  if (lane == 0) {
    B.col_pre[0] = 0;
    B.m = m;
  }
  for (int w = lane; w < kPcFilterWords; w += 32) B.filt[w] = 0u;

  const int nz = __shfl_sync(0xffffffffu, pre, m - 1);
  // copy: all lanes on one column, 8 columns' loads in flight
  for (int t0 = 0; t0 < m; t0 += 8) {
    int rr[8][2];
    float vv[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int t = t0 + q;
      const int64_t et = __shfl_sync(0xffffffffu, e0, t & 31);
      const int nt = __shfl_sync(0xffffffffu, nnz, t & 31);
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int k = lane + 32 * h2;
        if (t < m && k < nt) {
          rr[q][h2] = __ldg(A.ri + et + k);
          vv[q][h2] = __ldg(A.vals + et + k);
        }
      }
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
          B.row[bt + k] = rr[q][h2];
          B.val[bt + k] = vv[q][h2];
        }
      }
    }
#pragma unroll 1
    for (int q = 0; q < 8; ++q) {
      const int t = t0 + q;
      const int nt = __shfl_sync(0xffffffffu, nnz, t & 31);
      const int64_t et = __shfl_sync(0xffffffffu, e0, t & 31);
      const int bt = __shfl_sync(0xffffffffu, pre - nnz, t & 31);
      if (t < m && nt > 64)
        for (int k = 64 + lane; k < nt; k += 32) {
          B.row[bt + k] = __ldg(A.ri + et + k);
          B.val[bt + k] = __ldg(A.vals + et + k);
        }
    }
  }
  __syncwarp();
  // insert: 8 first-probe CASes in flight per lane; the inserting lane owns
  // the slot
  unsigned own = 0;
  for (int k0 = 0; k0 < kPcNnz / 32 && 32 * k0 < nz; k0 += 8) {
    int rq[8], pq[8];
    unsigned hq[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = lane + 32 * (k0 + q);
      rq[q] = e < nz ? B.row[e] : kEmpty;
      if (rq[q] != kEmpty && rq[q] < H) {  // resident hot row: no table entry
        B.slot[e] = (short)rq[q];
        rq[q] = kEmpty;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      hq[q] = pc_hash(rq[q]);
      pq[q] = rq[q] != kEmpty ? atomicCAS(&B.key[hq[q]], kEmpty, rq[q]) : kEmpty;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = lane + 32 * (k0 + q);
      if (rq[q] == kEmpty) continue;
      unsigned h = hq[q];
      int prev = pq[q];
      while (prev != kEmpty && prev != rq[q]) {
        h = (h + 1) & (kPcTable - 1);
        prev = atomicCAS(&B.key[h], kEmpty, rq[q]);
      }
      if (prev == kEmpty) {
        own |= 1u << (k0 + q);
        const unsigned fh = pc_fhash(rq[q]);
        atomicOr(&B.filt[fh >> 5], 1u << (fh & 31));
      }
      B.slot[e] = (short)(H + (int)h);
    }
  }
  // distinct-slot list (warp prefix over the owners' counts)
  const int cnt = __popc(own);
  int base = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, base, o);
    if (lane >= o) base += v;
  }
  if (lane == 31) B.n_uniq = base;
  base -= cnt;
  // gather u and the replica for owned slots (8 loads in flight; the
  // replica through L2: the consumer warp writes it)
  for (int k0 = 0; k0 < kPcNnz / 32 && 32 * k0 < nz; k0 += 8) {
    float uu[8];
    unsigned long long dw[8];
    int hh[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = k0 + q;
      hh[q] = -1;
      if ((own >> k) & 1u) {
        const int e = lane + 32 * k;
        const int r = B.row[e];
        hh[q] = B.slot[e] - H;
        uu[q] = __ldg(A.u + r);
        dw[q] = __ldcg(dv + r);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (hh[q] >= 0) {
        const float dd =
            (uint32_t)(dw[q] >> 32) == tag ? __uint_as_float((uint32_t)dw[q]) : 0.f;
        B.dvold[hh[q]] = dd;
        B.b[hh[q]] = fmaf(a, dd, uu[q]);
        B.acc[hh[q]] = 0.f;
        B.uniq[base++] = (short)hh[q];

      }
    }
  }
}

// patch the next buffer's copy of row r (gathered before this writeback)
__device__ __forceinline__ void pc_patch(PcBuf& N, int r, float nv, float a) {
  unsigned h = pc_hash(r);
  int k;
  while ((k = N.key[h]) != kEmpty) {
    if (k == r) {
      N.b[h] = fmaf(a, nv - N.dvold[h], N.b[h]);
      N.dvold[h] = nv;
      return;
    }
    h = (h + 1) & (kPcTable - 1);
  }
}

template <int KIND>
__global__ void __launch_bounds__(64) k_sparse_epoch(SparseArgs A, int W) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PcSmem& S = *reinterpret_cast<PcSmem*>(smem_raw);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int g = blockIdx.x;
  if (g >= W) return;
  for (int k = threadIdx.x; k < kPcTable; k += 64) {
    S.buf[0].key[k] = kEmpty;
    S.buf[1].key[k] = kEmpty;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], 1);
      S.buf[i].m = -1;
      S.buf[i].tag = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();
  int64_t p_lo, p_hi;
  if (A.one_part) {
    p_lo = g;
    p_hi = g + 1;
  } else {
    worker_parts(A.wp, A.n_parts, W, g, &p_lo, &p_hi);
  }
  unsigned long long* dv = A.dv_work + (int64_t)g * A.d;
  const float a = A.a;
  unsigned long long ph[4] = {0, 0, 0, 0};
  long long tq = clock64();
#define PC_PHASE(i)                         \
  if (A.prof) {                             \
    const long long tn = clock64();         \
    ph[i] += (unsigned long long)(tn - tq); \
    tq = tn;                                \
  }

  if (warp == 1) {
    // ---------------- producer ----------------
    // chunk k goes to buffer k&1; before refilling a buffer the producer
    // writes back the chunk it held (k-2): replica words and the node sum.
    auto writeback = [&](PcBuf& B) {
      if (B.m > 0) {
        const uint32_t tag = B.tag;
        const int nu = B.n_uniq;
        for (int i = lane; i < nu; i += 32) {
          const int h = B.uniq[i];
          const int r = B.key[h];
          const float cv = B.acc[h];
          if (cv != 0.f) {
            rep_store(dv, r, tag, B.dvold[h] + cv);
            if (!A.one_part) red_add_f32(A.delta_v + r, cv);
          }
          B.key[h] = kEmpty;
        }
      }
      __syncwarp();
    };
    int k = 0;
    for (int64_t p = p_lo; p <= p_hi; ++p) {
      const bool end = p == p_hi;
      const int64_t s0 = end ? 0 : A.wp[p], s1 = end ? 1 : A.wp[p + 1];
      int64_t c0 = s0;
      while (c0 < s1) {
        const int bi = k & 1;
        PcBuf& B = S.buf[bi];
        if (k >= 2) {
          mbar_wait(&S.empty[bi], ((k >> 1) - 1) & 1);
          PC_PHASE(0);
          writeback(B);
          PC_PHASE(1);
        }
        int m = 1;
        if (end) {
          if (lane == 0) B.m = -1;
        } else {
          pc_produce(A, B, lane, c0, s1, A.tag0 + (uint32_t)p, dv, &m);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.full[bi]);
        PC_PHASE(2);
        c0 += m > 0 ? m : 1;
        ++k;
      }
    }
    // k-1 is the end marker; chunk k-2 still holds updates
    if (k >= 2) {
      const int bi = k & 1;  // == (k-2)&1
      mbar_wait(&S.empty[bi], ((k >> 1) - 1) & 1);
      writeback(S.buf[bi]);
    }
  } else {
    // ---------------- consumer ----------------
    // Hot rows [0, H): the running partition's b = u + a dv and its dv stay
    // resident in shared memory for the whole partition (no gather, patch or
    // writeback per chunk); at a partition change they are written back as
    // replica words (and to the node sum in the atomic mode).  With rows in
    // descending frequency order (config 4's Zipf features are) this keeps
    // most of a chunk's distinct rows off HBM.
    const int H = A.hot;
    float* hot_b = reinterpret_cast<float*>(smem_raw + sizeof(PcSmem));
    float* hot_acc = hot_b + H;
    uint32_t hot_tag = 0;  // partition whose hot rows are resident (0: none)
    auto hot_flush = [&]() {
      for (int r = lane; r < H; r += 32) {
        const float cv = hot_acc[r];
        if (cv != 0.f) {
          rep_store(dv, r, hot_tag, cv);
          if (!A.one_part) red_add_f32(A.delta_v + r, cv);
        }
      }
    };
    for (int k = 0;; ++k) {
      const int bi = k & 1;
      mbar_wait(&S.full[bi], (k >> 1) & 1);
      PcBuf& C = S.buf[bi];
      const int m = C.m;
      if (m < 0) break;
      const uint32_t tag = C.tag;
      const int nb = (k + 1) & 1;
      PcBuf& N = S.buf[nb];
      if (H > 0 && tag != hot_tag) {  // a new partition: swap the hot rows
        if (hot_tag != 0) hot_flush();
        for (int r = lane; r < H; r += 32) {
          hot_b[r] = __ldg(A.u + r);
          hot_acc[r] = 0.f;
        }
        hot_tag = tag;
        __syncwarp();
      }
      PC_PHASE(0);
      if (m == 0) {
        // a single long column, streamed with the replica read and written in
        // place.  Chunk k+1 being staged means the producer has written back
        // chunk k-1, so the replica in memory is current.
        mbar_wait(&S.full[nb], ((k + 1) >> 1) & 1);
        const bool patch = N.m > 0 && N.tag == tag;
        const int jj = C.col_j[0];
        const int64_t a0 = A.cp[jj], a1 = A.cp[jj + 1];
        float part = 0.f;
        for (int64_t e = a0 + lane; e < a1; e += 32) {
          const int i = A.ri[e];
          const float bv = i < H ? hot_b[i] : fmaf(a, rep_load_cg(dv, i, tag), A.u[i]);
          part = fmaf(A.vals[e], bv, part);
        }
        part = warp_sum(part);
        const float aj = *(volatile float*)(A.alpha + jj);
        const float an = sparse_step<KIND>(A, part, aj, __ldg(A.sq + jj));
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
            if (i < H) {
              hot_b[i] = fmaf(a, c, hot_b[i]);
              hot_acc[i] += c;
              continue;
            }
            const float nv = rep_load_cg(dv, i, tag) + c;
            rep_store(dv, i, tag, nv);
            if (!A.one_part) red_add_f32(A.delta_v + i, c);
            if (patch) pc_patch(N, i, nv, a);
          }
        }
        __syncwarp();
        PC_PHASE(1);
      } else {
        if (A.iid && lane < m) C.alpha_c[lane] = *(volatile float*)(A.alpha + C.col_j[lane]);
        __syncwarp();
        // Columns of up to 64 nonzeros (two per lane) take a register path:
        // the next column's slots and values are loaded while this column's
        // dot reduces, b and acc are read once and written back from
        // registers (a column's rows are distinct, so no lane races another).
        int ps0 = 0, ps1 = 0, pb0 = C.col_pre[0], pb1 = C.col_pre[1];
        float pv0 = 0.f, pv1 = 0.f;
        if (pb0 + lane < pb1) { ps0 = C.slot[pb0 + lane]; pv0 = C.val[pb0 + lane]; }
        if (pb0 + 32 + lane < pb1) { ps1 = C.slot[pb0 + 32 + lane]; pv1 = C.val[pb0 + 32 + lane]; }
        for (int t = 0; t < m; ++t) {
          const int b0 = pb0, b1 = pb1;
          const int jt = C.col_j[t];
          const float aj = C.alpha_c[t];
          const float qt = C.q_c[t];
          float delta = 0.f;
          bool ok;
          if (b1 - b0 <= 64) {
            const bool in0 = b0 + lane < b1, in1 = b0 + 32 + lane < b1;
            const int s0 = ps0, s1 = ps1;
            const float v0 = pv0, v1 = pv1;
            float* bp0 = s0 < H ? hot_b + s0 : C.b + (s0 - H);
            float* ap0 = s0 < H ? hot_acc + s0 : C.acc + (s0 - H);
            float* bp1 = s1 < H ? hot_b + s1 : C.b + (s1 - H);
            float* ap1 = s1 < H ? hot_acc + s1 : C.acc + (s1 - H);
            const float bv0 = in0 ? *bp0 : 0.f, bv1 = in1 ? *bp1 : 0.f;
            const float av0 = in0 ? *ap0 : 0.f, av1 = in1 ? *ap1 : 0.f;
            // the next column's layout (static) under the reduction's latency
            if (t + 1 < m) {
              pb0 = b1;
              pb1 = C.col_pre[t + 2];
              ps0 = ps1 = 0;
              if (pb0 + lane < pb1) { ps0 = C.slot[pb0 + lane]; pv0 = C.val[pb0 + lane]; }
              if (pb0 + 32 + lane < pb1) { ps1 = C.slot[pb0 + 32 + lane]; pv1 = C.val[pb0 + 32 + lane]; }
            }
            const float lin = warp_sum(fmaf(v1, bv1, v0 * bv0));
            const float an = sparse_step<KIND>(A, lin, aj, qt);
            ok = isfinite(an);
            if (ok) delta = an - aj;
            if (delta != 0.f) {
              const float c0 = delta * v0, c1 = delta * v1;
              if (in0) {
                *bp0 = fmaf(a, c0, bv0);
                *ap0 = av0 + c0;
              }
              if (in1) {
                *bp1 = fmaf(a, c1, bv1);
                *ap1 = av1 + c1;
              }
            }
          } else {
            float part = 0.f;
            for (int e = b0 + lane; e < b1; e += 32) {
              const int sl = C.slot[e];
              part = fmaf(C.val[e], sl < H ? hot_b[sl] : C.b[sl - H], part);
            }
            const float lin = warp_sum(part);
            const float an = sparse_step<KIND>(A, lin, aj, qt);
            ok = isfinite(an);
            if (ok) delta = an - aj;
            if (delta != 0.f) {
              for (int e = b0 + lane; e < b1; e += 32) {
                const int sl = C.slot[e];
                const float c = delta * C.val[e];
                float* bp = sl < H ? hot_b + sl : C.b + (sl - H);
                float* ap = sl < H ? hot_acc + sl : C.acc + (sl - H);
                *bp = fmaf(a, c, *bp);
                *ap += c;
              }
            }
            if (t + 1 < m) {
              pb0 = b1;
              pb1 = C.col_pre[t + 2];
              ps0 = ps1 = 0;
              if (pb0 + lane < pb1) { ps0 = C.slot[pb0 + lane]; pv0 = C.val[pb0 + lane]; }
              if (pb0 + 32 + lane < pb1) { ps1 = C.slot[pb0 + 32 + lane]; pv1 = C.val[pb0 + 32 + lane]; }
            }
          }
          if (!ok && lane == 0) atomicOr(A.status, SYSCD_ENONFINITE);
          if (lane < m && lane > t && C.col_j[lane] == jt) C.alpha_c[lane] = aj + delta;
          if (lane == 0 && ok) A.alpha[jt] = aj + delta;
          __syncwarp();
        }
        PC_PHASE(1);
        // chunk k+1 was staged from the replica before this chunk's updates
        // reach memory: patch its copy of every row written here
        mbar_wait(&S.full[nb], ((k + 1) >> 1) & 1);
        PC_PHASE(2);
        if (N.m > 0 && N.tag == tag) {
          // both tables use the same hash, so most rows sit at their first
          // probe position: 4 rows' probes in flight per lane
          const int nu = C.n_uniq;
          for (int i0 = lane; i0 < nu; i0 += 128) {
            int rq[4], kq[4];
            unsigned hq[4];
            float nvq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int i = i0 + 32 * q;
              rq[q] = kEmpty;
              if (i < nu) {
                const int h = C.uniq[i];
                const float cv = C.acc[h];
                if (cv != 0.f) {
                  rq[q] = C.key[h];
                  nvq[q] = C.dvold[h] + cv;
                }
              }
              hq[q] = pc_hash(rq[q]);
              // rows the next chunk cannot hold are dropped by its filter
              const unsigned fh = pc_fhash(rq[q]);
              const bool maybe = rq[q] != kEmpty && ((N.filt[fh >> 5] >> (fh & 31)) & 1u);
              kq[q] = maybe ? N.key[hq[q]] : kEmpty;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (kq[q] == kEmpty) continue;
              int hn = kq[q] == rq[q] ? (int)hq[q] : pc_find(N, rq[q]);
              if (hn >= 0) {
                N.b[hn] = fmaf(a, nvq[q] - N.dvold[hn], N.b[hn]);
                N.dvold[hn] = nvq[q];
              }
            }
          }
        }
        __syncwarp();
      }
      if (lane == 0) mbar_arrive(&S.empty[bi]);
      PC_PHASE(3);
    }
    if (hot_tag != 0) hot_flush();
  }
#undef PC_PHASE
  if (A.prof && lane == 0)
    for (int i = 0; i < 4; ++i) A.prof[(int64_t)g * 8 + warp * 4 + i] = ph[i];
}

// delta_v[r] = sum over partitions p (ascending) of replica word (p, r) when
// it carries partition p's tag (else that partition left row r untouched)
__global__ void k_sparse_node_sum(const unsigned long long* __restrict__ dv_work, int32_t n_parts,
                                  int64_t d, uint32_t tag0, float* __restrict__ delta_v) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < d;
       r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < n_parts; ++p) {
      const unsigned long long x = __ldcs(dv_work + (int64_t)p * d + r);
      if ((uint32_t)(x >> 32) == tag0 + (uint32_t)p) s += (double)__uint_as_float((uint32_t)x);
    }
    delta_v[r] = (float)s;
  }
}

static unsigned long long* g_sparse_prof = nullptr;

// One resident wave of workers (a worker owns whole partitions; more workers
// than fit would only queue) and the hot-row count: the largest H whose
// shared memory (8 H bytes per worker) still lets every partition have its
// own worker -- the deterministic one-partition-per-worker mode -- else none.
struct SparsePlan {
  int workers;
  int hot;
};

static int sparse_per_sm(size_t smem) {
  int per_sm = 0;
  const void* fn = (const void*)k_sparse_epoch<SYSCD_LOGISTIC_DUAL>;  // most registers
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sparse_epoch<SYSCD_LOGISTIC_DUAL>,
                                                    64, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return per_sm;
}

static SparsePlan sparse_plan(int64_t d, int32_t n_parts) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const char* force = getenv("SYSCD_SPARSE_HOT");  // experiments: fixed H
  for (int H = 16384; H >= 32; H /= 2) {  // (H <= d/4: some rows stay hashed)
    if (force && atoi(force) != H) continue;
    if (4 * (int64_t)H > d) continue;
    const int per_sm = sparse_per_sm(sizeof(PcSmem) + 8 * (size_t)H);
    if (per_sm > 0 && (int64_t)sms * per_sm >= n_parts) return {n_parts, H};
  }
  const int per_sm = std::max(1, sparse_per_sm(sizeof(PcSmem)));
  return {std::max(1, std::min((int)n_parts, sms * per_sm)), 0};
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
  *n_workers = sparse_plan(d, n_parts).workers;
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
  A.inv_n_d = 1.0 / e->n_coords;
  A.kind = e->kind;
  A.iid = e->iid;
  A.dv_work = (unsigned long long*)e->dv_work;
  A.tag0 = e->replica_tag;
  A.delta_v = e->delta_v;
  A.status = e->status;
  A.prof = g_sparse_prof;
  A.one_part = W == e->n_parts ? 1 : 0;
  const SparsePlan plan = sparse_plan(e->d, e->n_parts);
  A.hot = plan.workers == W ? plan.hot : 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (!A.one_part) SYSCD_CUDA_TRY(cudaMemsetAsync(e->delta_v, 0, e->d * sizeof(float), s));
  const size_t smem = sizeof(PcSmem) + 8 * (size_t)A.hot;
  void (*fn)(SparseArgs, int) = e->kind == SYSCD_LASSO          ? k_sparse_epoch<SYSCD_LASSO>
                                : e->kind == SYSCD_SVM_DUAL        ? k_sparse_epoch<SYSCD_SVM_DUAL>
                                : e->kind == SYSCD_LOGISTIC_DUAL   ? k_sparse_epoch<SYSCD_LOGISTIC_DUAL>
                                                                   : k_sparse_epoch<SYSCD_RIDGE>;
  SYSCD_CUDA_TRY(
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fn<<<W, 64, smem, s>>>(A, W);
  SYSCD_CUDA_TRY(cudaGetLastError());
  if (A.one_part) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks = std::min<int64_t>((e->d + 255) / 256, (int64_t)sms * 8);
    k_sparse_node_sum<<<(int)blocks, 256, 0, s>>>(A.dv_work, e->n_parts, e->d, A.tag0,
                                                  e->delta_v);
    SYSCD_CUDA_TRY(cudaGetLastError());
  }
  return SYSCD_OK;
}

#ifdef SYSCD_NEWTON_HIST
// experiment hook: copy out (and reset) the fast-path iteration histogram
extern "C" int syscd_debug_newton_hist(unsigned long long* out24) {
  cudaMemcpyFromSymbol(out24, syscd::g_newton_hist, sizeof(unsigned long long) * 24);
  unsigned long long z[24] = {0};
  cudaMemcpyToSymbol(syscd::g_newton_hist, z, sizeof(z));
  return 0;
}
#endif
