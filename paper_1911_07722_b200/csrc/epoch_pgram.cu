// Partition-Gram SySCD round: many short partitions of tall dense columns
// (BASELINE config 2: 148 partitions of 8 or 16 Lasso updates per round over
// d = 400K rows).
//
// Same semantics as epoch_dense.cu (solvers.py:289-334): partition p walks
// its updates k = 0..m-1 on a private replica w = u + a dv_p,
//     lin_k = x_k . w,  alpha_k <- step(lin_k),  w += a delta_k x_k,
// and the round's result is sum_p dv_p (reduce_replicas, solvers.py:112-125).
// With w_k = u + a sum_{i<k} delta_i x_i that chain is, exactly in real
// arithmetic,
//     lin_k = c_k + a sum_{i<k} delta_i G_ik,   c_k = x_k . u,  G_ik = x_i . x_k,
// so a partition needs one pass over its m columns for the m + m(m-1)/2
// inner products, a 16-step scalar chain, and a second pass for
// dv += sum_k delta_k x_k.  No replica has to live on chip, so every SM
// streams (the cluster kernel holds each partition's 1.6 MB replica in the
// registers of 16 SMs of one GPC, and only 7 such clusters fit: 112 SMs).
//
// B200 mapping:
//  * one CTA per SM (cooperative grid); CTA c owns rows [c*R, (c+1)*R) of
//    every column, split into kPgNSB sub-blocks; a producer warp TMA-loads
//    the sub-block of all m columns of a partition into one ring stage;
//  * jobs in order: pass 1 of partition p, then pass 2 of partition p-LA; the
//    pass-1 loads are L2 evict_last, so the pass-2 loads of the same bytes
//    LA partitions later (~LA x 25 MB) hit L2 and HBM sees A once;
//  * pass 1: 6 math warps accumulate the 136 inner products of their rows in
//    registers, reduce them warp -> CTA (fixed order) and publish the CTA's
//    record as tagged 64-bit words (tag << 32 | fp32);
//  * grid reduction in two light stages (reducer warp): CTA v sums value v
//    over all CTAs in CTA order and publishes the total; every CTA gathers
//    the 136 totals, runs the chain (lane k holds update k: lin_k, its Gram
//    row, alpha_k) and hands the deltas to its math warps through an
//    mbarrier.  All CTAs compute bit-identical deltas; CTA 0 writes alpha;
//  * pass 2 accumulates dv for the CTA's rows in registers over the whole
//    round and writes it once at the end: out = sum_p dv_p, summed in
//    partition order by one thread per row (deterministic).
#include <stdio.h>
#include <stdlib.h>

#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)

#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace syscd {

constexpr int kPgM = 16;                              // max updates per partition
constexpr int kPgNV = kPgM + kPgM * (kPgM - 1) / 2;  // c_k and G_ik (i < k): 136
constexpr int kPgNSB = 4;                             // row sub-blocks per partition job
constexpr int kPgStages = 4;
constexpr int kPgMath = 6;                            // math warps
constexpr int kPgTC = kPgMath * 32;
constexpr int kPgThreads = (kPgMath + 2) * 32;        // + producer + reducer
constexpr int kPgRPT = 4;                             // rows per thread and sub-block
constexpr int kPgMaxSB = kPgTC * kPgRPT;              // 768 rows per sub-block
constexpr int kPgSlots = 8;                           // record / delta slots (> LA + 1)
constexpr int kPgQ = 5;                               // CTAs per reducer lane (G <= 160)
constexpr int kPgMB = 4;                              // max buckets per partition (B >= 4)

__host__ __device__ constexpr int pg_gidx(int i, int k) { return kPgM + k * (k - 1) / 2 + i; }

struct PgArgs {
  const float* A;
  int64_t lda;
  int64_t d;
  const float* sq;
  float* alpha;
  const float* u;
  const int32_t* seq;
  const int64_t* wp;
  int32_t n_parts;
  int32_t B;         // bucket columns: a partition's updates are whole buckets
  int64_t n_store;
  int32_t sb_rows;   // rows per sub-block (multiple of 32, <= kPgMaxSB)
  int64_t cta_rows;  // kPgNSB * sb_rows
  float a, lam_f, inv_n_f;
  double a_d, lam, n_coords;
  float* out;                // [d] sum of the partitions' dv
  unsigned long long* recs;  // [kPgSlots][G][kPgNV] tagged CTA partials
  unsigned long long* tots;  // [kPgSlots][kPgNV] tagged grid totals
  int32_t* status;
  unsigned long long* dbg;  // SYSCD_PG_TRACE builds: [p][cta][8] %globaltimer stamps
};

#ifdef SYSCD_PG_TRACE
#define PGT(k)                                                               \
  do {                                                                       \
    if (A.dbg && lane == 0) {                                                \
      unsigned long long t_;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      A.dbg[((size_t)p * gridDim.x + blockIdx.x) * 8 + (k)] = t_;            \
    }                                                                        \
  } while (0)
#else
#define PGT(k) \
  do {         \
  } while (0)
#endif

struct PgSmem {
  size_t ring, u, full, empty, dbar, red, dsm, gt, wp, seq, total;
};

// the round's tables live in shared memory -- work_prefix (int64), update
// columns (int32), each update's tile slot (int8), each partition's bucket
// count (int8) and bucket start columns (int32 x kPgMB) -- so no role ever
// waits on a dependent global load per job
constexpr int kPgMetaBytes = 16 * 1024;
__host__ __device__ inline bool pg_meta_fits(int64_t n_parts, int64_t updates) {
  return (n_parts + 1) * 8 + updates * 5 + n_parts * (1 + 4 * kPgMB) + 16 <= kPgMetaBytes;
}

// 3-D tile copy of a tensor map: box {32 rows, SB/32 row groups, B columns}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

__host__ __device__ inline size_t pg_align(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline PgSmem pg_smem(int sb_rows) {
  PgSmem L;
  size_t o = 0;
  L.ring = o;
  o += (size_t)kPgStages * kPgM * sb_rows * 4;
  L.u = o = pg_align(o, 128);
  o += (size_t)kPgNSB * sb_rows * 4;
  L.full = o = pg_align(o, 8);
  o += kPgStages * 8;
  L.empty = o;
  o += kPgStages * 8;
  L.dbar = o;
  o += kPgSlots * 8;
  L.red = o = pg_align(o, 16);
  o += (size_t)2 * kPgMath * kPgNV * 4;  // double-buffered warp deposits
  L.dsm = o;
  o += (size_t)kPgSlots * kPgM * 4;
  L.gt = o;
  o += (size_t)kPgNV * 4;
  L.wp = o = pg_align(o, 8);
  L.seq = o;  // wp and seq share kPgMetaBytes
  o += kPgMetaBytes;
  L.total = pg_align(o, 128);
  return L;
}

__device__ __forceinline__ void pg_st_tagged(unsigned long long* p, uint32_t tag, float v) {
  const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

__device__ __forceinline__ unsigned long long pg_ld_tagged(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}

// Sum 32 values over a warp with 31 shuffles (transposed butterfly); lane l
// returns the total of value pg_tidx(l).
__device__ __forceinline__ float pg_warp_sum32(float (&v)[32], int lane) {
  int cnt = 32;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const int half = cnt / 2;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k < half) {
        const float send = upper ? v[k] : v[k + half];
        const float keep = upper ? v[k + half] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    cnt = half;
  }
  return v[0];
}

__host__ __device__ constexpr int pg_tidx(int lane) {
  int idx = 0, cnt = 32, off = 16;
  for (int s = 0; s < 5; ++s) {
    cnt /= 2;
    if (lane & off) idx += cnt;
    off >>= 1;
  }
  return idx;
}

// pass 1 over one sub-block with MM columns staged: accumulate c_k and G_ik
template <int MM>
__device__ __forceinline__ void pg_gram_rows(float (&acc)[kPgNV], const float* stg, const float* us,
                                             int sb_rows, int tid, int valid_rows) {
#pragma unroll
  for (int i = 0; i < kPgRPT; ++i) {
    const int r = tid + kPgTC * i;
    if (r < valid_rows) {
      float x[MM];
#pragma unroll
      for (int k = 0; k < MM; ++k) x[k] = stg[(size_t)k * sb_rows + r];
      const float uu = us[r];
#pragma unroll
      for (int k = 0; k < MM; ++k) {
        acc[k] = fmaf(x[k], uu, acc[k]);
#pragma unroll
        for (int j = 0; j < k; ++j) acc[pg_gidx(j, k)] = fmaf(x[j], x[k], acc[pg_gidx(j, k)]);
      }
    }
  }
}

template <int KIND, int LA>
__global__ void __launch_bounds__(kPgThreads, 1)
    k_pgram_epoch(PgArgs A, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int SB = A.sb_rows;
  const PgSmem Lo = pg_smem(SB);
  float* ring = reinterpret_cast<float*>(smem + Lo.ring);
  float* us = reinterpret_cast<float*>(smem + Lo.u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lo.full);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + Lo.empty);
  uint64_t* dbar = reinterpret_cast<uint64_t*>(smem + Lo.dbar);
  float* red = reinterpret_cast<float*>(smem + Lo.red);
  float* dsm = reinterpret_cast<float*>(smem + Lo.dsm);
  float* gt = reinterpret_cast<float*>(smem + Lo.gt);
  int64_t* wps = reinterpret_cast<int64_t*>(smem + Lo.wp);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int P = A.n_parts;
  const int64_t row0 = (int64_t)cta * A.cta_rows;
  int64_t valid = A.d - row0;
  valid = valid < 0 ? 0 : (valid > A.cta_rows ? A.cta_rows : valid);

  // u for this CTA's rows (zero past d), staged once per round
  for (int64_t r = tid; r < (int64_t)kPgNSB * SB; r += blockDim.x)
    us[r] = r < valid ? A.u[row0 + r] : 0.f;
  for (int i = tid; i <= P; i += blockDim.x) wps[i] = A.wp[i];
  const int64_t sbase = A.wp[0];
  const int nupd = (int)(A.wp[P] - sbase);
  int32_t* seqs = reinterpret_cast<int32_t*>(wps + P + 1);
  for (int i = tid; i < nupd; i += blockDim.x) seqs[i] = A.seq[sbase + i];
  int32_t* bst = seqs + nupd;                                 // [P][kPgMB] bucket starts
  int8_t* nbs = reinterpret_cast<int8_t*>(bst + (size_t)P * kPgMB);  // [P] bucket counts
  int8_t* slots = nbs + P;                                    // [nupd] tile slot per update
  // a zeroed ring: a tile slot a partition does not stage holds finite bytes
  for (int i = tid; i < kPgStages * kPgM * SB; i += blockDim.x) ring[i] = 0.f;
  fence_proxy_async();
  __syncthreads();
  // each partition's buckets (in order of first appearance) and the slot of
  // every update in the partition's tile (bucket i, column c -> i * B + c)
  for (int p = warp; p < P; p += blockDim.x / 32) {
    const int s0 = (int)(wps[p] - sbase);
    const int m = (int)(wps[p + 1] - wps[p]);
    const int j = lane < m ? seqs[s0 + lane] : 0;
    const int bs = j / A.B * A.B;
    unsigned left = __ballot_sync(0xffffffffu, lane < m);
    int nb = 0;
    while (left) {
      const int bl = __shfl_sync(0xffffffffu, bs, __ffs(left) - 1);
      const bool mine = lane < m && bs == bl;
      if (mine) slots[s0 + lane] = (int8_t)(nb < kPgMB ? nb * A.B + (j - bl) : 0);
      if (lane == 0 && nb < kPgMB) bst[p * kPgMB + nb] = bl;
      left &= ~__ballot_sync(0xffffffffu, mine);
      ++nb;
    }
    if (lane == 0) {
      nbs[p] = (int8_t)min(nb, kPgMB);
      if (nb * A.B > kPgM) atomicOr(A.status, SYSCD_EINVAL);  // host contract broken
    }
  }
  if (tid == 0) {
    for (int s = 0; s < kPgStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPgMath);
    }
    for (int s = 0; s < kPgSlots; ++s) mbar_init(&dbar[s], 1);
    fence_mbar_init();
    fence_proxy_async();
  }
  __syncthreads();

  if (warp == kPgMath) {
    // ------------------------------------------------------------- producer
    // step p: sub-block b of pass 1 of partition p (HBM, kept in L2) then
    // sub-block b of pass 2 of partition p - LA (the same bytes, now L2
    // hits), so every stage in flight is half HBM, half L2 traffic
    uint32_t stage = 0, phase = 0;
    const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
    const uint32_t tile_bytes = (uint32_t)SB * (uint32_t)A.B * 4u;
    auto issue = [&](int pp, int b, uint64_t pol) {
      if (lane == 0) {
        const int nb = nbs[pp];
        mbar_wait(&empty[stage], phase ^ 1u);
        mbar_arrive_expect_tx(&full[stage], tile_bytes * (uint32_t)nb);
        float* dst = ring + (size_t)stage * kPgM * SB;
        const int c1 = (int)((row0 + (int64_t)b * SB) / 32);
        for (int i = 0; i < nb; ++i)
          tma_load_3d(dst + (size_t)i * A.B * SB, &tmap, 0, c1, bst[pp * kPgMB + i], &full[stage],
                      pol);
      }
      if (++stage == kPgStages) {
        stage = 0;
        phase ^= 1u;
      }
      __syncwarp();
    };
    for (int p = 0; p < P + LA; ++p) {
      const int p1 = p < P && wps[p + 1] > wps[p] ? p : -1;
      const int p2 = p >= LA && wps[p - LA + 1] > wps[p - LA] ? p - LA : -1;
#pragma unroll 1
      for (int b = 0; b < kPgNSB; ++b) {
        if (p1 >= 0) issue(p1, b, keep);
        if (p2 >= 0) issue(p2, b, drop);
      }
    }
  } else if (warp == kPgMath + 1) {
    // -------------------------------------------------------------- reducer
    // Two pipelined stages, polled without blocking: stage A of partition pa
    // (this CTA sums values v = cta, cta + G, ... over all CTAs and publishes
    // the totals) runs ahead of stage B of partition pb (gather the kPgNV
    // totals, run the chain, hand the deltas over), so one partition's
    // gather latency overlaps the next partition's.
    int pa = 0, pb = 0, qa = 0, qb = 0;
    int va = cta;  // next value of partition pa this CTA reduces
    unsigned long long wa[kPgQ], wb[(kPgNV + 31) / 32];
#pragma unroll
    for (int qq = 0; qq < kPgQ; ++qq) wa[qq] = 0ull;
#pragma unroll
    for (int qq = 0; qq < (kPgNV + 31) / 32; ++qq) wb[qq] = 0ull;
    while (pa < P && wps[pa + 1] == wps[pa]) ++pa;
    while (pb < P && wps[pb + 1] == wps[pb]) ++pb;
    while (pb < P) {
      bool prog = false;
      // ---- stage A (at most kPgSlots - 2 partitions ahead of stage B)
      if (pa < P && qa < qb + kPgSlots - 2) {
        if (va >= kPgNV) {
          // nothing (more) to reduce for pa: next non-empty partition
          ++qa;
          do {
            ++pa;
          } while (pa < P && wps[pa + 1] == wps[pa]);
          va = cta;
          prog = true;
        } else {
          const int slot = qa % kPgSlots;
          const uint32_t tag = (uint32_t)(pa + 1);
          const unsigned long long* rec = A.recs + (size_t)slot * G * kPgNV;
          bool ok = true;
#pragma unroll
          for (int qq = 0; qq < kPgQ; ++qq) {
            const int c = lane + 32 * qq;
            if (c < G && (uint32_t)(wa[qq] >> 32) != tag)
              wa[qq] = pg_ld_tagged(rec + (size_t)c * kPgNV + va);
          }
#pragma unroll
          for (int qq = 0; qq < kPgQ; ++qq)
            ok &= lane + 32 * qq >= G || (uint32_t)(wa[qq] >> 32) == tag;
          if (__all_sync(0xffffffffu, ok)) {
            float part = 0.f;
#pragma unroll
            for (int qq = 0; qq < kPgQ; ++qq)
              part += lane + 32 * qq < G ? __uint_as_float((uint32_t)wa[qq]) : 0.f;
            const float tot = warp_sum(part);
            if (lane == 0) pg_st_tagged(A.tots + (size_t)slot * kPgNV + va, tag, tot);
            {
              const int p = pa;
              PGT(2);
            }
            va += G;
            prog = true;
          }
        }
      }
      // ---- stage B
      {
        const int p = pb;
        const int slot = qb % kPgSlots;
        const uint32_t tag = (uint32_t)(p + 1);
        const unsigned long long* tt = A.tots + (size_t)slot * kPgNV;
        bool ok = true;
#pragma unroll
        for (int qq = 0; qq < (kPgNV + 31) / 32; ++qq) {
          const int v = lane + 32 * qq;
          if (v < kPgNV && (uint32_t)(wb[qq] >> 32) != tag) wb[qq] = pg_ld_tagged(tt + v);
        }
#pragma unroll
        for (int qq = 0; qq < (kPgNV + 31) / 32; ++qq)
          ok &= lane + 32 * qq >= kPgNV || (uint32_t)(wb[qq] >> 32) == tag;
        if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
          for (int qq = 0; qq < (kPgNV + 31) / 32; ++qq)
            if (lane + 32 * qq < kPgNV) gt[lane + 32 * qq] = __uint_as_float((uint32_t)wb[qq]);
          __syncwarp();
          PGT(3);
          const int s0 = (int)(wps[p] - sbase);
          const int m = (int)(wps[p + 1] - wps[p]);
          // lane k = update k of tile slot s_k (no repeats: perm rounds)
          int jk = 0, sk = 0;
          float ak = 0.f, qk = 0.f;
          if (lane < m) {
            jk = seqs[s0 + lane];
            sk = slots[s0 + lane];
            ak = __ldcg(A.alpha + jk);
            qk = __ldg(A.sq + jk);
          }
          float lin = lane < m ? gt[sk] : 0.f;
          float ag[kPgM];  // a * G(s_i, s_k), i < k
#pragma unroll
          for (int i = 0; i < kPgM; ++i) {
            const int si = __shfl_sync(0xffffffffu, sk, i);
            ag[i] = (i < lane && lane < m && si != sk)
                        ? A.a * gt[pg_gidx(min(si, sk), max(si, sk))]
                        : 0.f;
          }
          const float inv = step_inv(KIND, A.a, qk, A.lam_f);
          float dk = 0.f, an_k = ak;
          bool bad = false;
#pragma unroll
          for (int i = 0; i < kPgM; ++i) {
            if (i < m) {
              float an;
              if (KIND == SYSCD_LOGISTIC_DUAL) {
                an = ak;
                if (lane == i)
                  an = (float)coord_step(SYSCD_LOGISTIC_DUAL, (double)lin, A.a_d, (double)qk,
                                         A.lam, (double)ak, A.n_coords);
              } else {
                // every lane evaluates its own step (no divergence); lane i's is used
                an = coord_step_fr(KIND, lin, inv, A.lam_f, ak, A.inv_n_f);
              }
              const bool fin = isfinite(an);
              const float di = fin ? an - ak : 0.f;
              if (lane == i) {
                dk = di;
                an_k = fin ? an : ak;
                bad = !fin;
              }
              lin = fmaf(ag[i], __shfl_sync(0xffffffffu, di, i), lin);
            }
          }
          // pass-2 weights per tile slot
          if (lane < kPgM) dsm[slot * kPgM + lane] = 0.f;
          __syncwarp();
          if (lane < m) dsm[slot * kPgM + sk] = dk;
          if (cta == 0 && lane < m) {
            __stcg(A.alpha + jk, an_k);
            if (bad) atomicOr(A.status, SYSCD_ENONFINITE);
          }
          __syncwarp();
          PGT(4);
          if (lane == 0) mbar_arrive(&dbar[slot]);
          ++qb;
          do {
            ++pb;
          } while (pb < P && wps[pb + 1] == wps[pb]);
          prog = true;
        }
      }
      if (!prog) __nanosleep(32);
    }
  } else {
    // ----------------------------------------------------------- math warps
    float dv[kPgNSB][kPgRPT];
#pragma unroll
    for (int b = 0; b < kPgNSB; ++b)
#pragma unroll
      for (int i = 0; i < kPgRPT; ++i) dv[b][i] = 0.f;
    uint32_t stage = 0, phase = 0;
    // non-empty partitions seen by the pass-1 / pass-2 walks (slot and
    // mbarrier phase of the q-th non-empty partition: q % kPgSlots, q / kPgSlots)
    int q1 = 0, q2 = 0;
    auto next_stage = [&]() {
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kPgStages) {
        stage = 0;
        phase ^= 1u;
      }
    };
    for (int p = 0; p < P + LA; ++p) {
      const int p1 = p < P && wps[p + 1] > wps[p] ? p : -1;
      const int p2 = p >= LA && wps[p - LA + 1] > wps[p - LA] ? p - LA : -1;
      if (p1 < 0 && p2 < 0) continue;
      const int ns1 = p1 >= 0 ? nbs[p1] * A.B : 0;
      const int ns2 = p2 >= 0 ? nbs[p2] * A.B : 0;
      float dl[kPgM];
      if (p2 >= 0) {
        const int q = q2++;
        mbar_wait(&dbar[q % kPgSlots], (uint32_t)((q / kPgSlots) & 1));
        {
          const int p = p2;
          if (warp == 0) PGT(5);
        }
#pragma unroll
        for (int k = 0; k < kPgM; ++k) dl[k] = dsm[(q % kPgSlots) * kPgM + k];
      }
      float acc[kPgNV];
#pragma unroll
      for (int v = 0; v < kPgNV; ++v) acc[v] = 0.f;
#pragma unroll
      for (int b = 0; b < kPgNSB; ++b) {
        int64_t vr = valid - (int64_t)b * SB;
        const int vrows = vr < 0 ? 0 : (vr > SB ? SB : (int)vr);
        if (p1 >= 0) {
          mbar_wait(&full[stage], phase);
          if (b == 0) {
            const int p = p1;
            PGT(0);
          }
          const float* stg = ring + (size_t)stage * kPgM * SB;
          if (ns1 <= 8) {
            pg_gram_rows<8>(acc, stg, us + (size_t)b * SB, SB, tid, vrows);
          } else {
            pg_gram_rows<16>(acc, stg, us + (size_t)b * SB, SB, tid, vrows);
          }
          next_stage();
        }
        if (p2 >= 0) {
          // dv += sum_s D_s x_s (every slot holds finite bytes, unused ones weigh 0)
          mbar_wait(&full[stage], phase);
          const float* stg = ring + (size_t)stage * kPgM * SB;
#pragma unroll
          for (int i = 0; i < kPgRPT; ++i) {
            const int r = tid + kPgTC * i;
            if (r < vrows) {
              float sacc = dv[b][i];
              if (ns2 <= 8) {
#pragma unroll
                for (int k = 0; k < 8; ++k) sacc = fmaf(dl[k], stg[(size_t)k * SB + r], sacc);
              } else {
#pragma unroll
                for (int k = 0; k < kPgM; ++k) sacc = fmaf(dl[k], stg[(size_t)k * SB + r], sacc);
              }
              dv[b][i] = sacc;
            }
          }
          next_stage();
        }
      }
      if (p1 >= 0) {
        const int q = q1++;
        const int slot = q % kPgSlots;
        // slots past the staged tiles hold other partitions' bytes
#pragma unroll
        for (int k = 0; k < kPgM; ++k) {
          if (k >= ns1) {
            acc[k] = 0.f;
#pragma unroll
            for (int j = 0; j < k; ++j) acc[pg_gidx(j, k)] = 0.f;
          }
        }
        // warp totals (transposed), deposits, CTA total in warp order
        float* rb = red + (size_t)(q & 1) * kPgMath * kPgNV;
#pragma unroll
        for (int g = 0; g < (kPgNV + 31) / 32; ++g) {
          float vv[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) vv[k] = 32 * g + k < kPgNV ? acc[32 * g + k] : 0.f;
          const float tv = pg_warp_sum32(vv, lane);
          const int v = 32 * g + pg_tidx(lane);
          if (v < kPgNV) rb[warp * kPgNV + v] = tv;
        }
        named_bar_sync(1, kPgTC);
        if (warp == 0) {
          unsigned long long* rec = A.recs + ((size_t)slot * G + cta) * kPgNV;
          for (int v = lane; v < kPgNV; v += 32) {
            float sacc = 0.f;
#pragma unroll
            for (int w = 0; w < kPgMath; ++w) sacc += rb[w * kPgNV + v];
            pg_st_tagged(rec + v, (uint32_t)(p1 + 1), sacc);
          }
          {
            const int p = p1;
            PGT(1);
          }
        }
      }
    }
#pragma unroll
    for (int b = 0; b < kPgNSB; ++b)
#pragma unroll
      for (int i = 0; i < kPgRPT; ++i) {
        const int64_t r = (int64_t)b * SB + tid + kPgTC * i;
        if (tid + kPgTC * i < SB && r < valid) A.out[row0 + r] = dv[b][i];
      }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
#ifndef SYSCD_PG_LA
#define SYSCD_PG_LA 2
#endif
constexpr int kPgLA = SYSCD_PG_LA;  // partitions of lookahead between pass 1 and pass 2

static const void* pg_fn(int kind) {
  switch (kind) {
    case SYSCD_LASSO:
      return (const void*)&k_pgram_epoch<SYSCD_LASSO, kPgLA>;
    case SYSCD_SVM_DUAL:
      return (const void*)&k_pgram_epoch<SYSCD_SVM_DUAL, kPgLA>;
    case SYSCD_LOGISTIC_DUAL:
      return (const void*)&k_pgram_epoch<SYSCD_LOGISTIC_DUAL, kPgLA>;
    default:
      return (const void*)&k_pgram_epoch<SYSCD_RIDGE, kPgLA>;
  }
}

// Geometry: one CTA per SM; rows per CTA split into kPgNSB sub-blocks of at
// most kPgMaxSB rows (multiples of 4, so every bulk copy is 16-byte sized).
static bool pg_geometry(int64_t d, int* G, int* sb_rows, size_t* smem) {
  // sub-blocks are whole 32-row groups (tile coordinates in units of 128 B)
  int dev = 0, sms = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  const int64_t per_cta = (d + sms - 1) / sms;
  int64_t sb = (per_cta + kPgNSB - 1) / kPgNSB;
  sb = (sb + 31) / 32 * 32;
  if (sb > kPgMaxSB) return false;
  if ((d + kPgNSB * sb - 1) / (kPgNSB * sb) > 32 * kPgQ) return false;
  const size_t sm = pg_smem((int)sb).total;
  if (sm + 1024 > (size_t)optin) return false;
  *G = (int)((d + kPgNSB * sb - 1) / (kPgNSB * sb));
  *sb_rows = (int)sb;
  *smem = sm;
  return true;
}

// The partition-Gram kernel takes rounds whose partitions hold at most kPgM
// updates, on columns tall enough that every SM gets a slice (and the
// cluster kernel would leave SMs idle).
bool pgram_applicable(int64_t d, int32_t n_parts, int32_t max_part_updates, int32_t bucket_cols,
                      int64_t lda) {
  if (max_part_updates < 1 || max_part_updates > kPgM || n_parts < 2) return false;
  if (bucket_cols < 4 || bucket_cols > kPgM || lda % 32 != 0) return false;
  // whole buckets: at most ceil(max / B) tiles, and they must fit the slots
  if ((max_part_updates + bucket_cols - 1) / bucket_cols * bucket_cols > kPgM) return false;
  if (!pg_meta_fits(n_parts, (int64_t)n_parts * max_part_updates)) return false;
  if (d < 65536) return false;
  int G, sb;
  size_t sm;
  return pg_geometry(d, &G, &sb, &sm);
}

int64_t pgram_workspace_bytes(int64_t d) {
  int G, sb;
  size_t sm;
  if (!pg_geometry(d, &G, &sb, &sm)) return 0;
  return (int64_t)kPgSlots * ((int64_t)G + 1) * kPgNV * 8;
}

static void* g_pg_dbg = nullptr;

// cuTensorMapEncodeTiled (driver API, reached through the runtime's entry
// point query so the library does not link libcuda directly)
typedef CUresult (*PgEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int pgram_launch(const syscd_dense_epoch_args* e, cudaStream_t stream) {
  int G, sb;
  size_t smem;
  if (!pg_geometry(e->d, &G, &sb, &smem)) {
    set_error("syscd_dense_epoch: no partition-Gram geometry for d=%lld", (long long)e->d);
    return SYSCD_EINVAL;
  }
  const int64_t ws = (int64_t)kPgSlots * ((int64_t)G + 1) * kPgNV * 8;
  if (!e->workspace || e->workspace_bytes < ws) {
    set_error("syscd_dense_epoch: partition-Gram workspace too small");
    return SYSCD_EINVAL;
  }
  const void* fn = pg_fn(e->kind);
  SYSCD_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CUtensorMap tmap;
  {
    // A as a 3-D tensor {32 rows, lda/32 row groups, n_store columns}; one box
    // = SB rows of B consecutive columns (a bucket's sub-block)
    static std::mutex mu;
    static PgEncodeTiled encode = nullptr;
    {
      std::lock_guard<std::mutex> lock(mu);
      if (!encode) {
        cudaDriverEntryPointQueryResult qr;
        void* f = nullptr;
        SYSCD_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr));
        if (!f || qr != cudaDriverEntryPointSuccess) {
          set_error("syscd_dense_epoch: cuTensorMapEncodeTiled unavailable");
          return SYSCD_EINVAL;
        }
        encode = (PgEncodeTiled)f;
      }
    }
    const cuuint64_t dims[3] = {32, (cuuint64_t)(e->lda / 32), (cuuint64_t)e->n_store};
    const cuuint64_t strides[2] = {128, (cuuint64_t)e->lda * 4};
    const cuuint32_t box[3] = {32, (cuuint32_t)(sb / 32), (cuuint32_t)e->bucket_cols};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)e->A, dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("syscd_dense_epoch: tensor map encode failed (%d)", (int)r);
      return SYSCD_EINVAL;
    }
  }
  PgArgs A;
  A.A = e->A;
  A.lda = e->lda;
  A.d = e->d;
  A.sq = e->sq;
  A.alpha = e->alpha;
  A.u = e->u;
  A.seq = e->seq;
  A.wp = e->work_prefix;
  A.n_parts = e->n_parts;
  A.B = e->bucket_cols;
  A.n_store = e->n_store;
  A.sb_rows = sb;
  A.cta_rows = (int64_t)kPgNSB * sb;
  A.a = (float)e->a;
  A.lam_f = (float)e->lam;
  A.inv_n_f = (float)(1.0 / e->n_coords);
  A.a_d = e->a;
  A.lam = e->lam;
  A.n_coords = e->n_coords;
  A.out = e->partials;
  A.recs = (unsigned long long*)e->workspace;
  A.tots = A.recs + (size_t)kPgSlots * G * kPgNV;
  A.status = e->status;
  A.dbg = (unsigned long long*)g_pg_dbg;
  SYSCD_CUDA_TRY(cudaMemsetAsync(e->workspace, 0, ws, stream));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(kPgThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {&A, &tmap};
  SYSCD_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, params));
  return SYSCD_OK;
}

}  // namespace syscd

// Debug hook (not part of the header ABI): device buffer of >= n_parts * G * 8
// uint64 receiving the SYSCD_PG_TRACE build's per-partition stamps.
extern "C" void syscd_debug_set_pgram_timeline(void* device_buffer) {
  syscd::g_pg_dbg = device_buffer;
}
