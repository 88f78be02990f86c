// SySCD round for medium-height columns (32 < d <= kMidMaxD, e.g. BASELINE
// config 0: ridge with d = 20000).
//
// Semantics: _surrogate_thread_round (solvers.py:289-334) -- per coordinate
// lin = x_j . (u + a dv), alpha_j <- step, dv += delta x_j -- on a private
// replica per partition, exactly as epoch_dense.cu.
//
// At this height the per-coordinate chain of the cluster kernel is bound by
// its cluster-wide reduction latency (~0.9 us per update), not by bandwidth
// (A is L2-resident).  This kernel rewrites the chain exactly (in real
// arithmetic) over chunks of up to kMidM consecutive updates of a partition,
// the medium-height form of epoch_small.cu: with w = u + a dv at the chunk
// start,
//     c_t  = x_t . w ,   G_ts = x_t . x_s          (one pass over the chunk)
//     lin_t = c_t + a * sum_{s<t} delta_s G_ts     (sequential, scalar)
//     w   += a * sum_t delta_t x_t                 (one pass)
// so one cluster reduction serves kMidM updates.
//
// B200 mapping: a worker is a cluster of C CTAs; CTA r owns rows
// [r*Rc, (r+1)*Rc) and holds their w in shared memory.  A producer warp
// stages each chunk's column slices with 1-D bulk copies (TMA) into one of two
// tiles while the previous chunk is processed.  8 math warps compute the
// CTA's partial c / G over their row slices (register-blocked 2x4 outer
// products on 16-byte shared loads), reduce them in a fixed order, and every
// CTA pushes its 16x17 partials to every peer with st.async (DSMEM,
// mbarrier::complete_tx); each CTA sums the C partials in rank order (so
// every CTA takes bit-identical steps), runs the 16-step chain in one warp and
// updates its rows.  Partition ends fold (w-u)/a into the worker's partials
// row (plain store, then red.global.add: deterministic).
#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace syscd {

constexpr int kMidM = 16;            // updates per chunk
constexpr int kMidRowsMax = 1280;    // rows per CTA
constexpr int kMidMaxCluster = 16;
constexpr int kMidWarps = 8;         // math warps
constexpr int kMidThreads = 32 * kMidWarps;
constexpr int kMidBlock = kMidThreads + 32;  // + producer warp
// packed partials: the lower triangle G_ts (s <= t) then c_t
constexpr int kMidTri = kMidM * (kMidM + 1) / 2;
constexpr int kMidG = kMidTri + kMidM;
__host__ __device__ constexpr int mid_tri(int t, int s) { return t * (t + 1) / 2 + s; }
constexpr int64_t kMidMaxD = (int64_t)kMidRowsMax * kMidMaxCluster;

struct MidArgs {
  const float* A;
  int64_t lda;
  int64_t d;
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
  int32_t rows;  // Rc: rows per CTA (multiple of 8)
  int32_t rs;    // tile row stride in floats (>= rows, = 4 mod 32)
  unsigned long long* dbg;  // debug: per-chunk phase cycles of CTA 0 (nullptr = off)
};

struct MidSmem {
  size_t tile, w, wpart, inbox, gtot, delta, meta, mcount, full, empty, xbar, range, total;
};

__host__ __device__ inline size_t mid_align(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline MidSmem mid_smem(int rs) {
  MidSmem L;
  size_t o = 0;
  L.tile = o;
  o += (size_t)2 * kMidM * rs * 4;
  L.w = o;
  o += (size_t)rs * 4;
  L.wpart = o;
  o += (size_t)kMidWarps * kMidG * 4;
  L.inbox = mid_align(o, 16);
  o = L.inbox + (size_t)2 * kMidMaxCluster * kMidG * 4;
  L.gtot = o;
  o += (size_t)kMidG * 4;
  L.delta = o;
  o += kMidM * 4;
  L.meta = mid_align(o, 16);
  o = L.meta + 2 * kMidM * 16;
  L.mcount = o;
  o += 2 * 4;
  L.full = mid_align(o, 8);
  o = L.full + 2 * 8;
  L.empty = o;
  o += 2 * 8;
  L.xbar = o;
  o += 2 * 8;
  L.range = o;
  o += 2 * 8;
  L.total = mid_align(o, 128);
  return L;
}

__device__ __forceinline__ float dot4(float4 a, float4 b, float acc) {
  acc = fmaf(a.x, b.x, acc);
  acc = fmaf(a.y, b.y, acc);
  acc = fmaf(a.z, b.z, acc);
  return fmaf(a.w, b.w, acc);
}

// 3xTF32: x = hi + lo with both parts exact tf32; hi*hi + hi*lo + lo*hi
// carries ~fp32 accuracy (the lo*lo term is below fp32 rounding).
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  const float r = x - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int KIND>
__device__ __forceinline__ float mid_step(const MidArgs& A, float lin, float aj, float q,
                                          float inv) {
  if (KIND == SYSCD_LOGISTIC_DUAL)
    return (float)coord_step(KIND, (double)lin, A.a_d, (double)q, A.lam, (double)aj, A.n_coords);
  return coord_step_fr(KIND, lin, inv, A.lam_f, aj, A.inv_n_f);
}

template <int KIND>
__global__ void __launch_bounds__(kMidBlock, 1) k_mid_epoch(MidArgs A) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int rs = A.rs;
  const MidSmem L = mid_smem(rs);
  float* tile = reinterpret_cast<float*>(smem + L.tile);
  float* wv = reinterpret_cast<float*>(smem + L.w);
  float* wpart = reinterpret_cast<float*>(smem + L.wpart);
  float* inbox = reinterpret_cast<float*>(smem + L.inbox);
  float* gtot = reinterpret_cast<float*>(smem + L.gtot);
  float* delta_s = reinterpret_cast<float*>(smem + L.delta);
  int4* meta = reinterpret_cast<int4*>(smem + L.meta);
  int* mcount = reinterpret_cast<int*>(smem + L.mcount);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.full);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + L.empty);
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + L.xbar);
  int64_t* range = reinterpret_cast<int64_t*>(smem + L.range);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int C = (int)cluster_nctarank();
  const int rank = (int)cluster_rank();
  const int g = blockIdx.x / C;
  const int G = gridDim.x / C;
  const int Rc = A.rows;
  const int64_t row0 = (int64_t)rank * Rc;
  const int64_t d = A.d;
  int64_t valid = d - row0;
  valid = valid < 0 ? 0 : (valid > Rc ? Rc : valid);
  const uint32_t col_bytes = (uint32_t)(((valid + 3) / 4) * 16);

  // tiles start at zero: rows past d stay zero (they are never written)
  for (int i = tid; i < 2 * kMidM * rs; i += blockDim.x) tile[i] = 0.f;
  // every writer orders its generic-proxy zeros before the TMA (async
  // proxy) fills that follow the barrier; one fence by the issuing thread
  // does not cover the other threads' writes
  fence_proxy_async();
  for (int i = tid; i < rs; i += blockDim.x) wv[i] = i < valid ? A.u[row0 + i] : 0.f;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kMidWarps);
      mbar_init(&xbar[b], 1);
    }
    int64_t p_lo, p_hi;
    worker_parts(A.wp, A.n_parts, G, g, &p_lo, &p_hi);
    range[0] = p_lo < A.n_parts ? p_lo : A.n_parts;
    range[1] = p_hi < A.n_parts ? p_hi : A.n_parts;
    fence_mbar_init();
    fence_proxy_async();
  }
  const long long t_enter = clock64();
  __syncthreads();
  cluster_sync_all();
  const int64_t p_lo = range[0], p_hi = range[1];
  if (A.dbg && blockIdx.x == 0 && tid == 0) {
    A.dbg[255 * 8 + 0] = t_enter;
    A.dbg[255 * 8 + 1] = clock64();
  }
  if (A.dbg && rank == 0 && tid == 0 && g < 64) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    A.dbg[(128 + g) * 8 + 0] = gt;
  }

  if (warp == kMidWarps) {
    // ------------------------------------------------------------ producer
    const uint64_t policy = policy_evict_last();  // A is L2-resident at this height
    int k = 0;
    for (int64_t p = p_lo; p < p_hi; ++p) {
      const int64_t s1 = A.wp[p + 1];
      for (int64_t c0 = A.wp[p]; c0 < s1; c0 += kMidM, ++k) {
        const int m = (int)min((int64_t)kMidM, s1 - c0);
        const int b = k & 1;
        int j = 0;
        float aj = 0.f, qj = 0.f;
        if (lane < m) {
          j = A.seq[c0 + lane];
          aj = A.iid ? 0.f : A.alpha[j];
          qj = __ldg(A.sq + j);
        }
        if (k >= 2) mbar_wait(&empty[b], ((k >> 1) - 1) & 1);
        if (lane < m)
          meta[b * kMidM + lane] = make_int4(j, __float_as_int(aj), __float_as_int(qj),
                                            __float_as_int(step_inv(KIND, A.a, qj, A.lam_f)));
        if (lane == 0) {
          mcount[b] = m;
          if (col_bytes) {
            mbar_arrive_expect_tx(&full[b], col_bytes * (uint32_t)m);
          } else {
            mbar_arrive(&full[b]);
          }
        }
        __syncwarp();
        if (lane < m && col_bytes)
          tma_load_1d(tile + ((size_t)b * kMidM + lane) * rs, A.A + (int64_t)j * A.lda + row0,
                      col_bytes, &full[b], policy);
        __syncwarp();
      }
    }
    return;
  }

  // -------------------------------------------------------------- math warps
  // this warp's row slice in k-steps of 8 rows (Rc is a multiple of 8)
  const int ngroups = Rc / 4;
  const int nks = Rc / 8;
  const int kw0 = nks * warp / kMidWarps, kw1 = nks * (warp + 1) / kMidWarps;
  const float a = A.a;
  const float inv_a = (float)(1.0 / A.a_d);
  float* out = A.partials + (int64_t)g * A.part_ld + row0;
  bool flushed = false;
  int k = 0;
  for (int64_t p = p_lo; p < p_hi; ++p) {
    const int64_t s1 = A.wp[p + 1];
    if (s1 == A.wp[p]) continue;
    for (int64_t c0 = A.wp[p]; c0 < s1; c0 += kMidM, ++k) {
      const int b = k & 1;
#if defined(SYSCD_TRACE) || defined(SYSCD_DENSE_STAMPS)
      const bool dbg = A.dbg && blockIdx.x == 0 && tid == 0 && k < 256;
#else
      constexpr bool dbg = false;  // stamps only in the trace build (scripts/timeline_mid.py)
#endif
      if (dbg) A.dbg[k * 8 + 0] = clock64();
      mbar_wait(&full[b], (k >> 1) & 1);
      if (dbg) A.dbg[k * 8 + 1] = clock64();
      const int m = mcount[b];
      const float* tb = tile + (size_t)b * kMidM * rs;
      // ---- partial G_ts over this warp's rows on the tensor cores:
      // D(16 x 16) += X^T(16 x 8) X(8 x 16) per 8 rows (mma.m16n8k8 tf32,
      // 3 products per tile for fp32 accuracy); c_t = x_t . w with FMAs on
      // the same A fragments
      // one accumulator per (n-tile, product): six independent mma chains
      float acc[2][3][4] = {};
      float c_lo = 0.f, c_hi = 0.f;  // c for t = gid, gid + 8 (partial over tig)
      {
        const int gid = lane >> 2, tig = lane & 3;
        const float* ra = tb + (size_t)gid * rs;        // rows t = gid, gid + 8
        const float* rb = tb + (size_t)(gid + 8) * rs;
        for (int ks = kw0; ks < kw1; ++ks) {
          const int i0 = ks * 8 + tig;
          const float x0 = ra[i0], x1 = rb[i0], x2 = ra[i0 + 4], x3 = rb[i0 + 4];
          const float w0 = wv[i0], w1 = wv[i0 + 4];
          c_lo = fmaf(x2, w1, fmaf(x0, w0, c_lo));
          c_hi = fmaf(x3, w1, fmaf(x1, w0, c_hi));
          uint32_t ah[4], al[4];
          tf32_split(x0, ah[0], al[0]);
          tf32_split(x1, ah[1], al[1]);
          tf32_split(x2, ah[2], al[2]);
          tf32_split(x3, ah[3], al[3]);
          // n-tiles 0, 1: s = gid (+8): the same rows as the A operand
          uint32_t bh0, bl0, bh1, bl1;
          bh0 = ah[0]; bl0 = al[0]; bh1 = ah[2]; bl1 = al[2];
          mma_tf32(acc[0][0], ah, bh0, bh1);
          mma_tf32(acc[0][1], ah, bl0, bl1);
          mma_tf32(acc[0][2], al, bh0, bh1);
          bh0 = ah[1]; bl0 = al[1]; bh1 = ah[3]; bl1 = al[3];
          mma_tf32(acc[1][0], ah, bh0, bh1);
          mma_tf32(acc[1][1], ah, bl0, bl1);
          mma_tf32(acc[1][2], al, bh0, bh1);
        }
        c_lo += __shfl_xor_sync(0xffffffffu, c_lo, 1);
        c_lo += __shfl_xor_sync(0xffffffffu, c_lo, 2);
        c_hi += __shfl_xor_sync(0xffffffffu, c_hi, 1);
        c_hi += __shfl_xor_sync(0xffffffffu, c_hi, 2);
        // D fragment: rows t = gid, gid + 8; columns 2*tig, 2*tig + 1
        float* wp_w = wpart + warp * kMidG;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int t = gid + (e >= 2 ? 8 : 0);
            const int sc = nt * 8 + 2 * tig + (e & 1);
            if (sc <= t) wp_w[mid_tri(t, sc)] = acc[nt][0][e] + (acc[nt][1][e] + acc[nt][2][e]);
          }
        if (tig == 0) {
          wp_w[kMidTri + gid] = c_lo;
          wp_w[kMidTri + gid + 8] = c_hi;
        }
      }
      named_bar_sync(1, kMidThreads);
      if (dbg) A.dbg[k * 8 + 2] = clock64();
      // ---- CTA partial (fixed warp order), pushed to every peer
      for (int idx = tid; idx < kMidG; idx += kMidThreads) {
        float v = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < kMidWarps; ++w2) v += wpart[w2 * kMidG + idx];
        const uint32_t dst = smem_addr(inbox + ((size_t)b * kMidMaxCluster + rank) * kMidG + idx);
        const uint32_t bar = smem_addr(&xbar[b]);
        for (int r = 0; r < C; ++r) st_async_f32(cluster_map(dst, r), v, cluster_map(bar, r));
      }
      if (tid == 0) mbar_arrive_expect_tx(&xbar[b], (uint32_t)(C * kMidG * 4));
      if (dbg) A.dbg[k * 8 + 3] = clock64();
      mbar_wait_cluster(&xbar[b], (k >> 1) & 1);
      if (dbg) A.dbg[k * 8 + 4] = clock64();
      // ---- totals in rank order (identical in every CTA) and the chain
      for (int idx = tid; idx < kMidG; idx += kMidThreads) {
        float v = 0.f;
        for (int r = 0; r < C; ++r) v += inbox[((size_t)b * kMidMaxCluster + r) * kMidG + idx];
        gtot[idx] = v;
      }
      named_bar_sync(1, kMidThreads);
      if (warp == 0) {
        const int4 mt = lane < m ? meta[b * kMidM + lane] : make_int4(-1 - lane, 0, 0, 0);
        const int j = mt.x;
        float alpha_t = __int_as_float(mt.y);
        if (A.iid && lane < m) alpha_t = *(volatile float*)(A.alpha + j);
        const float q_t = __int_as_float(mt.z);
        const float inv_t = __int_as_float(mt.w);
        float r = lane < kMidM ? gtot[kMidTri + lane] : 0.f;
        float Gr[kMidM];
#pragma unroll
        for (int sc = 0; sc < kMidM; ++sc)
          Gr[sc] = (lane < kMidM && sc < lane) ? a * gtot[mid_tri(lane, sc)] : 0.f;
        const bool iid = A.iid != 0;
        float my_delta = 0.f;
        auto step_once = [&](int sc) {
          float cand = alpha_t;
          if (KIND != SYSCD_LOGISTIC_DUAL || lane == sc)
            cand = mid_step<KIND>(A, r, alpha_t, q_t, inv_t);
          const float dl = __shfl_sync(0xffffffffu, cand - alpha_t, sc);
          my_delta = lane == sc ? dl : my_delta;
          r = fmaf(dl, Gr[sc], r);
          if (iid) {
            const int js = __shfl_sync(0xffffffffu, j, sc);
            if (lane > sc && j == js) alpha_t += dl;
          }
        };
        if (m == kMidM) {
#pragma unroll
          for (int sc = 0; sc < kMidM; ++sc) step_once(sc);
        } else {
#pragma unroll
          for (int sc = 0; sc < kMidM; ++sc)
            if (sc < m) step_once(sc);
        }
        if (lane < m && !isfinite(my_delta)) {
          if (rank == 0) atomicOr(A.status, SYSCD_ENONFINITE);
          my_delta = 0.f;
        }
        // a repeated coordinate (iid) is written once, by its last occurrence
        const unsigned same = __match_any_sync(0xffffffffu, j);
        if (rank == 0 && lane < m && (31 - __clz(same)) == lane) A.alpha[j] = alpha_t + my_delta;
        if (lane < kMidM) delta_s[lane] = lane < m ? my_delta : 0.f;
      }
      named_bar_sync(1, kMidThreads);
      if (dbg) A.dbg[k * 8 + 5] = clock64();
      // ---- w += a sum_t delta_t x_t over this CTA's rows
      float dl[kMidM];
#pragma unroll
      for (int t = 0; t < kMidM; ++t) dl[t] = a * delta_s[t];
      // (columns t >= m of a partial chunk hold finite stale data and delta_t
      // = 0 there, so no guard: the 16 loads issue back to back)
      for (int gq = tid; gq < ngroups; gq += kMidThreads) {
        float4 w4 = reinterpret_cast<float4*>(wv)[gq];
#pragma unroll
        for (int t = 0; t < kMidM; ++t) {
          const float4 x = reinterpret_cast<const float4*>(tb + (size_t)t * rs)[gq];
          w4.x = fmaf(dl[t], x.x, w4.x);
          w4.y = fmaf(dl[t], x.y, w4.y);
          w4.z = fmaf(dl[t], x.z, w4.z);
          w4.w = fmaf(dl[t], x.w, w4.w);
        }
        reinterpret_cast<float4*>(wv)[gq] = w4;
      }
      fence_proxy_async();  // reads done before the TMA refill (async proxy) of this stage
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
      named_bar_sync(1, kMidThreads);
      if (dbg) A.dbg[k * 8 + 6] = clock64();
    }
    // ---- partition end: fold (w - u)/a into the worker's partial row, reset w
    for (int i = tid; i < valid; i += kMidThreads) {
      const float uu = __ldg(A.u + row0 + i);
      const float dv = (wv[i] - uu) * inv_a;
      if (flushed) {
        red_add_f32(out + i, dv);
      } else {
        out[i] = dv;
      }
      wv[i] = uu;
    }
    flushed = true;
    named_bar_sync(1, kMidThreads);
  }
  if (!flushed)
    for (int i = tid; i < valid; i += kMidThreads) out[i] = 0.f;
  if (A.dbg && blockIdx.x == 0 && tid == 0) A.dbg[255 * 8 + 2] = clock64();
  if (A.dbg && rank == 0 && tid == 0 && g < 64) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    A.dbg[(128 + g) * 8 + 1] = gt;
  }
  // (every push into this CTA's inbox happened before its last xbar wait
  // returned, so leaving now cannot race a peer's st.async)
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct MidChoice {
  int C, rows, rs, G;
  size_t smem;
};

// one cached configuration per cluster size (the attribute setting and the
// occupancy query are host calls; they are done once, not per launch)
static std::mutex g_mid_mu;
static int g_mid_clusters[kMidMaxCluster + 1];  // 0 = unknown, -1 = not launchable

static int mid_choose(int64_t d, int32_t n_parts, MidChoice* out) {
  if (d <= 32 || d > kMidMaxD) return SYSCD_EINVAL;
  const int C = (int)((d + kMidRowsMax - 1) / kMidRowsMax);
  int rows = (int)((d + C - 1) / C);
  rows = (rows + 7) / 8 * 8;  // k-steps of 8 rows (rows past d stay zero)
  int rs = rows;
  while (rs % 32 != 4) ++rs;  // fragment loads across t hit distinct banks
  const size_t smem = mid_smem(rs).total;
  std::lock_guard<std::mutex> lock(g_mid_mu);
  int& nclusters = g_mid_clusters[C];
  if (nclusters == 0) {
    nclusters = -1;
    const void* fns[4] = {(const void*)&k_mid_epoch<SYSCD_RIDGE>,
                          (const void*)&k_mid_epoch<SYSCD_LASSO>,
                          (const void*)&k_mid_epoch<SYSCD_SVM_DUAL>,
                          (const void*)&k_mid_epoch<SYSCD_LOGISTIC_DUAL>};
    const size_t smem_max = mid_smem(kMidRowsMax + 36).total;  // any rs this C can need
    bool ok = true;
    for (const void* f : fns) {
      ok &= cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max) ==
            cudaSuccess;
      if (C > 8) cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C, 1, 1);
    cfg.blockDim = dim3(kMidBlock, 1, 1);
    cfg.dynamicSmemBytes = smem_max;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (ok && cudaOccupancyMaxActiveClusters(&n, fns[0], &cfg) == cudaSuccess && n >= 1)
      nclusters = n;
    cudaGetLastError();
  }
  if (nclusters < 1) return SYSCD_EINVAL;
  out->C = C;
  out->rows = rows;
  out->rs = rs;
  out->G = std::max(1, std::min((int)n_parts, nclusters));
  out->smem = smem;
  return SYSCD_OK;
}

bool mid_applicable(int64_t d, int32_t n_parts, int* workers, int* cluster) {
  MidChoice ch;
  if (mid_choose(d, n_parts, &ch) != SYSCD_OK) return false;
  if (workers) *workers = ch.G;
  if (cluster) *cluster = ch.C;
  return true;
}

static void* g_mid_dbg = nullptr;

int mid_launch(const syscd_dense_epoch_args* e, cudaStream_t stream) {
  MidChoice ch;
  if (mid_choose(e->d, e->n_parts, &ch) != SYSCD_OK) {
    set_error("medium-height epoch: no configuration for d=%lld", (long long)e->d);
    return SYSCD_EINVAL;
  }
  MidArgs A;
  A.A = e->A;
  A.lda = e->lda;
  A.d = e->d;
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
  A.rows = ch.rows;
  A.rs = ch.rs;
  A.dbg = (unsigned long long*)g_mid_dbg;
  const void* fn = e->kind == SYSCD_LASSO          ? (const void*)&k_mid_epoch<SYSCD_LASSO>
                   : e->kind == SYSCD_SVM_DUAL      ? (const void*)&k_mid_epoch<SYSCD_SVM_DUAL>
                   : e->kind == SYSCD_LOGISTIC_DUAL ? (const void*)&k_mid_epoch<SYSCD_LOGISTIC_DUAL>
                                                    : (const void*)&k_mid_epoch<SYSCD_RIDGE>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ch.G * ch.C, 1, 1);
  cfg.blockDim = dim3(kMidBlock, 1, 1);
  cfg.dynamicSmemBytes = ch.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ch.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {&A};
  SYSCD_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, params));
  return SYSCD_OK;
}

}  // namespace syscd

// Debug hook (not part of the C-ABI contract): with a device buffer of
// 256*8 uint64, the next medium-height epochs record CTA 0's clock at the
// chunk phases (start, staged, Gram done, pushed, totals in, chain done,
// w updated).
extern "C" void syscd_debug_set_mid_timeline(void* device_buffer) { syscd::g_mid_dbg = device_buffer; }
