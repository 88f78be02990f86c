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
// update; afterwards w += a * sum_t delta_t x_t.  One worker is one block: a
// chain warp (lane t owns update t of the chunk) and kSmallHelpers staging
// warps that load the next chunk's columns and compute its Gram matrix into
// the other of two shared-memory buffers while the chain runs.  Workers take
// contiguous update-balanced ranges of partitions and fold (w-u)/a into their
// own partials row at each partition end (fixed order: deterministic).
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
  unsigned long long* prof;  // debug: per-worker chain-warp phase cycles (nullptr = off)
};

constexpr int kSmallHelpers = 7;  // staging / Gram warps per worker
constexpr int kSmallThreads = 32 * (1 + kSmallHelpers);
constexpr int kGramStride = 36;   // 16-byte aligned Gram rows

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
    return (float)logistic_dual_solve((double)r, A.a_d * (double)q, (double)alpha, A.n_coords,
                                      1.0 / A.n_coords);
  }
}

template <int D>
struct SmallSmem {
  static constexpr int DP = D + 4;  // 16-byte aligned rows, conflict-free 16-byte reads
  float tile[2][32][DP];            // [buffer][chunk column][row]
  float G[2][32][kGramStride];      // [buffer][t][s] = x_t . x_s (s < t used)
  int j[2][32];
  float q[2][32];
  float alpha[2][32];
  float inv_aq[2][32];
  float w[32];
  alignas(16) float delta[32];
  uint64_t full[2], empty[2];
};

// One worker = one block: warp 0 runs the chain, warps 1..kSmallHelpers stage
// the next chunk's columns and compute its Gram matrix (double-buffered), so
// the chain warp's per-chunk work is c_t, the 32 sequential steps and the w
// update.  Every worker walks the same chunk sequence: contiguous
// update-balanced partitions, chunks of 32 updates.
template <int D, int KIND>
__global__ void __launch_bounds__(kSmallThreads) k_small_epoch(SmallArgs A, int W) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmallSmem<D>& S = *reinterpret_cast<SmallSmem<D>*>(smem_raw);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int g = blockIdx.x;
  if (g >= W) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.full[i], kSmallHelpers);
      mbar_init(&S.empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int d = A.d;
  const float a = A.a;
  int64_t p_lo, p_hi;
  worker_parts(A.wp, A.n_parts, W, g, &p_lo, &p_hi);

  if (warp > 0) {
    // ------------------------------------------------------------ helpers
    const int hw = warp - 1;
    constexpr int kPer = (32 + kSmallHelpers - 1) / kSmallHelpers;
    const int tl = hw + kSmallHelpers * lane;  // the chunk column this lane indexes
    // Chunks are staged two ahead of their use: the registers hold the
    // columns (and q, alpha) of the next two chunks, so the global loads of
    // a chunk are in flight for about two chunk times before its buffer is
    // free.  A chunk cursor walks the partitions' chunks in order.
    struct Cursor {
      int64_t p, c0;
    };
    auto valid = [&](const Cursor& c) { return c.p < p_hi; };
    auto advance = [&](Cursor c) {
      c.c0 += 32;
      while (c.p < p_hi && c.c0 >= A.wp[c.p + 1]) {
        ++c.p;
        if (c.p < p_hi) c.c0 = A.wp[c.p];
      }
      return c;
    };
    struct Staged {
      float col[kPer];
      float q, alpha;
      int j, m;
    };
    // ids (the coordinate of each column) of a chunk are loaded one
    // iteration before its column data, so no load waits on another
    struct Ids {
      int j, m;
    };
    auto load_ids = [&](const Cursor& c) {
      Ids id{0, 0};
      if (valid(c)) id.m = (int)min((int64_t)32, A.wp[c.p + 1] - c.c0);
      if (lane < kPer && tl < id.m) id.j = A.seq[c.c0 + tl];
      return id;
    };
    auto load = [&](const Ids& id, Staged& st) {
      st.m = id.m;
      st.j = id.j;
      st.q = st.alpha = 0.f;
      const bool mine = lane < kPer && tl < st.m;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int t = hw + kSmallHelpers * i;
        const int jt = __shfl_sync(0xffffffffu, st.j, i);
        st.col[i] = (t < st.m && lane < d) ? __ldg(A.A + (int64_t)jt * A.lda + lane) : 0.f;
      }
      if (mine) {
        st.q = __ldg(A.sq + st.j);
        if (!A.iid) st.alpha = A.alpha[st.j];
      }
    };
    Cursor c_cur{p_lo, p_lo < p_hi ? A.wp[p_lo] - 32 : 0};
    c_cur = advance(c_cur);  // the first non-empty chunk
    Cursor c_nxt = advance(c_cur);
    Cursor c_nn = advance(c_nxt);
    Staged cur, nxt;
    load(load_ids(c_cur), cur);
    load(load_ids(c_nxt), nxt);
    Ids id_nn = load_ids(c_nn);
    for (int k = 0; valid(c_cur); ++k) {
      const int b = k & 1;
      const int m = cur.m;
      if (k >= 2) mbar_wait(&S.empty[b], ((k >> 1) - 1) & 1);
      if (lane < kPer && tl < 32) S.j[b][tl] = cur.j;
      if (lane < kPer && tl < m) {
        S.q[b][tl] = cur.q;
        S.inv_aq[b][tl] = cur.q > 0.f ? __fdiv_rn(1.f, a * cur.q) : 0.f;
        S.alpha[b][tl] = cur.alpha;
      }
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int t = hw + kSmallHelpers * i;
        if (t < 32 && lane < D) S.tile[b][t][lane] = cur.col[i];
      }
      // shift the staging window: the chunk after next goes in flight with
      // the ids loaded last iteration, the one after that gets its ids
      cur = nxt;
      c_cur = c_nxt;
      c_nxt = c_nn;
      load(id_nn, nxt);
      c_nn = advance(c_nn);
      id_nn = load_ids(c_nn);
      {
        named_bar_sync(2, 32 * kSmallHelpers);
        // Gram: lane t holds row x_t; this warp fills columns s of G
        float x[D];
#pragma unroll
        for (int i4 = 0; i4 < D / 4; ++i4) {
          const float4 v = reinterpret_cast<const float4*>(S.tile[b][lane])[i4];
          x[4 * i4] = v.x;
          x[4 * i4 + 1] = v.y;
          x[4 * i4 + 2] = v.z;
          x[4 * i4 + 3] = v.w;
        }
        for (int sc = hw; sc < m; sc += kSmallHelpers) {
          const float4* ts = reinterpret_cast<const float4*>(S.tile[b][sc]);
          float acc = 0.f;
#pragma unroll
          for (int i4 = 0; i4 < D / 4; ++i4) {
            const float4 v = ts[i4];
            acc = fmaf(x[4 * i4], v.x, acc);
            acc = fmaf(x[4 * i4 + 1], v.y, acc);
            acc = fmaf(x[4 * i4 + 2], v.z, acc);
            acc = fmaf(x[4 * i4 + 3], v.w, acc);
          }
          S.G[b][lane][sc] = acc;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.full[b]);
      }
    }
    return;
  }

  // -------------------------------------------------------------- chain warp
  unsigned long long ph[4] = {0, 0, 0, 0};
  long long tq = clock64();
#define SMALL_PHASE(i)                      \
  if (A.prof) {                             \
    const long long tn = clock64();         \
    ph[i] += (unsigned long long)(tn - tq); \
    tq = tn;                                \
  }
  const float inv_a = (float)(1.0 / A.a_d);
  float* out = A.partials + (int64_t)g * A.part_ld;
  const float u_l = lane < d ? A.u[lane] : 0.f;
  bool flushed = false;
  int k = 0;
  for (int64_t p = p_lo; p < p_hi; ++p) {
    const int64_t s0 = A.wp[p], s1 = A.wp[p + 1];
    if (s1 == s0) continue;
    S.w[lane] = u_l;  // w = u at the partition start
    __syncwarp();
    for (int64_t c0 = s0; c0 < s1; c0 += 32, ++k) {
      const int m = (int)min((int64_t)32, s1 - c0);
      const int b = k & 1;
      mbar_wait(&S.full[b], (k >> 1) & 1);
      SMALL_PHASE(0);
      // c_t = x_t . w and the Gram row of lane t
      float r = 0.f;
      {
        const float4* xr = reinterpret_cast<const float4*>(S.tile[b][lane]);
        const float4* wr = reinterpret_cast<const float4*>(S.w);
#pragma unroll
        for (int i4 = 0; i4 < D / 4; ++i4) {
          const float4 xv = xr[i4], wv = wr[i4];
          r = fmaf(xv.x, wv.x, r);
          r = fmaf(xv.y, wv.y, r);
          r = fmaf(xv.z, wv.z, r);
          r = fmaf(xv.w, wv.w, r);
        }
      }
      float G[32];
#pragma unroll
      for (int s4 = 0; s4 < 8; ++s4) {
        const float4 v = reinterpret_cast<const float4*>(S.G[b][lane])[s4];
        G[4 * s4] = v.x;
        G[4 * s4 + 1] = v.y;
        G[4 * s4 + 2] = v.z;
        G[4 * s4 + 3] = v.w;
      }
      const int j = S.j[b][lane];
      const float q_t = lane < m ? S.q[b][lane] : 0.f;
      // iid rounds may revisit a coordinate of an earlier chunk: reload
      float alpha_t = lane < m ? (A.iid ? *(volatile float*)(A.alpha + j) : S.alpha[b][lane]) : 0.f;
      const float inv_aq = lane < m ? S.inv_aq[b][lane] : 0.f;
      SMALL_PHASE(1);
      // ---- sequential chain: lane s finalises lin_s, broadcasts delta_s.
      // The critical path per update is the step, one shuffle and one FMA
      // (a G_ts is pre-scaled; a non-finite step is flagged after the chain --
      // the host then raises NonFiniteUpdateError and the round is void).
#pragma unroll
      for (int s4 = 0; s4 < 32; ++s4) G[s4] *= a;
      const bool iid = A.iid != 0;
      float my_delta = 0.f;
      auto step_once = [&](int s) {
        float cand;
        if (KIND == SYSCD_LOGISTIC_DUAL) {
          // Newton solve on the owning lane only (keeps the loop body small)
          cand = alpha_t;
          if (lane == s)
            cand = small_step<KIND>(r, alpha_t, q_t, a, inv_aq, A.lam_f, A.inv_n_f, A);
        } else {
          cand = small_step<KIND>(r, alpha_t, q_t, a, inv_aq, A.lam_f, A.inv_n_f, A);
        }
        const float delta = __shfl_sync(0xffffffffu, cand - alpha_t, s);
        my_delta = lane == s ? delta : my_delta;
        r = fmaf(delta, G[s], r);
        if (iid) {
          // a coordinate drawn twice in one chunk sees its new value
          const int js = __shfl_sync(0xffffffffu, j, s);
          if (lane > s && j == js) alpha_t += delta;
        }
      };
      if (m == 32) {  // full chunk: no per-step bound checks
#pragma unroll
        for (int s = 0; s < 32; ++s) step_once(s);
      } else {
#pragma unroll
        for (int s = 0; s < 32; ++s)
          if (s < m) step_once(s);
      }
      if (lane < m && !isfinite(my_delta)) atomicOr(A.status, SYSCD_ENONFINITE);
      {
        // a repeated coordinate (iid) is written once, by its last occurrence
        const unsigned act = __ballot_sync(0xffffffffu, lane < m);
        const unsigned same = __match_any_sync(0xffffffffu, lane < m ? j : -1 - lane) & act;
        if (lane < m && (31 - __clz(same)) == lane) A.alpha[j] = alpha_t + my_delta;
      }
      S.delta[lane] = lane < m ? my_delta : 0.f;
      __syncwarp();
      SMALL_PHASE(2);
      // ---- w += a * sum_t delta_t x_t   (lane = row)
      if (lane < d) {
        // four chains (deltas of t >= m are zero), summed in a fixed order
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        const float4* dl4 = reinterpret_cast<const float4*>(S.delta);
#pragma unroll
        for (int t4 = 0; t4 < 8; ++t4) {
          const float4 dv4 = dl4[t4];
          acc[0] = fmaf(dv4.x, S.tile[b][4 * t4][lane], acc[0]);
          acc[1] = fmaf(dv4.y, S.tile[b][4 * t4 + 1][lane], acc[1]);
          acc[2] = fmaf(dv4.z, S.tile[b][4 * t4 + 2][lane], acc[2]);
          acc[3] = fmaf(dv4.w, S.tile[b][4 * t4 + 3][lane], acc[3]);
        }
        S.w[lane] = fmaf(a, (acc[0] + acc[1]) + (acc[2] + acc[3]), S.w[lane]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[b]);
      SMALL_PHASE(3);
    }
    // ---- partition end: fold (w - u)/a into this worker's partial row
    if (lane < d) {
      const float dv = (S.w[lane] - u_l) * inv_a;
      out[lane] = flushed ? out[lane] + dv : dv;
    }
    flushed = true;
    __syncwarp();
  }
  if (!flushed && lane < d) out[lane] = 0.f;
#undef SMALL_PHASE
  if (A.prof && lane == 0)
    for (int i = 0; i < 4; ++i) A.prof[(int64_t)g * 4 + i] = ph[i];
}

int small_workers(int32_t n_parts) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, std::min((int)n_parts, sms * 8));
}

static unsigned long long* g_small_prof = nullptr;

int small_launch(const syscd_dense_epoch_args* e, cudaStream_t stream) {
  SmallArgs A;
  A.prof = g_small_prof;
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
  const size_t smem = Dsel == 8 ? sizeof(SmallSmem<8>)
                     : (Dsel == 16 ? sizeof(SmallSmem<16>) : sizeof(SmallSmem<32>));
  SYSCD_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fn<<<W, kSmallThreads, smem, stream>>>(A, W);
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}

}  // namespace syscd

// Debug hook (not part of the C-ABI contract): with a device buffer of
// n_workers * 4 uint64, the next small epochs record the chain warp's cycles
// in: waiting for the staged chunk, c_t + Gram row loads, the chain, w update.
extern "C" void syscd_debug_set_small_profile(void* device_buffer) {
  syscd::g_small_prof = (unsigned long long*)device_buffer;
}
