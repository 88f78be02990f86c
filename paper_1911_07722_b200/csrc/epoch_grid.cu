// Grid-wide SySCD round for tall columns (d too large for one cluster's
// registers, e.g. BASELINE config 3: d = 1M).
//
// Same semantics as epoch_dense.cu (solvers.py:289-334): partitions run their
// chains lin = x_j . w, alpha_j <- step, w += a delta x_j on a private replica
// w = u + a dv.  Here ALL CTAs of a cooperative grid work on one partition at
// a time; CTA c owns rows [c*CTA_ROWS, (c+1)*CTA_ROWS) and every coordinate's
// dot product is reduced across the grid through global memory.
//
// Latency hiding (s-step lookahead, exact in real arithmetic): when column e
// of a partition is staged, the latest applied update is e-L-1, so each CTA
// computes
//     s_e = x_e . w_{<= e-L-1}   and   g_{e,k} = x_e . x_{e-k},  k = 1..L
// publishes these L+1 partials, and resolves column e-L with
//     lin_{e-L} = S_{e-L} + a * sum_k delta_{e-L-k} G_{e-L,k}
// from grid totals published L events earlier (exact: w_{<=e-2L-1} plus the
// L updates e-2L..e-L-1 accounted through the cross terms).  The last L+1
// columns live in a register ring, so the cross terms cost FMAs only.
//
// Warp roles per CTA: 1 TMA producer warp (column slices into a shared-memory
// ring + (j, alpha_j, q_j) metadata ring), 1 reducer warp (waits on the grid
// counter of each published step, sums the G partial records in a fixed order
// and hands the totals to the math warps through an mbarrier), NTC/32 math
// warps.  Totals are summed in the same order in every CTA, so all CTAs take
// bit-identical steps and the result is deterministic.  Partitions run one
// after another; between them the pipeline drains, (w-u)/a is folded into
// `out` (each row has exactly one writer) and w is reset to u.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace syscd {

constexpr int kGNB = 16;    // global partial-record slots (> 2L+1)
constexpr int kGMeta = 64;  // metadata ring (steps)
constexpr int kGTot = 8;    // totals ring in shared memory (> L)
constexpr int kGRec = 8;    // floats per partial record (L+1 <= 8)

struct GridArgs {
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
  float lam_f;
  float inv_n_f;
  double a_d, lam, n_coords;
  int32_t kind;
  int32_t stages;
  int32_t evict_first;
  float* out;                   // [d] summed replicas (one worker row)
  unsigned long long* recs;     // [kGNB][G][kGRec] tagged partials, zeroed before launch
  int32_t* status;
  unsigned long long* dbg;      // optional timeline (CTA 0)
};

__device__ __forceinline__ unsigned long long gtimer_g() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct GridSmem {
  size_t ring, full, empty, totbar, tot, red, meta, total;
};

__host__ __device__ inline size_t galign(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline GridSmem grid_smem(int stages, int cta_rows) {
  GridSmem L;
  L.ring = 0;
  size_t o = galign((size_t)stages * cta_rows * 4, 128);
  L.full = o;
  o += (size_t)stages * 8;
  L.empty = o;
  o += (size_t)stages * 8;
  L.totbar = o;
  o += kGTot * 8;
  o = galign(o, 16);
  L.tot = o;
  o += kGTot * kGRec * 4;
  L.red = o;
  o += 2 * 32 * kGRec * 4;
  o = galign(o, 16);
  L.meta = o;
  o += kGMeta * 16;
  L.total = galign(o, 128);
  return L;
}

// A partial is published as one 64-bit word (tag << 32 | float bits): the
// word is single-copy atomic, so a reader that sees the expected tag also
// sees the value -- no counter, fence or acquire round trip is needed.
__device__ __forceinline__ void st_tagged(unsigned long long* p, uint32_t tag, float v) {
  const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

__device__ __forceinline__ void ld_tagged2(const unsigned long long* p, unsigned long long& a,
                                           unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];"
               : "=l"(a), "=l"(b)
               : "l"(p)
               : "memory");
}

template <int RR, int L>
__global__ void __launch_bounds__(512, 1) k_grid_epoch(GridArgs A) {
  constexpr int NTC = 416;  // 13 math warps + producer + 2 reducers = 16 warps
  constexpr int NWC = NTC / 32;
  constexpr int NS = L + 1;
  constexpr int CTA_ROWS = NTC * RR;

  extern __shared__ __align__(128) unsigned char smem[];
  const int S = A.stages;
  const GridSmem Lo = grid_smem(S, CTA_ROWS);
  float* ring = reinterpret_cast<float*>(smem + Lo.ring);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lo.full);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + Lo.empty);
  uint64_t* totbar = reinterpret_cast<uint64_t*>(smem + Lo.totbar);
  float* tot = reinterpret_cast<float*>(smem + Lo.tot);
  float* red = reinterpret_cast<float*>(smem + Lo.red);
  int4* meta = reinterpret_cast<int4*>(smem + Lo.meta);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int G = gridDim.x;
  const int cta = blockIdx.x;
  const int64_t row0 = (int64_t)cta * CTA_ROWS;
  const int64_t d = A.d;
  const int64_t s_begin = A.wp[0];
  const int64_t s_end = A.wp[A.n_parts];

  for (int i = tid; i < S * CTA_ROWS; i += blockDim.x) ring[i] = 0.f;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWC);
    }
    for (int s = 0; s < kGTot; ++s) mbar_init(&totbar[s], 1);
    fence_mbar_init();
    fence_proxy_async();
  }
  __syncthreads();

  if (warp == NWC) {
    // ---------------------------------------------------------------- producer
    int64_t valid = d - row0;
    valid = valid < 0 ? 0 : (valid > CTA_ROWS ? CTA_ROWS : valid);
    const uint32_t bytes = (uint32_t)(((valid + 3) / 4) * 16);
    const uint64_t policy = A.evict_first ? policy_evict_first() : policy_evict_last();
    uint32_t stage = 0, phase = 0;
    int jreg = 0;
    for (int64_t s = s_begin; s < s_end; ++s) {
      const int64_t rel = s - s_begin;
      if ((rel & 31) == 0) {
        const int64_t q = s + lane;
        jreg = q < s_end ? A.seq[q] : 0;
      }
      const int j = __shfl_sync(0xffffffffu, jreg, (int)(rel & 31));
      if (lane == 0) {
        const float aj = A.alpha[j];
        const float qj = __ldg(A.sq + j);
        mbar_wait(&empty[stage], phase ^ 1u);
        meta[rel & (kGMeta - 1)] = make_int4(j, __float_as_int(aj), __float_as_int(qj), 0);
        if (bytes) {
          mbar_arrive_expect_tx(&full[stage], bytes);
          tma_load_1d(ring + (size_t)stage * CTA_ROWS, A.A + (int64_t)j * A.lda + row0, bytes,
                      &full[stage], policy);
        } else {
          mbar_arrive(&full[stage]);
        }
        if (++stage == (uint32_t)S) {
          stage = 0;
          phase ^= 1u;
        }
      }
      __syncwarp();
    }
  } else if (warp > NWC) {
    // ---------------------------------------------------------------- reducers
    // Two warps take alternate published steps.  For step r every lane issues
    // the 16-byte loads of all its CTAs' records at once (CTAs c = lane +
    // 32q), checks the tags with a warp vote and re-polls until the step is
    // complete; then each lane sums its CTAs in order and the warp folds the
    // lanes with a fixed butterfly -- identical totals in every CTA.
    constexpr int NV = (NS + 1) / 2;  // 16-byte loads per record
    constexpr int NQ = 5;             // ceil(148 / 32) records per lane
    const int64_t pubs = s_end - s_begin;
    for (int64_t r = warp - NWC - 1; r < pubs; r += 2) {
      const unsigned long long* rec = A.recs + (size_t)(r % kGNB) * G * kGRec;
      const uint32_t tag = (uint32_t)(r + 1);
      unsigned long long wv[NQ][2 * NV];
      bool done;
      do {
        bool ok = true;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int c = lane + 32 * q;
          if (c < G) {
#pragma unroll
            for (int v = 0; v < NV; ++v)
              ld_tagged2(rec + (size_t)c * kGRec + 2 * v, wv[q][2 * v], wv[q][2 * v + 1]);
          }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int c = lane + 32 * q;
          if (c < G) {
#pragma unroll
            for (int k = 0; k < NS; ++k) ok &= (uint32_t)(wv[q][k] >> 32) == tag;
          }
        }
        done = __all_sync(0xffffffffu, ok);
        if (!done) __nanosleep(64);
      } while (!done);
      float acc[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        acc[k] = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (lane + 32 * q < G) acc[k] += __uint_as_float((uint32_t)wv[q][k]);
        acc[k] = warp_sum(acc[k]);
      }
      if (lane == 0) {
        if (A.dbg && cta == 0 && r < 1024) A.dbg[r * 8 + 5] = gtimer_g();
        float* t = tot + (r % kGTot) * kGRec;
#pragma unroll
        for (int k = 0; k < NS; ++k) t[k] = acc[k];
        mbar_arrive(&totbar[r % kGTot]);
      }
      __syncwarp();
    }
  } else {
    // -------------------------------------------------------------- math warps
    const int64_t rem = d - row0 - tid;
    const int rmax = rem <= 0 ? 0 : (int)min((int64_t)RR, (rem + NTC - 1) / NTC);
    const float* ub = A.u + row0 + tid;
    float* outp = A.out + row0 + tid;
    float w[RR];
    float xr[NS][RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) w[r] = r < rmax ? ub[r * NTC] : 0.f;
#pragma unroll
    for (int k = 0; k < NS; ++k)
#pragma unroll
      for (int r = 0; r < RR; ++r) xr[k][r] = 0.f;
    const float a = A.a;
    const float inv_a = (float)(1.0 / A.a_d);
    uint32_t stage = 0, phase = 0;
    bool flushed = false;
    for (int p = 0; p < A.n_parts; ++p) {
      const int64_t pbase = A.wp[p] - s_begin;  // publication index of column 0
      const int m = (int)(A.wp[p + 1] - A.wp[p]);
      if (m == 0) continue;
      float dh[L];  // deltas of the L most recently resolved columns (dh[0] newest)
#pragma unroll
      for (int k = 0; k < L; ++k) dh[k] = 0.f;
      for (int e0 = 0; e0 < m + L; e0 += NS) {
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const int e = e0 + i;  // e % NS == i: register slot of column e
          if (e < m + L) {
            const bool dbg = A.dbg && cta == 0 && tid == 0 && p == 0 && e < 1024;
            if (dbg) A.dbg[e * 8 + 0] = gtimer_g();
            if (e < m) {
              // stage column e, publish (s_e, g_e1..g_eL)
              mbar_wait(&full[stage], phase);
              if (dbg) A.dbg[e * 8 + 1] = gtimer_g();
              const float* x = ring + (size_t)stage * CTA_ROWS + tid;
#pragma unroll
              for (int r = 0; r < RR; ++r) xr[i][r] = x[r * NTC];
              __syncwarp();
              if (lane == 0) mbar_arrive(&empty[stage]);
              if (++stage == (uint32_t)S) {
                stage = 0;
                phase ^= 1u;
              }
              float pr[NS];
#pragma unroll
              for (int k = 0; k < NS; ++k) pr[k] = 0.f;
#pragma unroll
              for (int r = 0; r < RR; ++r) {
                const float xv = xr[i][r];
                pr[0] = fmaf(xv, w[r], pr[0]);
#pragma unroll
                for (int k = 1; k <= L; ++k) pr[k] = fmaf(xv, xr[(i + NS - k) % NS][r], pr[k]);
              }
#pragma unroll
              for (int k = 0; k < NS; ++k) pr[k] = warp_sum(pr[k]);
              const int64_t pub = pbase + e;
              const int rb = (int)(pub & 1);
              if (lane == 0) {
#pragma unroll
                for (int k = 0; k < NS; ++k) red[(rb * 32 + warp) * kGRec + k] = pr[k];
              }
              named_bar_sync(1, NTC);
              if (warp == 0 && lane < NS) {
                float v = 0.f;
                for (int q = 0; q < NWC; ++q) v += red[(rb * 32 + q) * kGRec + lane];
                st_tagged(A.recs + ((size_t)(pub % kGNB) * G + cta) * kGRec + lane,
                          (uint32_t)(pub + 1), v);
              }
            }
            if (dbg) A.dbg[e * 8 + 2] = gtimer_g();
            if (e >= L) {
              // resolve column c = e - L (register slot (i+1) % NS)
              const int c = e - L;
              const int64_t cpub = pbase + c;
              mbar_wait(&totbar[cpub % kGTot], (uint32_t)((cpub / kGTot) & 1));
              if (dbg) A.dbg[e * 8 + 3] = gtimer_g();
              const float* t = tot + (cpub % kGTot) * kGRec;
              float lin = t[0];
#pragma unroll
              for (int k = 1; k <= L; ++k) lin = fmaf(a * dh[k - 1], t[k], lin);
              const int4 mt = meta[(A.wp[p] - s_begin + c) & (kGMeta - 1)];
              const int j = mt.x;
              const float aj = __int_as_float(mt.y);
              const float qj = __int_as_float(mt.z);
              float an;
              if (A.kind == SYSCD_LOGISTIC_DUAL) {
                an = (float)coord_step(A.kind, (double)lin, A.a_d, (double)qj, A.lam, (double)aj,
                                       A.n_coords);
              } else {
                an = coord_step_f(A.kind, lin, a, qj, A.lam_f, aj, A.inv_n_f);
              }
              float delta = 0.f;
              if (isfinite(an)) {
                delta = an - aj;
                if (cta == 0 && tid == 0) A.alpha[j] = an;
              } else if (cta == 0 && tid == 0) {
                atomicOr(A.status, SYSCD_ENONFINITE);
              }
#pragma unroll
              for (int k = L - 1; k > 0; --k) dh[k] = dh[k - 1];
              dh[0] = delta;
              const float sd = a * delta;
              constexpr int OLD = (0 + 1) % NS;  // placeholder to keep NS in scope
              (void)OLD;
#pragma unroll
              for (int r = 0; r < RR; ++r) w[r] = fmaf(sd, xr[(i + 1) % NS][r], w[r]);
            }
            if (dbg) A.dbg[e * 8 + 4] = gtimer_g();
          }
        }
      }
      // partition done: fold (w - u)/a into out (one writer per row), reset w
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        if (r < rmax) {
          const float uu = __ldg(ub + r * NTC);
          const float dv = (w[r] - uu) * inv_a;
          if (flushed) {
            red_add_f32(outp + r * NTC, dv);
          } else {
            outp[r * NTC] = dv;
          }
          w[r] = uu;
        }
      }
      flushed = true;
    }
    if (!flushed) {
#pragma unroll
      for (int r = 0; r < RR; ++r)
        if (r < rmax) outp[r * NTC] = 0.f;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct GridEntry {
  int rr, l;
  const void* fn;
};

template <int RR, int L>
static GridEntry make_grid() {
  return {RR, L, (const void*)&k_grid_epoch<RR, L>};
}

static GridEntry g_grid_table[] = {
    make_grid<4, 6>(), make_grid<8, 5>(), make_grid<12, 4>(), make_grid<17, 3>(),
};
constexpr int kGridTable = sizeof(g_grid_table) / sizeof(g_grid_table[0]);

int grid_choose(int64_t d, int* idx, int* G, int* stages, size_t* smem_out) {
  int dev = 0, sms = 0, optin = 0;
  SYSCD_CUDA_TRY(cudaGetDevice(&dev));
  SYSCD_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SYSCD_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  for (int i = 0; i < kGridTable; ++i) {
    const int rows = 416 * g_grid_table[i].rr;
    const int64_t g = (d + rows - 1) / rows;
    if (g > sms) continue;
    const size_t fixed = grid_smem(0, rows).total + 1024;
    int s = (int)(((size_t)optin - 1024 - fixed) / ((size_t)rows * 4));
    s = std::min(s, 8);
    if (s < 3) continue;
    *idx = i;
    *G = (int)g;
    *stages = s;
    *smem_out = grid_smem(s, rows).total;
    return SYSCD_OK;
  }
  set_error("no grid configuration covers d=%lld", (long long)d);
  return SYSCD_EINVAL;
}

int64_t grid_workspace_bytes(int G) {
  return (int64_t)kGNB * G * kGRec * 8;
}

static void* g_grid_dbg = nullptr;

int grid_launch(const syscd_dense_epoch_args* e, void* workspace, int64_t ws_bytes,
                cudaStream_t stream) {
  int idx, G, stages;
  size_t smem;
  int st = grid_choose(e->d, &idx, &G, &stages, &smem);
  if (st) return st;
  if (ws_bytes < grid_workspace_bytes(G) || !workspace) {
    set_error("syscd_dense_epoch: grid workspace too small");
    return SYSCD_EINVAL;
  }
  if (e->iid) {
    set_error("iid sampling is not supported when d needs the grid-wide kernel");
    return SYSCD_EINVAL;
  }
  const GridEntry& ge = g_grid_table[idx];
  SYSCD_CUDA_TRY(cudaFuncSetAttribute(ge.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  GridArgs A;
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
  A.stages = stages;
  A.evict_first = ((double)e->lda * 4.0 * (double)e->n_store) > 64.0 * 1024 * 1024 ? 1 : 0;
  A.out = e->partials;
  A.recs = (unsigned long long*)workspace;
  A.status = e->status;
  A.dbg = (unsigned long long*)g_grid_dbg;
  SYSCD_CUDA_TRY(cudaMemsetAsync(A.recs, 0, grid_workspace_bytes(G), stream));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(512, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {&A};
  SYSCD_CUDA_TRY(cudaLaunchKernelExC(&cfg, ge.fn, params));
  return SYSCD_OK;
}

}  // namespace syscd

// Debug hook (not part of the header ABI): device buffer of >= 1024*8 uint64
// receiving %globaltimer stamps of CTA 0 for the first partition's events.
extern "C" void syscd_debug_set_grid_timeline(void* device_buffer) {
  syscd::g_grid_dbg = device_buffer;
}
