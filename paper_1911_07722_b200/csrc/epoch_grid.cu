// Grid-wide SySCD round for tall columns (d too large for one cluster's
// registers, e.g. BASELINE config 3: d = 1M).
//
// Same semantics as epoch_dense.cu (solvers.py:289-334): partitions run their
// chains lin = x_j . w, alpha_j <- step, w += a delta x_j on a private replica
// w = u + a dv.  Here ALL CTAs of a cooperative grid work on one partition at
// a time; CTA c owns rows [c*CTA_ROWS, (c+1)*CTA_ROWS) and every coordinate's
// dot product is reduced across the grid through global memory.
//
// Blocked lookahead (exact in real arithmetic).  Columns are taken BB at a
// time ("blocks"); when block e is staged, the updates of blocks <= e-LL-1 are
// already applied to w, and each CTA publishes, for its rows,
//     s_i      = x_{e,i} . w                      i < BB
//     gin(i,k) = x_{e,i} . x_{e,k}                k < i       (in-block Gram)
//     gx(l,i,k)= x_{e,i} . x_{e-l,k}              l = 1..LL   (cross-block Gram)
// Block e-LL is then resolved from the grid totals one column at a time:
//     lin_i = S_i + a sum_{l,k} delta_{e-LL-l,k} GX(l,i,k) + a sum_{k<i} delta_{e-LL,k} GIN(i,k)
// and w += a sum_i delta_i x_{e-LL,i}.  The last LL+1 blocks live in a
// register ring, so every Gram term is an FMA.  BB amortises the per-event
// synchronisation (CTA reduction, publication, grid gather) over BB columns;
// LL hides the grid-reduction latency behind LL events.
//
// Partials are published as 64-bit words (tag << 32 | float bits), one word
// per value, component-major: the word is single-copy atomic, so a reader that
// sees the expected tag also sees the value -- no counter, fence or acquire
// round trip.  Two reducer warps gather alternate events (each lane loads its
// CTAs' words of every component at once, warp vote on the tags), sum the G
// records in a fixed order and hand the totals to the math warps through an
// mbarrier.  Every CTA sums identically, so all CTAs take bit-identical steps
// and the result is deterministic.  Partitions run one after another; at a
// partition end the pipeline drains, (w-u)/a is folded into `out` (each row
// has exactly one writer) and w is reset to u.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace syscd {

constexpr int kGNB = 16;    // global record slots (events), > 2*LL+2
constexpr int kGMeta = 64;  // metadata ring (columns)
constexpr int kGTot = 8;    // totals ring in shared memory (events), > LL+1
constexpr int kGVal = 32;   // max values per event record
constexpr int kGRecent = 64;  // iid: recently resolved (j, alpha) per math warp, >= prefetch lead
constexpr int kGRed = 8;      // CTA-reduction slots (events)
#ifndef SYSCD_GRID_RSLOTS
#define SYSCD_GRID_RSLOTS 1  // events in flight per reducer warp (2: no gain measured)
#endif
#ifndef SYSCD_GRID_CHAINS
#define SYSCD_GRID_CHAINS 1  // accumulator chains per partial value
#endif
#ifndef SYSCD_GRID_TSUM
#define SYSCD_GRID_TSUM 1  // reducer: all totals in one shuffle-transposed warp sum
#endif
// Fixed-point exchange (default): the grid totals are summed by the L2 atomic
// units.  Every CTA adds (llrint(partial * 2^shift) << 8) + 1 into the event's
// NS accumulator words with red.add.u64; integer addition is associative, so
// the total is independent of arrival order (bit-identical in every CTA and
// run to run), and the low byte counts the contributions: a word whose low
// byte advanced by G since the slot's previous event is complete.  A reducer
// polls ONE 32-byte sector per event instead of G records (publish -> totals
// across 145 CTAs: 1.55-1.8 us against 2.9-3.1 us, scripts/grid_sync.cu, and
// no poll traffic competing with the A stream).  The shifts are powers of two
// derived from Cauchy-Schwarz bounds every CTA computes identically:
//   Gram words   |x_e . x_k| <= sqrt(q_e max_j q_j)
//   s words      |x_e . w|  <= sqrt(q_e) ||w||, with ||w||^2 tracked exactly
//                from the resolved steps (||w + t x||^2 = ||w||^2 + t (2 x.w +
//                t q)), starting from d max_i |u_i|^2.
// (q_e: the event's own column norm, so columns of very different scale keep
// their relative precision.)  The sums over CTAs obey the same bounds, so 55
// bits never overflow; the resolution is >= 2^-52 of the bound, far below the
// fp32 rounding of the partials themselves.  SYSCD_GRID_FXP=0 builds the tagged-float records.
#ifndef SYSCD_GRID_FXP
#define SYSCD_GRID_FXP 1
#endif
// reducer poll back-off (ns).  The fixed-point reducer polls one sector, so a
// short back-off costs no L2 bandwidth and the totals are seen sooner (config
// 3, LL = 2: 0 / 32 / 100 / 256 ns -> 5.27 / 5.28 / 5.28 / 5.38 ms); the
// tagged-record reducer (G records per poll) keeps 256.
#ifndef SYSCD_GRID_SLEEP
#define SYSCD_GRID_SLEEP (SYSCD_GRID_FXP ? 32 : 256)
#endif
#ifndef SYSCD_GRID_LATE_RELEASE
#define SYSCD_GRID_LATE_RELEASE 1  // release a ring stage after the partials consumed it (no proxy fence)
#endif
constexpr int kGSlotWords = 32;  // fixed-point: 64-bit words per event slot (one 256-byte line pair)

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
  int32_t iid;
  int32_t stages;
  int32_t evict_first;
  int64_t cta_rows;          // rows per CTA (<= NTC*RR, a multiple of 4)
  float* out;                // [d] summed replicas (one worker row)
  unsigned long long* recs;  // [kGNB][NS][G] tagged partials, zeroed before launch
  int32_t* status;
  unsigned long long* dbg;   // optional timeline (CTA 0)
};

__device__ __forceinline__ unsigned long long gtimer_g() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct GridSmem {
  size_t ring, full, empty, totbar, tot, red, meta, recent, prev, total;
};

__host__ __device__ inline size_t galign(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline GridSmem grid_smem(int stages, int cta_rows, int ns, int iid) {
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
  o += kGTot * kGVal * 4;
  L.red = o;
  o += (size_t)kGRed * 16 * ns * 4;
  o = galign(o, 16);
  L.meta = o;
  o += kGMeta * 16;
  L.recent = o;
  if (iid) o += 16 * kGRecent * 8;  // iid only: one ring per math warp (<= 16 warps)
  L.prev = o;
#if SYSCD_GRID_FXP
  o += (size_t)kGNB * ns * 8;  // accumulator words at each slot's previous event
#endif
  L.total = galign(o, 128);
  return L;
}

// A partial is one 64-bit word (tag << 32 | float bits).
__device__ __forceinline__ void st_tagged(unsigned long long* p, uint32_t tag, float v) {
  const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

__device__ __forceinline__ unsigned long long ld_tagged(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}

__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long w) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

// Two fp32 FMAs in one instruction (FFMA2 on sm_100): same IEEE results per
// lane as two FFMAs, half the issue slots.
#ifndef SYSCD_GRID_F2
#define SYSCD_GRID_F2 2  // 0 never, 1 always, 2 where it measured faster (the LL = 2 wide-warp instance)
#endif
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long p;
  asm("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(lo), "f"(hi));
  return p;
}
__device__ __forceinline__ void unpack2(unsigned long long p, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Biased exponent of a non-negative float, floored at 2^-60 (zero columns,
// w = 0): keeps every shift below in the normal range.
__device__ __forceinline__ int fexp60(float v) {
  const int e = __float_as_int(v) >> 23;
  return e < 67 ? 67 : e;
}
// 2^-shift for a value bounded by sqrt(A B), A < 2^(ea-126), B < 2^(eb-126)
// (ea, eb biased exponents): shift = 52 - ceil(log2 of the bound), so the
// scaled value stays below 2^52.  Publisher and decoders evaluate this same
// integer expression on the same bits.
__device__ __forceinline__ float inv_scale(int ea, int eb) {
  return __int_as_float((127 - 52 + ((ea + eb - 251) >> 1)) << 23);
}
__device__ __forceinline__ float recip_pow2(float p) {  // 1/p for a normal power of two
  return __int_as_float(0x7F000000 - __float_as_int(p));
}

// 2^sh as a float (sh clamped to the normal range) and the power-of-two pair
// (scale, 1/scale) for a bound whose biased float exponent sum is known
__device__ __forceinline__ float pow2f(int sh) {
  sh = sh < -100 ? -100 : (sh > 100 ? 100 : sh);
  return __int_as_float((sh + 127) << 23);
}

// Sum NV values (NV a power of two <= 32) over a warp with log2(NV) halving
// exchanges followed by the remaining butterfly: NV-1 + 5-log2(NV) shuffles
// instead of 5*NV.  On return v[0] of lane l holds the warp total of value
// multi_index<NV>(l) (identical in every lane of an aligned group of 32/NV).
template <int NV>
__device__ __forceinline__ float warp_sum_multi(float (&v)[NV], int lane) {
  int cnt = NV;
  int off = 16;
#pragma unroll
  for (int step = 0; step < 5; ++step) {
    if (cnt > 1) {
      const int half = cnt / 2;
      const bool upper = (lane & off) != 0;
#pragma unroll
      for (int k = 0; k < NV / 2; ++k) {
        if (k < half) {
          const float send = upper ? v[k] : v[k + half];
          const float keep = upper ? v[k + half] : v[k];
          v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      cnt = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
    off >>= 1;
  }
  return v[0];
}

template <int NV>
__host__ __device__ constexpr int multi_index(int lane) {
  int idx = 0, cnt = NV, off = 16;
  for (int step = 0; step < 5 && cnt > 1; ++step) {
    cnt /= 2;
    if (lane & off) idx += cnt;
    off >>= 1;
  }
  return idx;
}

__host__ __device__ constexpr int pow2_at_least(int x) {
  int p = 1;
  while (p < x) p *= 2;
  return p;
}

template <int BB, int LL>
struct GridLayout {
  static constexpr int kS = 0;
  static constexpr int kIn = BB;
  static constexpr int kX = BB + BB * (BB - 1) / 2;
  static constexpr int kNS = kX + LL * BB * BB;
  __host__ __device__ static constexpr int gin(int i, int k) { return kIn + i * (i - 1) / 2 + k; }
  __host__ __device__ static constexpr int gx(int l, int i, int k) {
    return kX + ((l - 1) * BB + i) * BB + k;
  }
};

// KIND: the step compiled in (SYSCD_RIDGE also serves the primal-logistic
// surrogate; the fp64 Newton exists only in the logistic-dual instance).
// IID: with-replacement sampling (the recently-resolved ring).  Fixing both
// at compile time takes their branches out of the event loop, whose
// instruction count bounds this kernel (config 3: 6.51 -> 6.31 ms).
// EARLY (BB = 1): one more register slot; column e+1 is copied to registers and
// its Gram cross terms are accumulated right after event e is published, i.e.
// while the CTA would otherwise wait for grid totals.  Only the s-term FMAs of a
// block (the ones that need the updated w) then sit between the arrival of the
// totals and the next publication, which is the chain that bounds the grid.
template <int RR, int BB, int LL, int KIND, bool IID, int NWM, int NWT, bool EARLY = false>
__global__ void __launch_bounds__(NWT * 32, 1) k_grid_epoch(GridArgs A) {
  static_assert(!EARLY || (BB == 1 && RR % 2 == 0 && SYSCD_GRID_FXP && SYSCD_GRID_LATE_RELEASE),
                "early staging: one column per event, fixed-point exchange, late release");
  // NWM math warps + the producer + NRED reducer warps = NWT warps
  constexpr int NTC = NWM * 32;
  constexpr int NRED = NWT - NWM - 1;
  constexpr int NRW = NRED;
  static_assert(NRED >= 1, "no reducer warp");
  constexpr int NWC = NTC / 32;
  constexpr int NSLOT = LL + 1 + (EARLY ? 1 : 0);
#ifndef SYSCD_GRID_PUBW
#define SYSCD_GRID_PUBW 2  // a warp whose scheduler it shares with a helper warp only (config 3: 5.22 -> 5.05 ms against warp 0)
#endif
  constexpr int PUBW = SYSCD_GRID_PUBW < NWC ? SYSCD_GRID_PUBW : 0;  // the publishing math warp
  // packed FMAs (config 3: 5.43 -> 5.38 ms with LL = 2; with LL = 3 they cost registers: 5.48 -> 5.60)
  constexpr bool F2 = SYSCD_GRID_F2 == 1 || (SYSCD_GRID_F2 == 2 && NWM == 6 && LL == 2 && BB == 1);
  static_assert(!F2 || (RR % 2 == 0 && SYSCD_GRID_CHAINS == 1), "packed FMAs: even RR, one chain");
  using Lay = GridLayout<BB, LL>;
  constexpr int NS = Lay::kNS;
  static_assert(NS <= kGVal, "event record too large");
  constexpr int NP = pow2_at_least(NS);
  constexpr int CTA_ROWS = NTC * RR;
  // record layout of one event: CTA-major (word cta * NS + c), so one CTA's
  // NS words share a 32-byte sector and few CTAs write into one L2 line.
  // (The component-major layout c * G + cta put 16 writers on every line and
  // every reducer's polls on the same few lines: config 3 ran at 12-18 ms per
  // epoch instead of 8.3, depending on how the CTAs happened to convoy.)
#define GREC_IDX(c, cta_) ((size_t)(cta_) * NS + (c))

  extern __shared__ __align__(128) unsigned char smem[];
  const int S = A.stages;
  const GridSmem Lo = grid_smem(S, CTA_ROWS, NS, IID ? 1 : 0);
  float* ring = reinterpret_cast<float*>(smem + Lo.ring);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lo.full);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + Lo.empty);
  uint64_t* totbar = reinterpret_cast<uint64_t*>(smem + Lo.totbar);
  float* tot = reinterpret_cast<float*>(smem + Lo.tot);
  float* red = reinterpret_cast<float*>(smem + Lo.red);
  int4* meta = reinterpret_cast<int4*>(smem + Lo.meta);
  int2* recent = reinterpret_cast<int2*>(smem + Lo.recent);
#if SYSCD_GRID_FXP
  unsigned long long* prevw = reinterpret_cast<unsigned long long*>(smem + Lo.prev);
#endif

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int G = gridDim.x;
  const int cta = blockIdx.x;
  // a CTA's slice may be shorter than the NTC*RR rows its threads can hold, so
  // the grid covers d with every SM (the rows past the slice stay zero)
  const int64_t cta_rows = A.cta_rows;
  const int64_t row0 = (int64_t)cta * cta_rows;
  const int64_t d = A.d;
  const int64_t s_begin = A.wp[0];
  const int64_t s_end = A.wp[A.n_parts];

  for (int i = tid; i < S * CTA_ROWS; i += blockDim.x) ring[i] = 0.f;
  // every writer orders its generic-proxy zeros before the TMA (async
  // proxy) fills that follow the barrier; one fence by the issuing thread
  // does not cover the other threads' writes
  fence_proxy_async();
  if (IID)
    for (int i = tid; i < 16 * kGRecent; i += blockDim.x) recent[i] = make_int2(-1, 0);
#if defined(SYSCD_TRACE) && defined(SYSCD_TRACE_LIGHT)
  if (A.dbg && tid == 0) {  // SM of every CTA (scripts/grid_skew.py)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    A.dbg[8192 + 2 * 1024 * 160 + cta] = smid;
  }
#endif
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

#if SYSCD_GRID_FXP
  // ---- the launch's fixed-point bounds (identical in every CTA: max is
  // order-independent).  qmax over the columns of this launch; wmax over u
  // (every partition starts from w = u), exchanged once through the workspace.
  float qmax_b, w2_init;
  {
    float* scr = red;  // scratch before the event loop uses it
    float qm = 0.f, wm = 0.f;
    for (int64_t q = s_begin + tid; q < s_end; q += blockDim.x)
      qm = fmaxf(qm, fabsf(__ldg(A.sq + A.seq[q])));
    const int64_t r_end = min(d, row0 + cta_rows);
    for (int64_t r = row0 + tid; r < r_end; r += blockDim.x) wm = fmaxf(wm, fabsf(__ldg(A.u + r)));
    qm = warp_max(qm);
    wm = warp_max(wm);
    if (lane == 0) {
      scr[warp] = qm;
      scr[32 + warp] = wm;
    }
    __syncthreads();
    unsigned int* gw = reinterpret_cast<unsigned int*>(A.recs + (size_t)kGNB * kGSlotWords);
    if (tid == 0) {
      for (int q = 1; q < NWT; ++q) {
        qm = fmaxf(qm, scr[q]);
        wm = fmaxf(wm, scr[32 + q]);
      }
      atomicMax(gw, __float_as_uint(wm));  // non-negative floats order like their bits
      __threadfence();
      atomicAdd(gw + 2, 1u);
      unsigned int seen;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(gw + 2) : "memory");
      } while (seen < (unsigned)G);
      scr[0] = qm;
      scr[32] = __uint_as_float(__ldcg(gw));
    }
    __syncthreads();
    qmax_b = fmaxf(scr[0], 8.6736174e-19f);  // floors (2^-60) keep the shifts in the normal range
    const float wg = scr[32];
    w2_init = fmaxf((float)d * wg * wg, 8.6736174e-19f);
    __syncthreads();  // scr is the CTA-reduction ring from here on
  }
  // Scales (per event, from bounds every CTA evaluates identically):
  //   s words     |x_e . w|   <= sqrt(q_e ||w||^2)   (||w||^2: running maximum, tracked)
  //   Gram words  |x_e . x_k| <= sqrt(q_e q_max)
  // both relative to the event's own column norm, so badly scaled columns
  // (norms apart by many orders of magnitude) keep their relative precision.
  const int eqm = fexp60(qmax_b);
#endif

  // ------------------------------------------------------------ reducer state
  // Each reducer warp keeps RSL events in flight (reducer w, slot k takes
  // events r = w + NRW*k (mod NRW*RSL), in order per slot): a slot whose event
  // is complete sums it and hands it over while the other slots keep polling,
  // so the totals of consecutive events are gathered concurrently.  A word
  // carrying its event's tag is final: later polls reload only the words
  // still missing (the records of the CTAs that are behind).
  // registers: RSL*NS*NQ words; a lone reducer keeps two events in flight
  constexpr int NQ = 5;  // ceil(148 / 32) CTAs per lane
  constexpr int RSL = NS <= 4 ? (NRW == 1 && SYSCD_GRID_RSLOTS < 2 ? 2 : SYSCD_GRID_RSLOTS) : 1;
  // one poll pass over the slots; returns whether any slot is still open and
  // sets *prog when an event was handed over
  auto reduce_pass = [&](int64_t (&rs_ev)[RSL], unsigned long long (&wv)[RSL][NS][NQ],
                         int64_t events, bool* prog) -> bool {
    bool any = false;
#pragma unroll
    for (int k = 0; k < RSL; ++k) {
      const int64_t r = rs_ev[k];
      if (r >= events) continue;
      any = true;
      const unsigned long long* rec = A.recs + (size_t)(r % kGNB) * kGVal * G;
      const uint32_t tag = (uint32_t)(r + 1);
#pragma unroll
      for (int c = 0; c < NS; ++c)
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int cc = lane + 32 * q;
          if ((uint32_t)(wv[k][c][q] >> 32) != tag)
            wv[k][c][q] = cc < G ? ld_tagged(rec + GREC_IDX(c, cc))
                                 : ((unsigned long long)tag << 32);
        }
      bool ok = true;
#pragma unroll
      for (int c = 0; c < NS; ++c)
#pragma unroll
        for (int q = 0; q < NQ; ++q) ok &= (uint32_t)(wv[k][c][q] >> 32) == tag;
      if (!__all_sync(0xffffffffu, ok)) continue;
      float* t = tot + (r % kGTot) * kGVal;
#if SYSCD_GRID_TSUM
      // the NS totals in one shuffle-transposed reduction (NP-1 + 5-log2 NP
      // shuffles instead of 5 NS): the hand-over is on the grid's critical
      // path (last publication -> totals -> next resolve)
      {
        float pv[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          float acc = 0.f;
          if (c < NS) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc += __uint_as_float((uint32_t)wv[k][c][q]);
          }
          pv[c] = acc;
        }
        const float tv = warp_sum_multi<NP>(pv, lane);
        const int idx = multi_index<NP>(lane);
        if ((lane & (32 / NP - 1)) == 0 && idx < NS) t[idx] = tv;
      }
      __syncwarp();
#else
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc += __uint_as_float((uint32_t)wv[k][c][q]);
        acc = warp_sum(acc);
        if (lane == 0) t[c] = acc;
      }
#endif
      if (lane == 0) {
#ifdef SYSCD_TRACE
#ifndef SYSCD_TRACE_LIGHT
        if (A.dbg && cta == 0 && r < 1024) A.dbg[r * 8 + 5] = gtimer_g();
#endif
        if (A.dbg && r < 1024) A.dbg[8192 + 1024 * 160 + r * 160 + cta] = gtimer_g();
#endif
        mbar_arrive(&totbar[r % kGTot]);
      }
      __syncwarp();
      rs_ev[k] = r + NRW * RSL;
      *prog = true;
    }
    return any;
  };

  if (warp >= NWC) {
    int64_t events = 0;
    for (int p = 0; p < A.n_parts; ++p) events += (A.wp[p + 1] - A.wp[p] + BB - 1) / BB;
    const int rw = warp - NWC - 1;  // reducer index (producer: unused)
    int64_t rs_ev[RSL];
    unsigned long long wv[RSL][NS][NQ];
#pragma unroll
    for (int k = 0; k < RSL; ++k) {
      rs_ev[k] = rw + NRW * k;
#pragma unroll
      for (int c = 0; c < NS; ++c)
#pragma unroll
        for (int q = 0; q < NQ; ++q) wv[k][c][q] = 0ull;
    }
    // producer state (warp NWC)
    int64_t valid = d - row0;
    valid = valid < 0 ? 0 : (valid > cta_rows ? cta_rows : valid);
#ifdef SYSCD_GRID_NODATA  // experiment: the event chain without the A stream (wrong results)
    const uint32_t bytes = 0;
#else
    const uint32_t bytes = (uint32_t)(((valid + 3) / 4) * 16);
#endif
    const uint64_t policy = A.evict_first ? policy_evict_first() : policy_evict_last();
    uint32_t stage = 0, phase = 0;
    // coordinate ids, alpha and q of 32 columns at a time (lane-parallel), so
    // no dependent global load sits between two TMA issues
    int jreg = 0;
    float areg = 0.f, qreg = 0.f;
    int64_t s = s_begin, loaded = -1;
    // issue the TMA of column s (lane 0) once its stage is free
    auto produce = [&]() {
      const int64_t rel = s - s_begin;
      if ((rel & 31) == 0 && loaded != rel) {
        const int64_t q = s + lane;
        jreg = q < s_end ? A.seq[q] : 0;
        // alpha is written by CTA 0 during the epoch: read it from L2
        // (ld.cg), never from a possibly stale L1 line (iid redraws)
        areg = q < s_end ? __ldcg(A.alpha + jreg) : 0.f;
        qreg = q < s_end ? __ldg(A.sq + jreg) : 0.f;
        loaded = rel;
      }
      const int j = __shfl_sync(0xffffffffu, jreg, (int)(rel & 31));
      const float aj = __shfl_sync(0xffffffffu, areg, (int)(rel & 31));
      const float qj = __shfl_sync(0xffffffffu, qreg, (int)(rel & 31));
      if (lane == 0) {
        mbar_wait(&empty[stage], phase ^ 1u);
        meta[rel & (kGMeta - 1)] = make_int4(j, __float_as_int(aj), __float_as_int(qj),
                                             __float_as_int(step_inv(KIND, A.a, qj, A.lam_f)));
        if (bytes) {
          mbar_arrive_expect_tx(&full[stage], bytes);
          tma_load_1d(ring + (size_t)stage * CTA_ROWS, A.A + (int64_t)j * A.lda + row0, bytes,
                      &full[stage], policy);
        } else {
          mbar_arrive(&full[stage]);
        }
      }
      if (++stage == (uint32_t)S) {
        stage = 0;
        phase ^= 1u;
      }
      ++s;
      __syncwarp();
    };
    if (warp == NWC) {
      // ------------------------------------------------------------ producer
      while (s < s_end) produce();
    } else {
      // ------------------------------------------------------------ reducers
#if SYSCD_GRID_FXP
      // Lane l watches word l % NP of the event of group l / NP (events r with
      // r % D == group; D events per load instruction), and the events are
      // handed over in order.  A word is complete when its low byte advanced
      // by G since the slot's previous event; the event total is the
      // difference of the two 64-bit values (exact modulo 2^64) without that
      // byte.
      constexpr int D = 32 / NP;
      const int c = lane % NP, k = lane / NP;
      const bool act = c < NS;
      for (int i = lane; i < kGNB * NS; i += 32) prevw[i] = 0ull;
      __syncwarp();
      int64_t r_me = k, r0 = 0;
      unsigned long long cur = 0ull;
      bool have = false;
      const unsigned long long gcount = (unsigned long long)(G & 0xFF);
      if (rw > 0) r0 = events;  // one warp gathers every event (a sector per event)
      // hand over, in order, the events whose group has every word complete
      auto hand_over = [&](unsigned m) -> bool {
        bool prog = false;
        while (r0 < events) {
          const int g = (int)(r0 % D);
          const unsigned gm = (NP == 32 ? 0xffffffffu : ((1u << NP) - 1u)) << (g * NP);
          if ((m & gm) != gm) break;
          if (k == g && act) {
            unsigned long long* pw = prevw + (r0 % kGNB) * NS + c;
            const long long total = (long long)(cur - *pw) >> 8;
            *pw = cur;
            tot[(r0 % kGTot) * kGVal + c] = __ll2float_rn(total);
            have = false;
            r_me += D;
          }
          m &= ~gm;  // the group's next event has not been polled yet
          __syncwarp();
          if (lane == 0) {
#ifdef SYSCD_TRACE
            if (A.dbg && r0 < 1024) A.dbg[8192 + 1024 * 160 + r0 * 160 + cta] = gtimer_g();
#endif
            mbar_arrive(&totbar[r0 % kGTot]);
          }
          ++r0;
          prog = true;
        }
        return prog;
      };
      while (r0 < events) {
        if (act && !have && r_me < events && r_me <= r0 + LL + 1) {
          cur = ld_tagged(A.recs + (size_t)(r_me % kGNB) * kGSlotWords + c);
          have = ((cur - prevw[(r_me % kGNB) * NS + c]) & 0xFFull) == gcount;
        }
        if (!hand_over(__ballot_sync(0xffffffffu, have || !act))) __nanosleep(SYSCD_GRID_SLEEP);
      }
#else
      for (;;) {
        bool prog = false;
        if (!reduce_pass(rs_ev, wv, events, &prog)) break;
        if (!prog) __nanosleep(SYSCD_GRID_SLEEP);
      }
#endif
    }
  } else {
    // -------------------------------------------------------------- math warps
    const int64_t rem = min(cta_rows, d - row0) - tid;
    const int rmax = rem <= 0 ? 0 : (int)min((int64_t)RR, (rem + NTC - 1) / NTC);
    const float* ub = A.u + row0 + tid;
    float* outp = A.out + row0 + tid;
    float w[RR];
    float xr[NSLOT][BB][RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) w[r] = r < rmax ? ub[r * NTC] : 0.f;
#pragma unroll
    for (int sl = 0; sl < NSLOT; ++sl)
#pragma unroll
      for (int b = 0; b < BB; ++b)
#pragma unroll
        for (int r = 0; r < RR; ++r) xr[sl][b][r] = 0.f;
    const float a = A.a;
    const float inv_a = (float)(1.0 / A.a_d);
#if SYSCD_GRID_FXP
    float w2 = w2_init, w2max = w2_init;  // ||w||^2 (tracked) and its running maximum
    int ewr[NSLOT];  // exponent of the ||w||^2 bound the event in each register slot was scaled with
#pragma unroll
    for (int sl = 0; sl < NSLOT; ++sl) ewr[sl] = 127;
    // column (within the event) whose norm scales the publisher lane's word
    int pub_b = 0;
    if (lane < NS) {
      if (lane < BB) {
        pub_b = lane;
      } else if (lane < Lay::kX) {
        int idx = lane - BB, bb = 1;
        while (idx >= bb) {
          idx -= bb;
          ++bb;
        }
        pub_b = bb;
      } else {
        pub_b = ((lane - Lay::kX) / BB) % BB;
      }
    }
#endif
    uint32_t stage = 0, phase = 0;
#ifdef SYSCD_GRID_CLK
    long long clk_acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long clk_last = clock64();
#endif
    bool flushed = false;
    int64_t ebase = 0;  // event (publication) index of the partition's block 0
    // iid: the prefetched alpha of a coordinate drawn again within the
    // prefetch window is stale; every math warp keeps the same ring of the
    // last kGRecent resolved (j, alpha) and takes the newest match
    int2* rcnt_ring = recent + warp * kGRecent;
    uint32_t rcnt = 0;
    for (int p = 0; p < A.n_parts; ++p) {
      const int64_t col0 = A.wp[p] - s_begin;  // flattened column index of column 0
      const int m = (int)(A.wp[p + 1] - A.wp[p]);
      if (m == 0) continue;
      const int nb = (m + BB - 1) / BB;
      float dh[LL > 0 ? LL : 1][BB];  // deltas of the LL most recent resolved blocks
#pragma unroll
      for (int l = 0; l < (LL > 0 ? LL : 1); ++l)
#pragma unroll
        for (int b = 0; b < BB; ++b) dh[l][b] = 0.f;
#define XS_OLD(l) ((i + NSLOT - (l)) % NSLOT)
#define XS_RES ((i + NSLOT - LL) % NSLOT)
      if constexpr (EARLY) {
#if SYSCD_GRID_FXP && SYSCD_GRID_LATE_RELEASE
        // ---- early-staging loop (BB = 1, packed FMAs).  Block e lives in slot
        // e % NSLOT with NSLOT = LL + 2.  Iteration e:
        //   1. resolve block c = e - LL - 1 (totals of event c) and add its step to w
        //   2. s_e = x_e . w, reduce it with the cross terms accumulated earlier, publish
        //   3. copy column e + 1 into the slot block c just left and accumulate its
        //      cross terms x_{e+1} . x_{e+1-l}, l = 1..LL (no w involved), release its stage
        float pg[LL > 0 ? LL : 1];  // cross terms of the block published next
        static_assert(LL == 2, "early staging: LL = 2");
        auto stage_next = [&](float (&xn)[RR], const float (&xa)[RR], const float (&xb)[RR]) {
          mbar_wait(&full[stage], phase);
          const float* x = ring + (size_t)stage * CTA_ROWS + tid;
#pragma unroll
          for (int r = 0; r < RR; ++r) xn[r] = x[r * NTC];
          uint64_t* bar = &empty[stage];
          if (++stage == (uint32_t)S) {
            stage = 0;
            phase ^= 1u;
          }
          unsigned long long ga = 0ull, gb = 0ull;
#pragma unroll
          for (int r = 0; r < RR; r += 2) {
            const unsigned long long xv = pack2(xn[r], xn[r + 1]);
            ga = ffma2(xv, pack2(xa[r], xa[r + 1]), ga);
            gb = ffma2(xv, pack2(xb[r], xb[r + 1]), gb);
          }
          float lo, hi;
          unpack2(ga, lo, hi);
          pg[0] = lo + hi;
          unpack2(gb, lo, hi);
          pg[1] = lo + hi;
          // every loaded register has been consumed by an FMA: release the stage
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];  // after %1"
                         ::"r"(smem_addr(bar)), "f"(pg[0]) : "memory");
        };
        stage_next(xr[0][0], xr[NSLOT - 1][0], xr[NSLOT - 2][0]);
        for (int e0 = 0; e0 < nb + LL + 1; e0 += NSLOT) {
#pragma unroll
          for (int i = 0; i < NSLOT; ++i) {
            const int e = e0 + i;
            if (e < nb + LL + 1) {
              const int SR = (i + 1) % NSLOT;  // slot of block e - LL - 1, then of block e + 1
              if (e >= LL + 1) {
                // ---- 1. resolve block c
                const int c = e - LL - 1;
                const int64_t cpub = ebase + c;
                mbar_wait(&totbar[cpub % kGTot], (uint32_t)((cpub / kGTot) & 1));
                const float* t = tot + (cpub % kGTot) * kGVal;
                const int4 mt = meta[(col0 + c) & (kGMeta - 1)];
                const int j = mt.x;
                float aj = __int_as_float(mt.y);
                const float qj = __int_as_float(mt.z);
                const int eqj = fexp60(qj);
                const float aG = a * inv_scale(eqj, eqm);
                float lin = t[0] * inv_scale(eqj, ewr[SR]);
#pragma unroll
                for (int l = 1; l <= LL; ++l) lin = fmaf(aG * dh[l - 1][0], t[l], lin);
                if (IID) {
                  const int2 r0 = rcnt_ring[(rcnt - 1 - lane) & (kGRecent - 1)];
                  const int2 r1 = rcnt_ring[(rcnt - 33 - lane) & (kGRecent - 1)];
                  const unsigned m0 = __ballot_sync(0xffffffffu, r0.x == j);
                  const unsigned m1 = __ballot_sync(0xffffffffu, r1.x == j);
                  if (m0 | m1) {
                    const int kk = m0 ? __ffs(m0) - 1 : 32 + __ffs(m1) - 1;
                    aj = __int_as_float(rcnt_ring[(rcnt - 1 - kk) & (kGRecent - 1)].y);
                  }
                }
                float an;
                if (KIND == SYSCD_LOGISTIC_DUAL) {
                  an = (float)coord_step(SYSCD_LOGISTIC_DUAL, (double)lin, A.a_d, (double)qj, A.lam,
                                         (double)aj, A.n_coords);
                } else {
                  an = coord_step_fr(KIND, lin, __int_as_float(mt.w), A.lam_f, aj, A.inv_n_f);
                }
                float dc = 0.f;
                if (isfinite(an)) {
                  dc = an - aj;
                  const float tq = a * dc;
                  w2 = fmaf(tq, fmaf(tq, qj, lin + lin), w2);
                  w2max = fmaxf(w2max, w2);
                  if (cta == 0 && tid == 0) __stcg(A.alpha + j, an);
                } else if (cta == 0 && tid == 0) {
                  atomicOr(A.status, SYSCD_ENONFINITE);
                }
                if (IID) {
                  __syncwarp();
                  if (lane == 0) rcnt_ring[rcnt & (kGRecent - 1)] = make_int2(j, __float_as_int(aj + dc));
                  __syncwarp();
                  ++rcnt;
                }
#pragma unroll
                for (int l = LL - 1; l > 0; --l) dh[l][0] = dh[l - 1][0];
                dh[0][0] = dc;
                const float sd = a * dc;
                const unsigned long long sd2 = pack2(sd, sd);
#pragma unroll
                for (int r = 0; r < RR; r += 2) {
                  const unsigned long long wn =
                      ffma2(sd2, pack2(xr[SR][0][r], xr[SR][0][r + 1]), pack2(w[r], w[r + 1]));
                  unpack2(wn, w[r], w[r + 1]);
                }
              }
              if (e < nb) {
                // ---- 2. s_e with the updated w, reduce, publish
                unsigned long long s2 = 0ull;
#pragma unroll
                for (int r = 0; r < RR; r += 2)
                  s2 = ffma2(pack2(xr[i][0][r], xr[i][0][r + 1]), pack2(w[r], w[r + 1]), s2);
                float pv[NP];
                {
                  float lo, hi;
                  unpack2(s2, lo, hi);
                  pv[0] = lo + hi;
                }
#pragma unroll
                for (int k = 1; k < NP; ++k) pv[k] = k < NS ? pg[k - 1] : 0.f;
                const int64_t pub = ebase + e;
                float* rslot = red + (size_t)(pub % kGRed) * 16 * NS;
                const float tv = warp_sum_multi<NP>(pv, lane);
                {
                  const int idx = multi_index<NP>(lane);
                  if ((lane & (32 / NP - 1)) == 0 && idx < NS) rslot[warp * NS + idx] = tv;
                }
                ewr[i] = __float_as_int(w2max) >> 23;
                const int eqe = fexp60(__int_as_float(meta[(col0 + e) & (kGMeta - 1)].z));
                named_bar_sync(1, NTC);
                if (warp == PUBW && lane < NS) {
                  float v = 0.f;
                  for (int q = 0; q < NWC; ++q) v += rslot[q * NS + lane];
                  const float sc = recip_pow2(inv_scale(eqe, lane < BB ? ewr[i] : eqm));
                  float f = v * sc;
                  if (!(fabsf(f) < 1.8014399e16f)) {  // 2^54: NaN/Inf or bounds violated (bad sq)
                    atomicOr(A.status, SYSCD_ENONFINITE);
                    f = 0.f;
                  }
                  red_add_u64(A.recs + (size_t)(pub % kGNB) * kGSlotWords + lane,
                              ((unsigned long long)__float2ll_rn(f) << 8) + 1ull);
                }
              }
              if (e + 1 < nb) {
                // ---- 3. column e + 1 and its cross terms (slots of blocks e, e-1, ...)
                stage_next(xr[SR][0], xr[i][0], xr[(i + NSLOT - 1) % NSLOT][0]);
              }
            }
          }
        }
#endif
      } else
      for (int e0 = 0; e0 < nb + LL; e0 += NSLOT) {
#pragma unroll
        for (int i = 0; i < NSLOT; ++i) {
          const int e = e0 + i;  // e % NSLOT == i: register slot of block e
          if (e < nb + LL) {
#if defined(SYSCD_TRACE) && !defined(SYSCD_TRACE_LIGHT)
            const bool dbg = A.dbg && cta == 0 && tid == 0 && p == 0 && e < 1024;
            // all-CTA stamps (thread 0 of each CTA): [e][cta][k]
            unsigned long long* da = (A.dbg && tid == 0 && p == 0 && e < 1024)
                                         ? A.dbg + 8192 + 2 * 1024 * 160 + ((size_t)e * 160 + cta) * 8
                                         : nullptr;
#define GSTAMP(k)                          \
  do {                                     \
    if (dbg) A.dbg[e * 8 + k] = gtimer_g(); \
    if (da) da[k] = gtimer_g();            \
  } while (0)
#else
            // no stamps in production: the runtime-gated CTA-0 stamps cost 13%
            // of config 3 (7.49 -> 6.53 ms) once the grid stopped convoying
#define GSTAMP(k) \
  do {            \
  } while (0)
#endif
#ifdef SYSCD_GRID_CLK  // experiment: per-phase SM cycles of a few warps (printf at the end)
#define GCLK(k)                         \
  do {                                  \
    const long long t_ = clock64();     \
    clk_acc[k] += t_ - clk_last;        \
    clk_last = t_;                      \
  } while (0)
#else
#define GCLK(k) \
  do {          \
  } while (0)
#endif
            GSTAMP(0);
            GCLK(0);
            // One iteration: stage block e and publish its partials, then resolve
            // block e - LL from its grid totals.  (Resolving first, so that the
            // warp reduction and the axpy share a basic block, was measured:
            // 5.80 against 5.47 ms on config 3 -- the publication then waits for
            // one more set of totals.)
            if (e < nb) {
              // ---- stage block e and publish its partials
              // A ring stage is copied to registers and released LATE: after
              // the warp reduction below, through an arrive that takes the
              // reduced value as an operand.  Every loaded register has then
              // been consumed by an FMA the warp issued, so the loads have
              // landed and the TMA refill (async proxy) cannot overtake them
              // -- an arrive right after the loads can (config 3 went
              // nondeterministic once the grid ran fast enough), and the
              // proxy fence that prevents it serialises loads and FMAs
              // (SYSCD_GRID_LATE_RELEASE=0: 5.72 against 5.47 ms on config 3).
              auto load_col = [&](float (&dst)[RR]) -> uint64_t* {
                mbar_wait(&full[stage], phase);
                const float* x = ring + (size_t)stage * CTA_ROWS + tid;
#pragma unroll
                for (int r = 0; r < RR; ++r) dst[r] = x[r * NTC];
                uint64_t* bar = &empty[stage];
#if !SYSCD_GRID_LATE_RELEASE
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar);
#endif
                if (++stage == (uint32_t)S) {
                  stage = 0;
                  phase ^= 1u;
                }
                return bar;
              };
              GCLK(7);
              uint64_t* rel[BB];
#pragma unroll
              for (int b = 0; b < BB; ++b) {
                if (e * BB + b < m) {
                  rel[b] = load_col(xr[i][b]);
                } else {
                  rel[b] = nullptr;
#pragma unroll
                  for (int r = 0; r < RR; ++r) xr[i][b][r] = 0.f;
                }
              }
              GSTAMP(1);
              GCLK(1);
#ifdef SYSCD_GRID_DCHK
              if (A.dbg && ebase + e < 8192) {  // integer checksums of x_e and w per CTA
                unsigned int cx = 0, cw = 0;
#pragma unroll
                for (int r = 0; r < RR; ++r) {
                  cx += __float_as_uint(xr[i][0][r]) * (unsigned)(r + 1);
                  cw += __float_as_uint(w[r]) * (unsigned)(r + 1);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                  cx += __shfl_xor_sync(0xffffffffu, cx, o);
                  cw += __shfl_xor_sync(0xffffffffu, cw, o);
                }
                if (lane == 0) {
                  unsigned long long* cs = A.dbg + 8192 + 2 * 1024 * 160 + 1024 * 160 * 8 +
                                           8192 * 160 + 8192 * 160 * 4 + ((ebase + e) * 160 + cta) * 2;
                  atomicAdd(cs, (unsigned long long)cx);
                  atomicAdd(cs + 1, (unsigned long long)cw);
                }
              }
#endif
              // NCH independent accumulator chains per value (rows r with
              // r % NCH == h), summed in a fixed order: shorter FMA
              // dependency chains on the per-event critical path
              constexpr int NCH = SYSCD_GRID_CHAINS;
              float prc[NCH][NS];
#pragma unroll
              for (int h = 0; h < NCH; ++h)
#pragma unroll
                for (int k = 0; k < NS; ++k) prc[h][k] = 0.f;
#ifdef SYSCD_GRID_NOMATH  // experiment: data-delivery ceiling (wrong results)
              prc[0][0] = xr[i][0][0];
#else
              if constexpr (F2) {  // rows in pairs through FFMA2 (even / odd rows accumulate apart)
                unsigned long long p2[NS];
#pragma unroll
                for (int k = 0; k < NS; ++k) p2[k] = 0ull;
#pragma unroll
                for (int r = 0; r < RR; r += 2) {
#pragma unroll
                  for (int b = 0; b < BB; ++b) {
                    const unsigned long long xv = pack2(xr[i][b][r], xr[i][b][r + 1]);
                    p2[Lay::kS + b] = ffma2(xv, pack2(w[r], w[r + 1]), p2[Lay::kS + b]);
#pragma unroll
                    for (int k = 0; k < b; ++k)
                      p2[Lay::gin(b, k)] =
                          ffma2(xv, pack2(xr[i][k][r], xr[i][k][r + 1]), p2[Lay::gin(b, k)]);
#pragma unroll
                    for (int l = 1; l <= LL; ++l)
#pragma unroll
                      for (int k = 0; k < BB; ++k)
                        p2[Lay::gx(l, b, k)] =
                            ffma2(xv, pack2(xr[XS_OLD(l)][k][r], xr[XS_OLD(l)][k][r + 1]),
                                  p2[Lay::gx(l, b, k)]);
                  }
                }
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                  float lo, hi;
                  unpack2(p2[k], lo, hi);
                  prc[0][k] = lo + hi;
                }
              } else {
#pragma unroll
              for (int r = 0; r < RR; ++r) {
                float* pr = prc[r % NCH];
#pragma unroll
                for (int b = 0; b < BB; ++b) {
                  const float xv = xr[i][b][r];
                  pr[Lay::kS + b] = fmaf(xv, w[r], pr[Lay::kS + b]);
#pragma unroll
                  for (int k = 0; k < b; ++k)
                    pr[Lay::gin(b, k)] = fmaf(xv, xr[i][k][r], pr[Lay::gin(b, k)]);
#pragma unroll
                  for (int l = 1; l <= LL; ++l)
#pragma unroll
                    for (int k = 0; k < BB; ++k)
                      pr[Lay::gx(l, b, k)] =
                          fmaf(xv, xr[XS_OLD(l)][k][r], pr[Lay::gx(l, b, k)]);
                }
              }
              }
#endif
              float pr[NS];
#pragma unroll
              for (int k = 0; k < NS; ++k) {
                pr[k] = prc[0][k];
#pragma unroll
                for (int h = 1; h < NCH; ++h) pr[k] += prc[h][k];
              }
              GCLK(2);
              // warp totals (shuffle-transposed: NP-1 + 5-log2(NP) shuffles
              // instead of 5*NS), then one warp sums the warps' deposits in
              // warp order and publishes the CTA's record
              const int64_t pub = ebase + e;
              float* rslot = red + (size_t)(pub % kGRed) * 16 * NS;
              float pv[NP];
#pragma unroll
              for (int k = 0; k < NP; ++k) pv[k] = k < NS ? pr[k] : 0.f;
              const float tv = warp_sum_multi<NP>(pv, lane);
              GCLK(3);
#if SYSCD_GRID_LATE_RELEASE
              if (lane == 0) {
#pragma unroll
                for (int b = 0; b < BB; ++b)
                  if (rel[b])
                    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];  // after %1"
                                 ::"r"(smem_addr(rel[b])), "f"(tv) : "memory");
              }
#endif
              {
                const int idx = multi_index<NP>(lane);
                if ((lane & (32 / NP - 1)) == 0 && idx < NS) rslot[warp * NS + idx] = tv;
              }
              named_bar_sync(1, NTC);
#ifdef SYSCD_TRACE
              if (A.dbg && warp == PUBW && lane == 0 && pub < 1024)
                A.dbg[8192 + pub * 160 + cta] = gtimer_g();
#endif
#if SYSCD_GRID_FXP
              // this event's s-scale comes from the running bound on ||w||^2 (the w
              // of the partials above: every step resolved so far is tracked)
              ewr[i] = __float_as_int(w2max) >> 23;
#endif
              if (warp == PUBW && lane < NS) {
                float v = 0.f;
                for (int q = 0; q < NWC; ++q) v += rslot[q * NS + lane];
#if SYSCD_GRID_FXP
                const int eqe = fexp60(
                    __int_as_float(meta[(col0 + min(e * BB + pub_b, m - 1)) & (kGMeta - 1)].z));
                const float sc = recip_pow2(inv_scale(eqe, lane < BB ? ewr[i] : eqm));
                float f = v * sc;
                if (!(fabsf(f) < 1.8014399e16f)) {  // 2^54: NaN/Inf or bounds violated (bad sq)
                  atomicOr(A.status, SYSCD_ENONFINITE);
                  f = 0.f;
                }
                red_add_u64(A.recs + (size_t)(pub % kGNB) * kGSlotWords + lane,
                            ((unsigned long long)__float2ll_rn(f) << 8) + 1ull);
#else
                st_tagged(A.recs + (size_t)(pub % kGNB) * kGVal * G + GREC_IDX(lane, cta),
                          (uint32_t)(pub + 1), v);
#endif
#ifdef SYSCD_GRID_DCHK
                if (A.dbg && pub < 8192)  // every CTA's published partials
                  A.dbg[8192 + 2 * 1024 * 160 + 1024 * 160 * 8 + 8192 * 160 +
                        ((size_t)pub * 160 + cta) * 4 + lane] = __float_as_uint(v);
#endif
              }
            }
            GSTAMP(2);
            GCLK(5);
            if (e >= LL) {
              // ---- resolve block c = e - LL (register slot XS_RES)
              const int c = e - LL;
              const int64_t cpub = ebase + c;
              mbar_wait(&totbar[cpub % kGTot], (uint32_t)((cpub / kGTot) & 1));
              GSTAMP(3);
              GCLK(6);
              const float* t = tot + (cpub % kGTot) * kGVal;
              float dcur[BB];
#pragma unroll
              for (int b = 0; b < BB; ++b) {
                dcur[b] = 0.f;
                const int col = c * BB + b;
                if (col < m) {
                  const int4 mt = meta[(col0 + col) & (kGMeta - 1)];
                  const int j = mt.x;
                  float aj = __int_as_float(mt.y);
                  const float qj = __int_as_float(mt.z);
#if SYSCD_GRID_FXP
                  const int eqj = fexp60(qj);
                  const float aG = a * inv_scale(eqj, eqm);  // Gram totals decode inside a * delta
                  float lin = t[Lay::kS + b] * inv_scale(eqj, ewr[XS_RES]);
#else
                  const float aG = a;
                  float lin = t[Lay::kS + b];
#endif
#pragma unroll
                  for (int l = 1; l <= LL; ++l)
#pragma unroll
                    for (int k = 0; k < BB; ++k)
                      lin = fmaf(aG * dh[l - 1][k], t[Lay::gx(l, b, k)], lin);
#pragma unroll
                  for (int k = 0; k < b; ++k) lin = fmaf(aG * dcur[k], t[Lay::gin(b, k)], lin);
                  if (IID) {
                    const int2 r0 = rcnt_ring[(rcnt - 1 - lane) & (kGRecent - 1)];
                    const int2 r1 = rcnt_ring[(rcnt - 33 - lane) & (kGRecent - 1)];
                    const unsigned m0 = __ballot_sync(0xffffffffu, r0.x == j);
                    const unsigned m1 = __ballot_sync(0xffffffffu, r1.x == j);
                    if (m0 | m1) {
                      const int kk = m0 ? __ffs(m0) - 1 : 32 + __ffs(m1) - 1;
                      aj = __int_as_float(rcnt_ring[(rcnt - 1 - kk) & (kGRecent - 1)].y);
                    }
                  }
                  float an;
                  if (KIND == SYSCD_LOGISTIC_DUAL) {
                    an = (float)coord_step(SYSCD_LOGISTIC_DUAL, (double)lin, A.a_d, (double)qj, A.lam,
                                           (double)aj, A.n_coords);
                  } else {
                    an = coord_step_fr(KIND, lin, __int_as_float(mt.w), A.lam_f, aj,
                                       A.inv_n_f);
                  }
                  if (isfinite(an)) {
                    dcur[b] = an - aj;
#if SYSCD_GRID_FXP
                    {  // ||w + t x||^2 = ||w||^2 + t (2 x.w + t q), t = a delta
                      const float tq = a * dcur[b];
                      w2 = fmaf(tq, fmaf(tq, qj, lin + lin), w2);
                      w2max = fmaxf(w2max, w2);
                    }
#endif
                    if (cta == 0 && tid == 0) __stcg(A.alpha + j, an);
                  } else if (cta == 0 && tid == 0) {
                    atomicOr(A.status, SYSCD_ENONFINITE);
                  }
                  if (IID) {
                    __syncwarp();
                    if (lane == 0)
                      rcnt_ring[rcnt & (kGRecent - 1)] = make_int2(j, __float_as_int(aj + dcur[b]));
                    __syncwarp();
                    ++rcnt;
                  }
                }
              }
#pragma unroll
              for (int l = LL - 1; l > 0; --l)
#pragma unroll
                for (int b = 0; b < BB; ++b) dh[l][b] = dh[l - 1][b];
              if (LL > 0) {
#pragma unroll
                for (int b = 0; b < BB; ++b) dh[0][b] = dcur[b];
              }
#pragma unroll
              for (int b = 0; b < BB; ++b) {
                const float sd = a * dcur[b];
                if constexpr (F2) {
                  const unsigned long long sd2 = pack2(sd, sd);
#pragma unroll
                  for (int r = 0; r < RR; r += 2) {
                    const unsigned long long wn = ffma2(
                        sd2, pack2(xr[XS_RES][b][r], xr[XS_RES][b][r + 1]), pack2(w[r], w[r + 1]));
                    unpack2(wn, w[r], w[r + 1]);
                  }
                } else {
#pragma unroll
                  for (int r = 0; r < RR; ++r) w[r] = fmaf(sd, xr[XS_RES][b][r], w[r]);
                }
              }
            }
            GSTAMP(4);
            GCLK(8);
#if (defined(SYSCD_TRACE) && !defined(SYSCD_TRACE_LIGHT)) || defined(SYSCD_GRID_DCHK)
            if (A.dbg && tid == 0 && e >= LL && ebase + e - LL < 8192) {
              // every event's first delta per CTA (divergence check)
              A.dbg[8192 + 2 * 1024 * 160 + 1024 * 160 * 8 + (ebase + e - LL) * 160 + cta] =
                  ((unsigned long long)__float_as_uint(dh[0][0]) << 32) |
                  __float_as_uint(tot[((ebase + e - LL) % kGTot) * kGVal]);
            }
#endif
#if defined(SYSCD_TRACE) && !defined(SYSCD_TRACE_LIGHT)
            if (da && e >= LL) {
              const float* tt = tot + ((ebase + e - LL) % kGTot) * kGVal;
              da[5] = ((unsigned long long)__float_as_uint(dh[0][0]) << 32) | __float_as_uint(tt[0]);
              da[6] = ((unsigned long long)__float_as_uint(tt[1]) << 32) | __float_as_uint(tt[2]);
              da[7] = ((unsigned long long)__float_as_uint(w[0]) << 32) | __float_as_uint(tt[NS - 1]);
            }
#endif
          }
        }
      }
      ebase += nb;
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
#if SYSCD_GRID_FXP
      w2 = w2_init;
#endif
      flushed = true;
    }
    if (!flushed) {
#pragma unroll
      for (int r = 0; r < RR; ++r)
        if (r < rmax) outp[r * NTC] = 0.f;
    }
#ifdef SYSCD_GRID_CLK
    if (lane == 0 && (cta == 0 || cta == 77) && ebase > 0)
      printf("clk cta %d warp %d events %lld: loop %lld | wait-full+lds %lld | fma %lld | warpsum %lld | "
             "release+deposit+bar+publish %lld | wait-tot %lld | resolve+axpy %lld (cycles/event)\n",
             cta, warp, (long long)ebase, clk_acc[0] / ebase, (clk_acc[7] + clk_acc[1]) / ebase,
             clk_acc[2] / ebase, clk_acc[3] / ebase, clk_acc[5] / ebase, clk_acc[6] / ebase,
             clk_acc[8] / ebase);
#endif
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct GridEntry {
  int rr, bb, ll, ns, ntc, nthreads;
  const void* fn[4][2];  // [ridge / primal logistic, lasso, svm dual, logistic dual][iid]
};

template <int RR, int BB, int LL, int NWM, int NWT, bool EARLY, int KIND>
static void grid_fill(GridEntry& g, int k) {
  g.fn[k][0] = (const void*)&k_grid_epoch<RR, BB, LL, KIND, false, NWM, NWT, EARLY>;
  g.fn[k][1] = (const void*)&k_grid_epoch<RR, BB, LL, KIND, true, NWM, NWT, EARLY>;
}

template <int RR, int BB, int LL, int NWM = 13, int NWT = 16, bool EARLY = false>
static GridEntry make_grid() {
  GridEntry g{RR, BB, LL, GridLayout<BB, LL>::kNS, NWM * 32, NWT * 32, {}};
  grid_fill<RR, BB, LL, NWM, NWT, EARLY, SYSCD_RIDGE>(g, 0);
  grid_fill<RR, BB, LL, NWM, NWT, EARLY, SYSCD_LASSO>(g, 1);
  grid_fill<RR, BB, LL, NWM, NWT, EARLY, SYSCD_SVM_DUAL>(g, 2);
  grid_fill<RR, BB, LL, NWM, NWT, EARLY, SYSCD_LOGISTIC_DUAL>(g, 3);
  return g;
}

// (rows per thread, columns per event, lookahead events[, math warps]).  The
// first entry whose grid fits the GPU wins (SYSCD_GRID_CFG=<index>
// overrides).  14 math warps + one reducer warp (two events in flight) at 16
// rows per thread beat 13 warps + two reducers at 17 rows (config 3: 7.64 vs
// 8.39 ms per epoch); the other geometries measured on config 3 (DESIGN.md:
// BB=2 or 4 with less lookahead, L=2 or 4 at 16 rows, the producer and
// reducer in one warp) were slower and are not instantiated.
static GridEntry g_grid_table[] = {
    make_grid<4, 2, 2>(),
    make_grid<8, 2, 2>(),
    make_grid<12, 2, 1>(),
    make_grid<16, 1, 3, 14>(),
    // fewer, wider math warps: the per-warp event overhead (waits, warp
    // reductions, the redundant step) is paid by 6 warps instead of 14
    // (config 3: 6.34 -> 5.80 ms).  Measured and not kept:
    // <24,1,3,9 of 12 warps> 5.89, <22,1,3,10/12> 7.46, <27,1,2,8/12> 10.8,
    // <36,1,4,6/8> 7.44 ms (255 registers); fewer, longer slices
    // <38,1,3,6/8> (138 CTAs) 5.92, <40,...> (131) 5.99, <43,1,3,5/7> 6.39.
    // With the fixed-point exchange the totals arrive early enough for
    // LL = 2 (one FMA per row less, room for packed FMAs), and that instance is
    // bound by the exchange chain, so the early-staging loop (only the s-term
    // FMAs between totals and publication) is the one selected: config 3 at
    // 5.21 ms against 5.28 (LL = 2 without it) and 5.48 (LL = 3, bound by the
    // CTA's own work per event).  The other two stay reachable through
    // SYSCD_GRID_CFG=5 / 6 (ties go to the earlier entry).
#if SYSCD_GRID_FXP && SYSCD_GRID_LATE_RELEASE
    make_grid<36, 1, 2, 6, 8, true>(),
#endif
    make_grid<36, 1, 2, 6, 8>(),
    make_grid<36, 1, 3, 6, 8>(),
#ifdef SYSCD_GRID_EXPERIMENTS
    make_grid<36, 2, 1, 6, 8>(),
#endif
};
constexpr int kGridTable = sizeof(g_grid_table) / sizeof(g_grid_table[0]);

static void* g_grid_dbg = nullptr;

int grid_choose(int64_t d, int* idx, int* G, int* stages, size_t* smem_out, int64_t* cta_rows,
                int iid) {
  int dev = 0, sms = 0, optin = 0;
  SYSCD_CUDA_TRY(cudaGetDevice(&dev));
  SYSCD_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SYSCD_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const char* force = getenv("SYSCD_GRID_CFG");
  // the entry with the most CTAs (row slices) that still fits one wave wins;
  // ties go to the earlier entry (SYSCD_GRID_CFG=<index> overrides)
  constexpr int kNQ = 5;  // reducer lanes gather kNQ CTAs each (k_grid_epoch NQ)
  int best = -1, best_g = 0, best_s = 0;
  for (int i = 0; i < kGridTable; ++i) {
    if (force && atoi(force) != i) continue;
    const int rows = g_grid_table[i].ntc * g_grid_table[i].rr;
    const int64_t g = (d + rows - 1) / rows;
    if (g > sms || g > 32 * kNQ) continue;
    // feasibility with the iid layout (the larger one), so the geometry does
    // not depend on the sampling mode
    const size_t fixed = grid_smem(0, rows, g_grid_table[i].ns, 1).total;
    int s = (int)(((size_t)optin - fixed) / ((size_t)rows * 4));
    s = std::min(s, 8);
    if (s < g_grid_table[i].bb + 2) continue;
    if (g > best_g) {
      best = i;
      best_g = (int)g;
      best_s = s;
    }
  }
  if (best >= 0) {
    const int rows = g_grid_table[best].ntc * g_grid_table[best].rr;
    *idx = best;
    *G = best_g;
    // the kernel has no static shared memory: everything up to the opt-in
    // limit goes to the ring (the iid layout carries the recently-resolved
    // rings; without them config 3 gets an 8th stage)
    {
      const size_t fixed = grid_smem(0, rows, g_grid_table[best].ns, iid).total;
      best_s = std::min((int)(((size_t)optin - fixed) / ((size_t)rows * 4)), 8);
      if (const char* fs = getenv("SYSCD_GRID_STAGES")) best_s = std::min(best_s, atoi(fs));
    }
    *stages = best_s;
    *smem_out = grid_smem(best_s, rows, g_grid_table[best].ns, iid).total;
    // Slices are the entry's full capacity.  Spreading d over every SM
    // (148 slices of 6784 rows instead of 145 of 6912, 128-byte aligned or
    // not) measured slower on config 3: 6.01 against 5.80 ms per epoch.
    int64_t cr = rows;
    if (const char* fr = getenv("SYSCD_GRID_ROWS")) {  // experiments: shorter slices on more SMs
      const int64_t r = atoll(fr) / 4 * 4;
      if (r >= 4 && r <= rows && (d + r - 1) / r <= sms) cr = r;
    }
    if (cta_rows) *cta_rows = cr;
    *G = (int)((d + cr - 1) / cr);
    return SYSCD_OK;
  }
  set_error("no grid configuration covers d=%lld", (long long)d);
  return SYSCD_EINVAL;
}

int64_t grid_workspace_bytes(int G) { return (int64_t)kGNB * kGVal * (G + 1) * 8; }

int grid_launch(const syscd_dense_epoch_args* e, void* workspace, int64_t ws_bytes,
                cudaStream_t stream) {
  int idx, G, stages;
  size_t smem;
  int64_t cta_rows = 0;
  int st = grid_choose(e->d, &idx, &G, &stages, &smem, &cta_rows, e->iid ? 1 : 0);
  if (st) return st;
  if (ws_bytes < grid_workspace_bytes(G) || !workspace) {
    set_error("syscd_dense_epoch: grid workspace too small");
    return SYSCD_EINVAL;
  }
  const GridEntry& ge = g_grid_table[idx];
  const int ks = e->kind == SYSCD_LASSO ? 1
                 : e->kind == SYSCD_SVM_DUAL ? 2
                 : e->kind == SYSCD_LOGISTIC_DUAL ? 3 : 0;
  const void* fn = ge.fn[ks][e->iid ? 1 : 0];
  SYSCD_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  A.iid = e->iid;
  A.a = (float)e->a;
  A.lam_f = (float)e->lam;
  A.inv_n_f = (float)(1.0 / e->n_coords);
  A.a_d = e->a;
  A.lam = e->lam;
  A.n_coords = e->n_coords;
  A.kind = e->kind;
  A.stages = stages;
  A.evict_first = ((double)e->lda * 4.0 * (double)e->n_store) > 64.0 * 1024 * 1024 ? 1 : 0;
  A.cta_rows = cta_rows;
  A.out = e->partials;
  A.recs = (unsigned long long*)workspace;
  A.status = e->status;
  A.dbg = (unsigned long long*)g_grid_dbg;
#if SYSCD_GRID_FXP
  SYSCD_CUDA_TRY(cudaMemsetAsync(A.recs, 0, ((size_t)kGNB * kGSlotWords + 8) * 8, stream));
#else
  SYSCD_CUDA_TRY(cudaMemsetAsync(A.recs, 0, grid_workspace_bytes(G), stream));
#endif
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(ge.nthreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {&A};
  SYSCD_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, params));
  return SYSCD_OK;
}

}  // namespace syscd

// Debug hook (not part of the header ABI): device buffer of >= 1024*8 uint64
// receiving %globaltimer stamps of CTA 0 for the first partition's events.
extern "C" void syscd_debug_set_grid_timeline(void* device_buffer) {
  syscd::g_grid_dbg = device_buffer;
}
