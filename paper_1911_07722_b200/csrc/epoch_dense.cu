// Dense SySCD round on sm_100a.
//
// Reference semantics (pkg/src/syscd/solvers.py:289-334, 384-393): every
// partition p walks its coordinate sequence j_1..j_m; per coordinate
//     lin   = x_j . u + a x_j . dv          (u = lin_vec, dv = private replica)
//     alpha_j <- step(lin, a, q_j, lam, alpha_j)
//     dv   += delta x_j
// and the node replica becomes v + sum_p dv_p.
//
// B200 mapping (DESIGN.md section "dense epoch kernel"):
//  * a partition runs on one thread-block cluster of C CTAs; CTA `rank` owns
//    rows [rank*CTA_ROWS, (rank+1)*CTA_ROWS) of the shared vector;
//  * the replica lives in registers as w = u + a dv (one fp32 per owned row,
//    so lin = x_j . w and the axpy is w += a delta x_j); at the end of a
//    partition the cluster folds (w - u)/a into its slice of `partials`;
//  * one producer warp per CTA streams the CTA's slice of each column into a
//    ring of shared-memory stages with 1-D bulk TMA (cp.async.bulk +
//    mbarrier complete_tx), running ahead of the consumers by the ring depth;
//    the column sequence is known from the plan, so prefetch crosses bucket
//    and partition boundaries;
//  * consumer warps read each staged chunk twice (dot, then axpy) from smem,
//    reduce the dot warp -> CTA (named barrier) -> cluster (st.async of one
//    float into every peer's smem, completing the peer's mbarrier); every CTA
//    then sums the C partials in rank order, so lin is bit-identical across
//    the cluster and the step is computed redundantly in fp64;
//  * clusters process disjoint contiguous ranges of partitions (balanced by
//    update count) and accumulate their partitions' replicas into one
//    partials row each, in a fixed order: the result is deterministic.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace syscd {

struct DenseArgs {
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
  double a_d;
  double lam;
  float lam_f;
  float inv_n_f;
  double n_coords;
  int32_t kind;
  int32_t iid;
  int32_t stages;
  int32_t cluster;
  int32_t evict_first;
  float* partials;
  int64_t part_ld;
  int32_t* status;
  unsigned long long* dbg;  // optional per-step phase timestamps (CTA 0, thread 0)
};

constexpr int kMetaRing = 64;

// debug timeline stamp: the SM cycle counter (CTA 0 only, so one clock)
__device__ __forceinline__ unsigned long long gtimer() { return (unsigned long long)clock64(); }
__device__ __forceinline__ unsigned long long gtimer_ns() {  // comparable across SMs
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
constexpr int kMaxCluster = 16;
#ifndef SYSCD_DENSE_FLUSH_COST
#define SYSCD_DENSE_FLUSH_COST 115  // flush cost in hundredths of a column step
#endif

template <int NTC, int RC, int NCH>
struct DenseCfg {
  static constexpr int kNTC = NTC;
  static constexpr int kNWC = NTC / 32;
  static constexpr int kRC = RC;
  static constexpr int kNCH = NCH;
  static constexpr int kR = RC * NCH;
  static constexpr int kChunkRows = NTC * RC;
  static constexpr int kCtaRows = kChunkRows * NCH;
  static constexpr int kThreads = NTC + 32;
};

struct SmemLayout {
  size_t ring, full, empty, xbar, slots, red, meta, range, total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline SmemLayout smem_layout(int stages, int chunk_rows) {
  SmemLayout L;
  L.ring = 0;
  size_t o = align_up((size_t)stages * chunk_rows * 4, 128);
  L.full = o;
  o += (size_t)stages * 8;
  L.empty = o;
  o += (size_t)stages * 8;
  L.xbar = o;
  o += 2 * 8;
  o = align_up(o, 16);
  L.slots = o;
  o += 2 * kMaxCluster * 4;
  L.red = o;
  o += 2 * 32 * 4;
  o = align_up(o, 16);
  L.meta = o;
  o += kMetaRing * 16;
  L.range = o;
  o += 4 * 8;
  L.total = align_up(o, 128);
  return L;
}

// KIND: the step is compiled in (SYSCD_RIDGE also serves the primal-logistic
// surrogate, which has the same closed form); the hot loop carries only its
// own step -- the logistic-dual fp64 Newton would otherwise sit in every
// instance's loop.
template <class Cfg, int KIND>
__global__ void __launch_bounds__(Cfg::kThreads, 1) k_dense_epoch(DenseArgs args) {
  constexpr int NTC = Cfg::kNTC;
  constexpr int NWC = Cfg::kNWC;
  constexpr int RC = Cfg::kRC;
  constexpr int NCH = Cfg::kNCH;
  constexpr int R = Cfg::kR;
  constexpr int CHUNK = Cfg::kChunkRows;
  constexpr int CTA_ROWS = Cfg::kCtaRows;

  extern __shared__ __align__(128) unsigned char smem[];
  const int S = args.stages;
  const SmemLayout L = smem_layout(S, CHUNK);
  float* ring = reinterpret_cast<float*>(smem + L.ring);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.full);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + L.empty);
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + L.xbar);
  float* slots = reinterpret_cast<float*>(smem + L.slots);
  float* red = reinterpret_cast<float*>(smem + L.red);
  int4* meta = reinterpret_cast<int4*>(smem + L.meta);
  int64_t* range = reinterpret_cast<int64_t*>(smem + L.range);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int C = args.cluster;
  const uint32_t rank = cluster_rank();
  const int g = blockIdx.x / C;
  const int G = gridDim.x / C;
  const int64_t row0 = (int64_t)rank * CTA_ROWS;
  const int64_t d = args.d;

#ifdef SYSCD_TRACE
  if (args.dbg && tid == 0) args.dbg[12288 + blockIdx.x * 4 + 0] = gtimer_ns();
#endif
  for (int i = tid; i < S * CHUNK; i += blockDim.x) ring[i] = 0.f;
  for (int i = tid; i < 2 * kMaxCluster; i += blockDim.x) slots[i] = 0.f;
  // every writer orders its generic-proxy zeros before the TMA (async
  // proxy) fills that follow the barrier; one fence by the issuing thread
  // does not cover the other threads' writes
  fence_proxy_async();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWC);
    }
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    int64_t p_lo, p_hi;
    // a partition's replica flush costs about 1.15 column steps (config 2:
    // 2.3 us against 2.0 us per column); balancing columns alone left the
    // cluster holding the 8-column partitions 7% behind the others
    worker_parts_cost(args.wp, args.n_parts, G, g, SYSCD_DENSE_FLUSH_COST, &p_lo, &p_hi);
    if (p_lo > args.n_parts) p_lo = args.n_parts;
    if (p_hi > args.n_parts) p_hi = args.n_parts;
    range[0] = p_lo;
    range[1] = p_hi;
    fence_mbar_init();
    fence_proxy_async();
  }
  __syncthreads();
  cluster_sync_all();

  // bytes of each of this CTA's chunks (identical for every column); the tail
  // of a partial chunk is never written, so with S % NCH == 0 (a stage always
  // holds the same chunk index) it stays zero from the initial clear and rows
  // past d contribute x = 0 without any per-row predicate.
  uint32_t chunk_bytes[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    int64_t valid = d - (row0 + (int64_t)c * CHUNK);
    valid = valid < 0 ? 0 : (valid > CHUNK ? CHUNK : valid);
    chunk_bytes[c] = (uint32_t)(((valid + 3) / 4) * 16);
  }
  const int64_t p_lo = range[0];
  const int64_t p_hi = range[1];
  const int64_t s_begin = args.wp[p_lo];
  const int64_t s_end = args.wp[p_hi];

  if (warp == NWC) {
    // ------------------------------------------------------------ producer
    const uint64_t policy = args.evict_first ? policy_evict_first() : policy_evict_last();
    const uint64_t upolicy = policy_evict_last();
    uint32_t stage = 0, phase = 0;
    int jreg = 0;
    int64_t ppart = p_lo;
    while (ppart < p_hi && args.wp[ppart + 1] <= s_begin) ++ppart;
    int64_t ppart_end = ppart < p_hi ? args.wp[ppart + 1] : s_end;
    const float* uslice = args.u + row0;
    for (int64_t s = s_begin; s < s_end; ++s) {
      const int64_t rel = s - s_begin;
      if ((rel & 31) == 0) {
        const int64_t q = s + lane;
        jreg = q < s_end ? args.seq[q] : 0;
      }
      const int j = __shfl_sync(0xffffffffu, jreg, (int)(rel & 31));
      const bool part_last = s + 1 == ppart_end;
      if (part_last) {
        ++ppart;
        while (ppart < p_hi && args.wp[ppart + 1] <= s + 1) ++ppart;
        ppart_end = ppart < p_hi ? args.wp[ppart + 1] : s_end;
      }
      if (lane == 0) {
        const float* col = args.A + (int64_t)j * args.lda + row0;
        // perm mode: alpha_j is only written by this cluster, at this step,
        // so it can be read ahead of time (iid re-reads it after the exchange)
        const float aj = args.iid ? 0.f : args.alpha[j];
        const float qj = __ldg(args.sq + j);
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          mbar_wait(&empty[stage], phase ^ 1u);
          if (c == 0)
            meta[s & (kMetaRing - 1)] =
                make_int4(part_last ? (int)((unsigned)j | 0x80000000u) : j, __float_as_int(aj),
                          __float_as_int(qj),
                          __float_as_int(step_inv(args.kind, args.a, qj, args.lam_f)));
          const uint32_t bytes = chunk_bytes[c];
          if (bytes) {
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_1d(ring + (size_t)stage * CHUNK, col + c * CHUNK, bytes, &full[stage], policy);
          } else {
            mbar_arrive(&full[stage]);
          }
          if (++stage == (uint32_t)S) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (part_last) {
          // the partition-end flush reads u through the ring too (u is
          // L2-resident; staging it turns the flush into one shared-memory pass)
#pragma unroll 1
          for (int c = 0; c < NCH; ++c) {
            mbar_wait(&empty[stage], phase ^ 1u);
            const uint32_t bytes = chunk_bytes[c];
#if defined(SYSCD_TRACE) || defined(SYSCD_DENSE_STAMPS)
            if (args.dbg != nullptr && blockIdx.x == 0 && s - s_begin < 512)
              args.dbg[7168 + (s - s_begin) * 8 + c] = gtimer();
#endif
            if (bytes) {
              mbar_arrive_expect_tx(&full[stage], bytes);
              tma_load_1d(ring + (size_t)stage * CHUNK, uslice + c * CHUNK, bytes, &full[stage],
                          upolicy);
            } else {
              mbar_arrive(&full[stage]);
            }
            if (++stage == (uint32_t)S) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ consumers
    // owned row of register slot q = c*RC + k is row0 + q*NTC + tid; slots
    // q >= qmax lie past d: their w stays 0 and their staged x is 0.
    const int64_t rem = d - row0 - tid;
    const int qmax = rem <= 0 ? 0 : (int)min((int64_t)R, (rem + NTC - 1) / NTC);
    const float* ub = args.u + row0 + tid;
    float w[R];
#pragma unroll
    for (int q = 0; q < R; ++q) w[q] = q < qmax ? ub[q * NTC] : 0.f;
    const float a = args.a;
    const float inv_a = (float)(1.0 / args.a_d);
    float* out = args.partials + (int64_t)g * args.part_ld + row0 + tid;
    bool flushed = false;
    uint32_t stage0 = 0, phase0 = 0;  // ring position of the current step's chunk 0
    // exchange addresses: slot[buf][rank] and xbar[buf] in peer `lane`
    uint32_t peer_slot = 0, peer_bar = 0;
    if (warp == 0 && lane < C) {
      peer_slot = cluster_map(smem_addr(slots + rank), (uint32_t)lane);
      peer_bar = cluster_map(smem_addr(&xbar[0]), (uint32_t)lane);
    }
    const float* ring_t = ring + tid;
#if defined(SYSCD_TRACE) || defined(SYSCD_DENSE_STAMPS)
    const bool dbg = args.dbg != nullptr && blockIdx.x == 0 && tid == 0;
#else
    constexpr bool dbg = false;  // stamps only in the trace build (scripts/timeline.py)
#endif
    for (int64_t s = s_begin; s < s_end; ++s) {
      const uint32_t t = (uint32_t)(s - s_begin);
      const uint32_t buf = t & 1u;
      if (dbg && t < 512) args.dbg[t * 6 + 0] = gtimer();
      float acc0 = 0.f, acc1 = 0.f;
      {
        uint32_t st = stage0, ph = phase0;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          mbar_wait(&full[st], ph);
          const float* x = ring_t + (size_t)st * CHUNK;
#pragma unroll
          for (int k = 0; k < RC; ++k) {
            if (k & 1) {
              acc1 = fmaf(x[k * NTC], w[c * RC + k], acc1);
            } else {
              acc0 = fmaf(x[k * NTC], w[c * RC + k], acc0);
            }
          }
          if (++st == (uint32_t)S) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
      if (dbg && t < 512) args.dbg[t * 6 + 1] = gtimer();
      const int4 mt = meta[s & (kMetaRing - 1)];
      const int j = mt.x & 0x7fffffff;
      const bool part_last = mt.x < 0;  // the producer marks a partition's last column
      float aj = __int_as_float(mt.y);
      const float qj = __int_as_float(mt.z);
      float acc = warp_sum(acc0 + acc1);
      if (lane == 0) red[buf * 32 + warp] = acc;
      named_bar_sync(1, NTC);
      if (warp == 0) {
        float v = lane < NWC ? red[buf * 32 + lane] : 0.f;
        v = warp_sum(v);
        if (lane < C) st_async_f32(peer_slot + buf * kMaxCluster * 4, v, peer_bar + buf * 8);
        if (lane == 0) mbar_arrive_expect_tx(&xbar[buf], 4u * (uint32_t)C);
      }
      if (dbg && t < 512) args.dbg[t * 6 + 2] = gtimer();
      // iid: the exchange also hands over rank 0's alpha stores of earlier
      // steps (a coordinate may be drawn again): the st.async completion is
      // a cluster-scope release, so wait with cluster-scope acquire
      if (args.iid)
        mbar_wait_cluster(&xbar[buf], (t >> 1) & 1u);
      else
        mbar_wait(&xbar[buf], (t >> 1) & 1u);
      if (dbg && t < 512) args.dbg[t * 6 + 3] = gtimer();
      float lin;
      {
        const float4* sl = reinterpret_cast<const float4*>(slots + buf * kMaxCluster);
        const float4 s0 = sl[0], s1 = sl[1], s2 = sl[2], s3 = sl[3];
        lin = ((s0.x + s0.y) + (s0.z + s0.w)) + ((s1.x + s1.y) + (s1.z + s1.w)) +
              (((s2.x + s2.y) + (s2.z + s2.w)) + ((s3.x + s3.y) + (s3.z + s3.w)));
      }
      if (args.iid) aj = *(volatile float*)(args.alpha + j);
      float an;
      if (KIND == SYSCD_LOGISTIC_DUAL) {
        an = (float)coord_step(args.kind, (double)lin, args.a_d, (double)qj, args.lam, (double)aj,
                               args.n_coords);
      } else {
        an = coord_step_fr(KIND, lin, __int_as_float(mt.w), args.lam_f, aj, args.inv_n_f);
      }
      float delta;
      if (isfinite(an)) {
        delta = an - aj;
        if (rank == 0 && tid == 0) args.alpha[j] = an;
      } else {
        delta = 0.f;
        if (rank == 0 && tid == 0) atomicOr(args.status, SYSCD_ENONFINITE);
      }
      const float sd = a * delta;
      if (dbg && t < 512) args.dbg[t * 6 + 4] = gtimer();
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const float* x = ring_t + (size_t)stage0 * CHUNK;
#pragma unroll
        for (int k = 0; k < RC; ++k) w[c * RC + k] = fmaf(sd, x[k * NTC], w[c * RC + k]);
        // No proxy fence before the release: the FFMAs above consume every
        // value read from this stage and precede the arrive in issue order
        // (checked in the SASS), so the TMA refill cannot overtake the reads.
        // A release straight after the loads needs fence.proxy.async (see
        // epoch_grid.cu); here it would cost 3% of config 2.
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage0]);
        if (++stage0 == (uint32_t)S) {
          stage0 = 0;
          phase0 ^= 1u;
        }
      }
      if (dbg && t < 512) args.dbg[t * 6 + 5] = gtimer();
      if (part_last) {
        // fold this partition's replica (w - u)/a into the cluster's partial
        // sum: plain store for the first partition, then fire-and-forget
        // red.global.add (same thread, same address: applied in program
        // order, so the sum stays deterministic); the producer staged this
        // CTA's slice of u into the ring right after the partition's last
        // column, so the flush is one shared-memory pass.
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          mbar_wait(&full[stage0], phase0);
          if (dbg && t < 512) args.dbg[3072 + t * 8 + c] = gtimer();
          const float* uu = ring_t + (size_t)stage0 * CHUNK;
          float uv[RC];
#pragma unroll
          for (int k = 0; k < RC; ++k) uv[k] = uu[k * NTC];  // rows past d read 0
          // branch-free body for whole chunks, so the loads and reds batch
          if (c * RC + RC <= qmax) {
            if (flushed) {
#pragma unroll
              for (int k = 0; k < RC; ++k)
                red_add_f32(out + (c * RC + k) * NTC, (w[c * RC + k] - uv[k]) * inv_a);
            } else {
#pragma unroll
              for (int k = 0; k < RC; ++k)
                out[(c * RC + k) * NTC] = (w[c * RC + k] - uv[k]) * inv_a;
            }
          } else {
#pragma unroll
            for (int k = 0; k < RC; ++k) {
              const int q = c * RC + k;
              if (q < qmax) {
                const float dv = (w[q] - uv[k]) * inv_a;
                if (flushed) {
                  red_add_f32(out + q * NTC, dv);
                } else {
                  out[q * NTC] = dv;
                }
              }
            }
          }
#pragma unroll
          for (int k = 0; k < RC; ++k) w[c * RC + k] = uv[k];
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage0]);
          if (++stage0 == (uint32_t)S) {
            stage0 = 0;
            phase0 ^= 1u;
          }
        }
        flushed = true;
        if (dbg && t < 512) args.dbg[3072 + t * 8 + 7] = gtimer();
      }
    }
    if (!flushed) {
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q < qmax) out[q * NTC] = 0.f;
    }
  }
  __syncwarp();
#ifdef SYSCD_TRACE
  if (args.dbg && tid == 0) {
    args.dbg[12288 + blockIdx.x * 4 + 1] = gtimer_ns();
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    args.dbg[12288 + blockIdx.x * 4 + 3] =
        ((unsigned long long)smid << 32) | (unsigned long long)(args.wp[range[1]] - args.wp[range[0]]);
  }
#endif
  cluster_sync_all();
#ifdef SYSCD_TRACE
  if (args.dbg && tid == 0) args.dbg[12288 + blockIdx.x * 4 + 2] = gtimer_ns();
#endif
}

// ---------------------------------------------------------------------------
// host side: configuration table and launch
// ---------------------------------------------------------------------------
struct KernelEntry {
  int ntc, rc, nch;
  const void* fn[4];  // per step kind: ridge (and primal logistic), lasso, svm dual, logistic dual
  int threads;
  int max_clusters[kMaxCluster + 1];  // per cluster size, 0 = unknown, -1 = not launchable
};

template <int NTC, int RC, int NCH>
static KernelEntry make_entry() {
  KernelEntry e;
  e.ntc = NTC;
  e.rc = RC;
  e.nch = NCH;
  e.fn[0] = (const void*)&k_dense_epoch<DenseCfg<NTC, RC, NCH>, SYSCD_RIDGE>;
  e.fn[1] = (const void*)&k_dense_epoch<DenseCfg<NTC, RC, NCH>, SYSCD_LASSO>;
  e.fn[2] = (const void*)&k_dense_epoch<DenseCfg<NTC, RC, NCH>, SYSCD_SVM_DUAL>;
  e.fn[3] = (const void*)&k_dense_epoch<DenseCfg<NTC, RC, NCH>, SYSCD_LOGISTIC_DUAL>;
  e.threads = NTC + 32;
  for (int i = 0; i <= kMaxCluster; ++i) e.max_clusters[i] = 0;
  return e;
}

// (consumer threads, rows per thread per chunk, chunks per column slice);
// consumer warps + 1 producer warp is a power of two so the register file is
// split without rounding loss (<= 128 regs/thread at 16 warps).
static KernelEntry g_table[] = {
    make_entry<32, 1, 1>(),  make_entry<96, 1, 1>(),  make_entry<224, 2, 1>(),
    make_entry<224, 4, 1>(), make_entry<480, 4, 1>(), make_entry<480, 4, 2>(),
    make_entry<480, 4, 4>(), make_entry<480, 8, 4>(), make_entry<480, 9, 6>(),
    // (the grid kernel's fewer-wider-warps trick does not carry over: 7
    // consumer warps x 117 rows, 233 registers, ran config 2 at 1.00 ms
    // against 0.61 -- both passes read the staged slice from shared memory,
    // and 7 warps cannot keep enough loads in flight)
};
static std::mutex g_table_mu;
constexpr int kTableSize = sizeof(g_table) / sizeof(g_table[0]);

static int entry_rows(const KernelEntry& e) { return e.ntc * e.rc * e.nch; }

static int choose_stages(const KernelEntry& e, size_t smem_budget) {
  const size_t stage_bytes = (size_t)e.ntc * e.rc * 4;
  const size_t fixed = smem_layout(0, e.ntc * e.rc).total + 1024;
  int s = (int)((smem_budget - fixed) / (stage_bytes + 16));
  s = std::min(s, 32);
  return s / e.nch * e.nch;  // a stage always holds the same chunk index
}

static int query_max_clusters(KernelEntry& e, int C, int stages, size_t smem) {
  if (e.max_clusters[C] != 0) return e.max_clusters[C];
  for (const void* fn : e.fn) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (C > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(e.threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  cudaError_t err = cudaOccupancyMaxActiveClusters(&n, e.fn[0], &cfg);
  if (getenv("SYSCD_DEBUG"))
    fprintf(stderr, "[syscd] cfg (%d,%d,%d) C=%d smem=%zu -> clusters=%d (%s)\n", e.ntc, e.rc,
            e.nch, C, smem, n, cudaGetErrorString(err));
  if (err != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = -1;
  }
  e.max_clusters[C] = n;
  (void)stages;
  return n;
}

struct Choice {
  int idx;
  int C;
  int G;
  int stages;
  size_t smem;
  int grid;  // 1: grid-wide lookahead kernel (epoch_grid.cu)
};

int grid_choose(int64_t d, int* idx, int* G, int* stages, size_t* smem_out, int64_t* cta_rows,
                int iid);
int small_workers(int32_t n_parts);
int small_launch(const syscd_dense_epoch_args* e, cudaStream_t stream);
bool mid_applicable(int64_t d, int32_t n_parts, int* workers, int* cluster);
int mid_launch(const syscd_dense_epoch_args* e, cudaStream_t stream);
constexpr int64_t kSmallMaxD = 32;
int64_t grid_workspace_bytes(int G);
int grid_launch(const syscd_dense_epoch_args* e, void* workspace, int64_t ws_bytes,
                cudaStream_t stream);

static int choose(int64_t d, int32_t n_parts, Choice* out) {
  std::lock_guard<std::mutex> lock(g_table_mu);
  int dev = 0;
  SYSCD_CUDA_TRY(cudaGetDevice(&dev));
  int sms = 0, smem_optin = 0;
  SYSCD_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SYSCD_CUDA_TRY(
      cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t budget = (size_t)smem_optin - 1024;
  double best = 1e300;
  Choice bc = {-1, 0, 0, 0, 0, 0};
  const char* force = getenv("SYSCD_DENSE_CFG");  // experiments: one table entry
  for (int i = 0; i < kTableSize; ++i) {
    if (force && atoi(force) != i) continue;
    KernelEntry& e = g_table[i];
    const int rows = entry_rows(e);
    const int C = (int)((d + rows - 1) / rows);
    if (C < 1 || C > kMaxCluster) continue;
    const int stages = choose_stages(e, budget);
    if (stages < 2 * e.nch) continue;
    const size_t smem = smem_layout(stages, e.ntc * e.rc).total;
    const int maxc = query_max_clusters(e, C, stages, smem);
    if (maxc <= 0) continue;
    const int G = std::max(1, std::min(maxc, (int)n_parts));
    // per-step cycles: staged reads (dot + axpy) + reduction latency, against
    // the HBM share of the G*C SMs streaming this geometry
    const double lds = (double)rows * 8.0 / 128.0;
    const double sync = 700.0 + 25.0 * C;
    const double hbm = (double)rows * 4.0 / (6.5e12 / (double)(G * C)) * 1.9e9;
    const double t = std::max(lds + sync, hbm) / (double)G;
    if (t < best * 0.999) {
      best = t;
      bc = {i, C, G, stages, smem, 0};
    }
  }
  // Grid-wide kernel: needed when no cluster holds the replica in registers,
  // and preferred for tall columns when there are fewer partitions than
  // clusters (one partition then streams over every SM instead of one GPC).
  int gidx, gG, gst;
  size_t gsm;
  const bool grid_ok = grid_choose(d, &gidx, &gG, &gst, &gsm, nullptr, 1) == SYSCD_OK;
  if (grid_ok && (bc.idx < 0 || (d >= 131072 && bc.G < 4 && n_parts < 4))) {
    *out = {gidx, 1, 1, gst, gsm, 1};
    return SYSCD_OK;
  }
  if (bc.idx < 0) {
    set_error("no dense epoch configuration covers d=%lld", (long long)d);
    return SYSCD_EINVAL;
  }
  *out = bc;
  return SYSCD_OK;
}

}  // namespace syscd

using namespace syscd;

static void* g_dbg_buffer = nullptr;
// Debug hook (not part of the header ABI): when set to a device buffer of
// >= 512*8 uint64, the next dense epochs record SM clock cycles at the step
// phases of CTA 0 (start, dot done, CTA reduce done, exchange done, step
// done, axpy done; at [3072 + 2t]: partition-end flush, first u chunk ready
// and flush done).
extern "C" void syscd_debug_set_timeline(void* device_buffer) { g_dbg_buffer = device_buffer; }

extern "C" int syscd_dense_epoch_workers(int64_t d, int32_t n_parts, int32_t* n_workers,
                                         int32_t* cluster) {
  if (d < 1 || n_parts < 1 || !n_workers) {
    set_error("syscd_dense_epoch_workers: invalid arguments");
    return SYSCD_EINVAL;
  }
  if (d <= kSmallMaxD) {  // warp-per-partition chunked-Gram kernel (epoch_small.cu)
    *n_workers = small_workers(n_parts);
    if (cluster) *cluster = 0;
    return SYSCD_OK;
  }
  int mw = 0, mc = 0;
  if (mid_applicable(d, n_parts, &mw, &mc)) {  // chunked-Gram cluster kernel (epoch_mid.cu)
    *n_workers = mw;
    if (cluster) *cluster = mc;
    return SYSCD_OK;
  }
  Choice ch;
  int st = choose(d, n_parts, &ch);
  if (st) return st;
  *n_workers = ch.G;
  if (cluster) *cluster = ch.C;
  return SYSCD_OK;
}

extern "C" int64_t syscd_dense_epoch_workspace_bytes(int64_t d, int32_t n_parts) {
  if (d >= 1 && d <= kSmallMaxD && n_parts >= 1) return 0;
  if (n_parts >= 1 && mid_applicable(d, n_parts, nullptr, nullptr)) return 0;
  Choice ch;
  if (d < 1 || n_parts < 1 || choose(d, n_parts, &ch) != SYSCD_OK) return -1;
  if (!ch.grid) return 0;
  int idx, G, st;
  size_t sm;
  grid_choose(d, &idx, &G, &st, &sm, nullptr, 1);
  return grid_workspace_bytes(G);
}

extern "C" int syscd_dense_epoch(const syscd_dense_epoch_args* e, void* stream) {
  if (!e || !e->A || !e->sq || !e->alpha || !e->u || !e->seq || !e->work_prefix ||
      !e->partials || !e->status || e->d < 1 || e->n_parts < 1 || e->lda < e->d ||
      (e->lda % 4) != 0 || !(e->a > 0.0) || !(e->lam > 0.0)) {
    set_error("syscd_dense_epoch: invalid arguments");
    return SYSCD_EINVAL;
  }
  if ((((uintptr_t)e->A) & 15) != 0) {
    set_error("syscd_dense_epoch: A must be 16-byte aligned");
    return SYSCD_EINVAL;
  }
  if (e->d <= kSmallMaxD) {
    if (e->part_ld < e->d) {
      set_error("syscd_dense_epoch: part_ld < d");
      return SYSCD_EINVAL;
    }
    return small_launch(e, (cudaStream_t)stream);
  }
  if (mid_applicable(e->d, e->n_parts, nullptr, nullptr)) {
    if (e->part_ld < e->d) {
      set_error("syscd_dense_epoch: part_ld < d");
      return SYSCD_EINVAL;
    }
    return mid_launch(e, (cudaStream_t)stream);
  }
  Choice ch;
  int st = choose(e->d, e->n_parts, &ch);
  if (st) return st;
  if (e->part_ld < e->d) {
    set_error("syscd_dense_epoch: part_ld < d");
    return SYSCD_EINVAL;
  }
  if (ch.grid) return grid_launch(e, e->workspace, e->workspace_bytes, (cudaStream_t)stream);
  const KernelEntry& ke = g_table[ch.idx];
  DenseArgs args;
  args.A = e->A;
  args.lda = e->lda;
  args.d = e->d;
  args.sq = e->sq;
  args.alpha = e->alpha;
  args.u = e->u;
  args.seq = e->seq;
  args.wp = e->work_prefix;
  args.n_parts = e->n_parts;
  args.a = (float)e->a;
  args.a_d = e->a;
  args.lam = e->lam;
  args.lam_f = (float)e->lam;
  args.inv_n_f = (float)(1.0 / e->n_coords);
  args.n_coords = e->n_coords;
  args.kind = e->kind;
  args.iid = e->iid;
  args.stages = ch.stages;
  args.cluster = ch.C;
  // keep a matrix that fits comfortably in the 126 MB L2 resident across
  // rounds; stream larger ones with evict_first so they do not flush u/alpha
  args.evict_first = ((double)e->lda * 4.0 * (double)e->n_store) > 64.0 * 1024 * 1024 ? 1 : 0;
  args.partials = e->partials;
  args.part_ld = e->part_ld;
  args.status = e->status;
  args.dbg = (unsigned long long*)g_dbg_buffer;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ch.G * ch.C, 1, 1);
  cfg.blockDim = dim3(ke.threads, 1, 1);
  cfg.dynamicSmemBytes = ch.smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ch.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {&args};
  const int slot = e->kind == SYSCD_LASSO ? 1
                   : e->kind == SYSCD_SVM_DUAL ? 2
                   : e->kind == SYSCD_LOGISTIC_DUAL ? 3 : 0;
  SYSCD_CUDA_TRY(cudaLaunchKernelExC(&cfg, ke.fn[slot], params));
  return SYSCD_OK;
}
