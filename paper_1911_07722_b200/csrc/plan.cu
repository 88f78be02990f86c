// Device-side round planning: the seeded re-partitioning of buckets across
// workers and the within-bucket coordinate permutations, bit-exact with the
// reference's numpy streams (rng.cuh).
//
// Per round r (rid = rid0 + r) and local node k:
//   k_plan_order   : order = permutation(len(node_buckets)) with key (1,k,rid)
//                    (static mode: rid 0)      -- partitioning.py:99-109
//   k_plan_offsets : per partition (k,p) the update count of its bucket list
//                    shuffled[p::P] (partitioning.py:85-86) truncated by T3/T4
//                    (solvers.py:316-322,327-328), exclusive scan -> work_prefix,
//                    and each used slot's offset inside its partition
//   k_plan_perm    : per used slot, permutation(hi-lo) with key (2,rid,b)
//                    (partitioning.py:112-117) written as store columns
//   k_plan_iid     : per partition, iid draws with key (3,k,p,rid)
//                    (solvers.py:326-333)
// Rounds are independent, so a batch of rounds is planned in one pass (the
// permutations are data-independent and can run ahead on a side stream).
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "rng.cuh"

namespace syscd {

constexpr int kMaxLocalNodes = 64;

struct PlanParams {
  uint64_t seed;
  int64_t n_global;
  int64_t rid0;
  int32_t B;
  int32_t n_nodes;
  int32_t node0;
  int32_t P;
  int32_t T3, T4;
  int32_t sampling, repartition;
  int32_t nb_total;  // sum of node bucket counts
  int32_t n_parts;   // n_nodes * P
  int32_t node_ptr[kMaxLocalNodes + 1];
  const int32_t* node_buckets;
  const int64_t* store_col;
  int32_t* order;     // [R][nb_total]
  int32_t* slot_off;  // [R][nb_total]
  int64_t* lens;      // [R][n_parts]
  int32_t* scratch;   // [R][nb_total*B] (only when B > kLocalPerm)
  int32_t* seq;
  int64_t seq_stride;
  int64_t* work_prefix;  // [R][n_parts+1]
  int64_t* round_updates;  // optional [rid]: total updates of the round
};

constexpr int kLocalPerm = 64;

__device__ __forceinline__ int node_of_slot(const PlanParams& pp, int gi) {
  int k = 0;
  while (k + 1 < pp.n_nodes && pp.node_ptr[k + 1] <= gi) ++k;
  return k;
}

__device__ __forceinline__ int64_t bucket_len(const PlanParams& pp, int64_t gb) {
  int64_t lo = gb * pp.B;
  int64_t hi = lo + pp.B;
  if (hi > pp.n_global) hi = pp.n_global;
  return hi - lo;
}

// One block per (round, node); thread 0 runs the Fisher-Yates chain in shared
// memory (uint16 positions) when the node's list fits, else in global memory.
__global__ void k_plan_order(PlanParams pp) {
  extern __shared__ uint16_t s_pos[];
  const int r = blockIdx.x;
  const int k = blockIdx.y;
  const int off = pp.node_ptr[k];
  const int nb = pp.node_ptr[k + 1] - off;
  int32_t* out = pp.order + (int64_t)r * pp.nb_total + off;
  const int64_t rid = pp.repartition == 1 ? 0 : pp.rid0 + r;
  const bool in_smem = nb <= 65536;
  if (in_smem) {
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s_pos[i] = (uint16_t)i;
  } else {
    for (int i = threadIdx.x; i < nb; i += blockDim.x) out[i] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Pcg64 g;
    pcg_seed3(&g, pp.seed, 1u, (uint64_t)(pp.node0 + k), (uint64_t)rid, 3);
    if (in_smem) {
      pcg_shuffle(&g, s_pos, (int64_t)nb);
    } else {
      pcg_shuffle(&g, out, (int64_t)nb);
    }
  }
  __syncthreads();
  if (in_smem) {
    for (int i = threadIdx.x; i < nb; i += blockDim.x) out[i] = s_pos[i];
  }
}

// One block per round.
__global__ void k_plan_offsets(PlanParams pp) {
  typedef cub::BlockScan<int64_t, 256> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t carry;
  const int r = blockIdx.x;
  const int32_t* order = pp.order + (int64_t)r * pp.nb_total;
  int32_t* slot_off = pp.slot_off + (int64_t)r * pp.nb_total;
  int64_t* lens = pp.lens + (int64_t)r * pp.n_parts;
  for (int part = threadIdx.x; part < pp.n_parts; part += blockDim.x) {
    const int k = part / pp.P;
    const int p = part % pp.P;
    const int off = pp.node_ptr[k];
    const int nb = pp.node_ptr[k + 1] - off;
    const int cnt = (nb - p + pp.P - 1) / pp.P;
    int64_t len = 0;
    if (pp.sampling == 0) {
      const int t3 = pp.T3 < 0 ? cnt : min(pp.T3, cnt);
      for (int t = 0; t < cnt; ++t) {
        const int slot = p + t * pp.P;
        if (t < t3) {
          const int64_t gb = pp.node_buckets[off + order[off + slot]];
          const int64_t bl = bucket_len(pp, gb);
          const int64_t t4 = pp.T4 < 0 ? bl : min((int64_t)pp.T4, bl);
          slot_off[off + slot] = (int32_t)len;
          len += t4;
        } else {
          slot_off[off + slot] = -1;
        }
      }
    } else {
      const int64_t t3 = pp.T3 < 0 ? cnt : pp.T3;
      const int64_t t4 = pp.T4 < 0 ? pp.B : pp.T4;
      len = t3 * t4;
    }
    lens[part] = len;
  }
  __syncthreads();
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  int64_t* wp = pp.work_prefix + (int64_t)r * (pp.n_parts + 1);
  for (int base = 0; base < pp.n_parts; base += 256) {
    const int part = base + threadIdx.x;
    int64_t v = part < pp.n_parts ? lens[part] : 0;
    int64_t excl, total;
    Scan(tmp).ExclusiveSum(v, excl, total);
    if (part < pp.n_parts) wp[part] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    wp[pp.n_parts] = carry;
    if (pp.round_updates) pp.round_updates[pp.rid0 + r] = carry;
  }
}

__global__ void k_plan_perm(PlanParams pp, int n_rounds) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)n_rounds * pp.nb_total) return;
  const int r = (int)(gid / pp.nb_total);
  const int gi = (int)(gid % pp.nb_total);
  const int32_t rel = pp.slot_off[(int64_t)r * pp.nb_total + gi];
  if (rel < 0) return;
  const int k = node_of_slot(pp, gi);
  const int off = pp.node_ptr[k];
  const int slot = gi - off;
  const int part = k * pp.P + slot % pp.P;
  const int ell = off + pp.order[(int64_t)r * pp.nb_total + gi];
  const int64_t gb = pp.node_buckets[ell];
  const int64_t base = pp.store_col[ell];
  const int64_t bl = bucket_len(pp, gb);
  const int64_t t4 = pp.T4 < 0 ? bl : min((int64_t)pp.T4, bl);
  const int64_t rid = pp.rid0 + r;
  int32_t* out = pp.seq + (int64_t)r * pp.seq_stride +
                 pp.work_prefix[(int64_t)r * (pp.n_parts + 1) + part] + rel;
  Pcg64 g;
  pcg_seed3(&g, pp.seed, 2u, (uint64_t)rid, (uint64_t)gb, 3);
  if (bl <= kLocalPerm) {
    int32_t perm[kLocalPerm];
    for (int i = 0; i < bl; ++i) perm[i] = i;
    pcg_shuffle(&g, perm, bl);
    for (int i = 0; i < t4; ++i) out[i] = (int32_t)(base + perm[i]);
  } else {
    int32_t* perm = pp.scratch + ((int64_t)r * pp.nb_total + gi) * pp.B;
    for (int i = 0; i < bl; ++i) perm[i] = i;
    pcg_shuffle(&g, perm, bl);
    for (int i = 0; i < t4; ++i) out[i] = (int32_t)(base + perm[i]);
  }
}

__global__ void k_plan_iid(PlanParams pp, int n_rounds) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)n_rounds * pp.n_parts) return;
  const int r = (int)(gid / pp.n_parts);
  const int part = (int)(gid % pp.n_parts);
  const int k = part / pp.P;
  const int p = part % pp.P;
  const int off = pp.node_ptr[k];
  const int nb = pp.node_ptr[k + 1] - off;
  const int cnt = (nb - p + pp.P - 1) / pp.P;
  const int64_t t3 = pp.T3 < 0 ? cnt : pp.T3;
  const int64_t t4 = pp.T4 < 0 ? pp.B : pp.T4;
  const int64_t rid = pp.rid0 + r;
  const int32_t* order = pp.order + (int64_t)r * pp.nb_total + off;
  int32_t* out = pp.seq + (int64_t)r * pp.seq_stride +
                 pp.work_prefix[(int64_t)r * (pp.n_parts + 1) + part];
  Pcg64 g;
  uint64_t key[4] = {3u, (uint64_t)(pp.node0 + k), (uint64_t)p, (uint64_t)rid};
  pcg_seed_keyed(&g, pp.seed, key, 4);
  int64_t w = 0;
  for (int64_t t = 0; t < t3; ++t) {
    const int64_t bpos = pcg_integers(&g, 0, cnt);
    const int ell = off + order[p + bpos * pp.P];
    const int64_t gb = pp.node_buckets[ell];
    const int64_t lo = gb * pp.B;
    const int64_t bl = bucket_len(pp, gb);
    const int64_t base = pp.store_col[ell];
    for (int64_t s = 0; s < t4; ++s) {
      const int64_t j = pcg_integers(&g, lo, lo + bl);
      out[w++] = (int32_t)(base + (j - lo));
    }
  }
}

static int plan_check(const syscd_plan_desc* d) {
  if (!d || d->n_nodes_local < 1 || d->n_nodes_local > kMaxLocalNodes || d->P < 1 ||
      d->bucket_size < 1 || d->n_global < 1 || !d->node_bucket_ptr) {
    set_error("syscd_plan: invalid descriptor");
    return SYSCD_EINVAL;
  }
  for (int k = 0; k < d->n_nodes_local; ++k) {
    int nb = d->node_bucket_ptr[k + 1] - d->node_bucket_ptr[k];
    if (nb < 1) {
      set_error("empty bucket list");
      return SYSCD_EINVAL;
    }
    if (d->P > nb) {
      set_error("more threads than buckets on this node");
      return SYSCD_EINVAL;
    }
  }
  return SYSCD_OK;
}

static int64_t align256(int64_t x) { return (x + 255) / 256 * 256; }

}  // namespace syscd

using namespace syscd;

extern "C" int64_t syscd_plan_workspace_bytes(const syscd_plan_desc* d, int32_t n_rounds) {
  if (plan_check(d) != SYSCD_OK || n_rounds < 1) return -1;
  const int64_t nbt = d->node_bucket_ptr[d->n_nodes_local];
  const int64_t parts = (int64_t)d->n_nodes_local * d->P;
  int64_t bytes = 0;
  bytes += align256(n_rounds * nbt * 4);      // order
  bytes += align256(n_rounds * nbt * 4);      // slot_off
  bytes += align256(n_rounds * parts * 8);    // lens
  if (d->bucket_size > kLocalPerm) bytes += align256(n_rounds * nbt * d->bucket_size * 4);
  return bytes;
}

extern "C" int64_t syscd_plan_max_updates(const syscd_plan_desc* d) {
  if (plan_check(d) != SYSCD_OK) return -1;
  int64_t total = 0;
  for (int k = 0; k < d->n_nodes_local; ++k) {
    const int64_t nb = d->node_bucket_ptr[k + 1] - d->node_bucket_ptr[k];
    if (d->sampling == 0) {
      total += nb * (int64_t)d->bucket_size;  // upper bound (last bucket may be partial)
    } else {
      for (int p = 0; p < d->P; ++p) {
        const int64_t cnt = (nb - p + d->P - 1) / d->P;
        const int64_t t3 = d->T3 < 0 ? cnt : d->T3;
        const int64_t t4 = d->T4 < 0 ? d->bucket_size : d->T4;
        total += t3 * t4;
      }
    }
  }
  return total;
}

extern "C" int syscd_plan(const syscd_plan_desc* d, int64_t rid0, int32_t n_rounds, int32_t* seq,
                          int64_t seq_stride, int64_t* work_prefix, void* workspace,
                          int64_t workspace_bytes, void* stream) {
  int st = plan_check(d);
  if (st != SYSCD_OK) return st;
  if (n_rounds < 1 || !seq || !work_prefix || !workspace) {
    set_error("syscd_plan: missing buffers");
    return SYSCD_EINVAL;
  }
  if (workspace_bytes < syscd_plan_workspace_bytes(d, n_rounds)) {
    set_error("syscd_plan: workspace too small");
    return SYSCD_EINVAL;
  }
  if (seq_stride < syscd_plan_max_updates(d)) {
    set_error("syscd_plan: seq_stride too small");
    return SYSCD_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  PlanParams pp = {};
  pp.seed = d->seed;
  pp.n_global = d->n_global;
  pp.rid0 = rid0;
  pp.B = d->bucket_size;
  pp.n_nodes = d->n_nodes_local;
  pp.node0 = d->node0;
  pp.P = d->P;
  pp.T3 = d->T3;
  pp.T4 = d->T4;
  pp.sampling = d->sampling;
  pp.repartition = d->repartition;
  for (int k = 0; k <= d->n_nodes_local; ++k) pp.node_ptr[k] = d->node_bucket_ptr[k];
  pp.nb_total = pp.node_ptr[d->n_nodes_local];
  pp.n_parts = d->n_nodes_local * d->P;
  pp.node_buckets = d->node_buckets;
  pp.store_col = d->bucket_store_col;
  char* ws = (char*)workspace;
  pp.order = (int32_t*)ws;
  ws += align256((int64_t)n_rounds * pp.nb_total * 4);
  pp.slot_off = (int32_t*)ws;
  ws += align256((int64_t)n_rounds * pp.nb_total * 4);
  pp.lens = (int64_t*)ws;
  ws += align256((int64_t)n_rounds * pp.n_parts * 8);
  pp.scratch = d->bucket_size > kLocalPerm ? (int32_t*)ws : nullptr;
  pp.seq = seq;
  pp.seq_stride = seq_stride;
  pp.work_prefix = work_prefix;
  pp.round_updates = d->round_updates;

  int nb_max = 0;
  for (int k = 0; k < d->n_nodes_local; ++k)
    nb_max = max(nb_max, pp.node_ptr[k + 1] - pp.node_ptr[k]);
  size_t smem = nb_max <= 65536 ? (size_t)nb_max * sizeof(uint16_t) : 0;
  if (smem > 48 * 1024)
    SYSCD_CUDA_TRY(cudaFuncSetAttribute(k_plan_order, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  k_plan_order<<<dim3(n_rounds, d->n_nodes_local), 128, smem, s>>>(pp);
  SYSCD_CUDA_TRY(cudaGetLastError());
  k_plan_offsets<<<n_rounds, 256, 0, s>>>(pp);
  SYSCD_CUDA_TRY(cudaGetLastError());
  if (d->sampling == 0) {
    const int64_t work = (int64_t)n_rounds * pp.nb_total;
    k_plan_perm<<<(unsigned)((work + 127) / 128), 128, 0, s>>>(pp, n_rounds);
  } else {
    const int64_t work = (int64_t)n_rounds * pp.n_parts;
    k_plan_iid<<<(unsigned)((work + 127) / 128), 128, 0, s>>>(pp, n_rounds);
  }
  SYSCD_CUDA_TRY(cudaGetLastError());
  return SYSCD_OK;
}
