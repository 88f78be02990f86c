/*
 * syscd_b200 — C ABI of the B200-native SySCD training epoch.
 *
 * The reference (arxiv/paper_1911_07722, pure Python package `syscd`) has no
 * native FFI; its drop-in boundary for this path is the Python call
 *     syscd.run_syscd(problem, cfg, f_star)      pkg/src/syscd/solvers.py:337
 *     syscd.run_solver(problem, cfg, f_star)     pkg/src/syscd/solvers.py:456
 * The entry points below are what that call decomposes into on a GPU; the
 * Python package paper_1911_07722_b200 binds them with ctypes (see
 * INTEGRATION.md for the stub a syscd maintainer would add).  Each function
 * names the reference code it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device pointers are borrowed for the
 *    duration of the call; no allocation happens on the hot calls (workspace
 *    is passed in).  `stream` is a cudaStream_t passed as void*.
 *  - Every function returns a status: SYSCD_OK, SYSCD_EINVAL (configuration
 *    error -> ValueError, solvers.py:63-79,346-353, partitioning.py:78-106),
 *    SYSCD_ENONFINITE (-> NonFiniteUpdateError, objective.py:13-14,
 *    solvers.py:307-308), SYSCD_ECUDA (CUDA/NCCL error -> RuntimeError).
 *    syscd_last_error() returns a thread-local message for the last failure.
 *  - No global mutable state besides that message, per-device caches of the
 *    kernel-configuration queries (guarded) and the debug hooks (not part of
 *    this ABI): concurrent calls on distinct problems are safe.
 */
#ifndef SYSCD_B200_H_
#define SYSCD_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SYSCD_ABI_VERSION 1

/* status codes */
#define SYSCD_OK 0
#define SYSCD_EINVAL 1
#define SYSCD_ENONFINITE 2
#define SYSCD_ECUDA 3

/* objective kinds: f(A alpha) + sum_j g_j(alpha_j) */
#define SYSCD_RIDGE 0          /* squared loss + l2 (objective.py:26,62-63)          */
#define SYSCD_LOGISTIC 1       /* primal logistic + l2 (objective.py:30,36-42)       */
#define SYSCD_LASSO 2          /* squared loss + l1             */
#define SYSCD_SVM_DUAL 3       /* hinge SVM dual, columns y_i x_i (Appendix A)      */
#define SYSCD_LOGISTIC_DUAL 4  /* logistic dual, columns y_i x_i (Appendix A)       */

int syscd_abi_version(void);
const char* syscd_last_error(void);

/* ------------------------------------------------------------------------
 * RNG contract (host).  Bit-exact restatement of
 *   np.random.default_rng(np.random.SeedSequence(seed, spawn_key=key))
 * (partitioning.py:30-38) consumed by Generator.permutation
 * (partitioning.py:95,107,117) and Generator.integers (solvers.py:159-166).
 * Replaces: RngStream.generator().permutation / .integers.
 * ------------------------------------------------------------------------ */
int syscd_rng_permutation(uint64_t seed, const uint64_t* key, int32_t key_len, int64_t n,
                          int64_t* out);
int syscd_rng_integers(uint64_t seed, const uint64_t* key, int32_t key_len, int64_t lo,
                       int64_t hi, int64_t count, int64_t* out);

/* ------------------------------------------------------------------------
 * Device planning of one or more rounds (the seeded device-side
 * re-partitioning).  Replaces per round: _worker_bucket_order +
 * dynamic_repartition (solvers.py:174-178, partitioning.py:99-109) and the
 * per-bucket permute_within_bucket / iid draws of _surrogate_thread_round
 * (solvers.py:315-333, partitioning.py:112-117).
 *
 * Output per round r (0 <= r < n_rounds, rid = rid0 + r):
 *   seq[r*seq_stride + i]           store column of the i-th update, the
 *                                   partitions' sequences laid out back to back
 *                                   in (local node, thread) order;
 *   work_prefix[r*(n_parts+1) + p]  start of partition p in seq (exclusive
 *                                   prefix of the per-partition update counts),
 *                                   n_parts = n_nodes_local * P.
 * ------------------------------------------------------------------------ */
typedef struct {
  uint64_t seed;
  int64_t n_global;        /* coordinates of the whole problem                    */
  int32_t bucket_size;     /* B (solvers.py:81-84)                                */
  int32_t n_nodes_local;   /* node groups planned here                            */
  int32_t node0;           /* global id k of the first local node                 */
  int32_t P;               /* threads per node                                    */
  int32_t T3;              /* buckets per thread per round, -1 = all               */
  int32_t T4;              /* updates per bucket, -1 = bucket length / B (iid)     */
  int32_t sampling;        /* 0 = perm, 1 = iid                                   */
  int32_t repartition;     /* 0 = dynamic, 1 = static                             */
  const int32_t* node_bucket_ptr;  /* [n_nodes_local+1] host array                */
  const int32_t* node_buckets;     /* device: global bucket ids per node, in
                                      static_node_partition order                 */
  const int64_t* bucket_store_col; /* device: store column of each listed
                                      bucket's first coordinate                   */
  int64_t* round_updates;          /* optional device array: round_updates[rid] =
                                      total updates of round rid (NULL: skipped)  */
} syscd_plan_desc;

/* bytes of workspace syscd_plan needs for n_rounds rounds */
int64_t syscd_plan_workspace_bytes(const syscd_plan_desc* desc, int32_t n_rounds);
/* upper bound of the per-round update count (size seq_stride >= this) */
int64_t syscd_plan_max_updates(const syscd_plan_desc* desc);
int syscd_plan(const syscd_plan_desc* desc, int64_t rid0, int32_t n_rounds, int32_t* seq,
               int64_t seq_stride, int64_t* work_prefix, void* workspace, int64_t workspace_bytes,
               void* stream);

/* ------------------------------------------------------------------------
 * One node-local round on the GPU: every partition of the plan runs its
 * chain  lin = x_j.(u + a dv) ; alpha_j <- step ; dv += delta x_j  on a
 * private replica, and the replicas are summed into `partials`
 * (_surrogate_thread_round solvers.py:289-334 + the intra-node part of
 * reduce_replicas solvers.py:393).  Dense column-major fp32 store.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t kind;            /* SYSCD_* objective                                     */
  int64_t d;               /* shared-vector length (rows)                           */
  int64_t lda;             /* leading dimension (floats), multiple of 4, >= d       */
  const float* A;          /* device, store columns                                 */
  const float* sq;         /* device, column squared norms per store column         */
  float* alpha;            /* device, model per store column (read/write)           */
  const float* u;          /* device, lin_vec = grad f(v) (+ drift), length d, 16-B
                              aligned and readable up to round_up(d, 4) (bulk copies
                              move 16-byte multiples; the padding is ignored)       */
  const int32_t* seq;      /* device, one round of syscd_plan output                */
  const int64_t* work_prefix; /* device, [n_parts+1]                                */
  int32_t n_parts;
  double a;                /* surrogate curvature gamma*K*P (solvers.py:359)        */
  double lam;
  double n_coords;         /* global coordinate count (dual objectives' 1/n)        */
  int32_t iid;             /* 1 if coordinates may repeat within a round            */
  int64_t n_store;         /* columns in the store (L2 residency hint)              */
  float* partials;         /* device, [n_workers][part_ld] fp32, written here       */
  int64_t part_ld;
  int32_t* status;         /* device int, OR-ed with 2 on a non-finite step         */
  void* workspace;         /* device scratch, >= syscd_dense_epoch_workspace_bytes   */
  int64_t workspace_bytes;
} syscd_dense_epoch_args;

/* workers the dense epoch uses for this geometry (partials must hold that many rows) */
int syscd_dense_epoch_workers(int64_t d, int32_t n_parts, int32_t* n_workers, int32_t* cluster);
/* device scratch the epoch needs for this geometry (0 for the cluster kernel;
 * the grid-wide kernel used for very tall columns needs its reduction slots) */
int64_t syscd_dense_epoch_workspace_bytes(int64_t d, int32_t n_parts);
int syscd_dense_epoch(const syscd_dense_epoch_args* e, void* stream);



/* Sparse CSC store (int64 col_ptr, int32 row_idx, fp32 values); sparse
 * col_dot / col_axpy of dataset.py:77-78,90-91.  A worker is one 64-thread
 * block (a chain warp and a staging warp).  The
 * private replicas live in dv_work (n_workers x d 64-bit words, zero-filled
 * once at allocation): each word is (tag << 32 | fp32 bits) and reads as 0
 * unless its tag is the running partition's, so replicas never need
 * re-zeroing.  Partition p of a call uses tag replica_tag + p: the caller
 * advances replica_tag by n_parts per call (skipping 0; a wrap of the 32-bit
 * tag space needs a re-zero).  delta_v (d) receives the sum of the replicas.
 * When n_workers == n_parts (syscd_sparse_epoch_workers returns n_parts
 * whenever that many workers are resident) worker p runs partition p and the
 * sum is a fixed ascending-partition reduction of the replica words after
 * the chains (bitwise reproducible, reduce_replicas solvers.py:112-125);
 * otherwise it is accumulated with fp32 atomics. */
typedef struct {
  int32_t kind;
  int64_t d;
  const int64_t* col_ptr;  /* device [n_store+1]                                    */
  const int32_t* row_idx;  /* device [nnz]                                          */
  const float* vals;       /* device [nnz]                                          */
  const float* sq;
  float* alpha;
  const float* u;
  const int32_t* seq;
  const int64_t* work_prefix;
  int32_t n_parts;
  double a, lam, n_coords;
  int32_t iid;
  uint64_t* dv_work;
  int32_t n_workers;
  float* delta_v;
  int32_t* status;
  uint32_t replica_tag;
} syscd_sparse_epoch_args;

int syscd_sparse_epoch_workers(int64_t d, int32_t n_parts, int32_t* n_workers);
int syscd_sparse_epoch(const syscd_sparse_epoch_args* e, void* stream);

/* K = P = 1 primal logistic: exact coordinate updates on the live shared
 * vector with the reference's safeguarded Newton (solvers.py:403-410,
 * objective.py:113-184); v (fp64) is updated in place.  Dense (A != NULL) or
 * CSC store.  One round = the single partition of a K=P=1 plan. */
typedef struct {
  int64_t d;
  int64_t lda;
  const float* A;
  const int64_t* col_ptr;
  const int32_t* row_idx;
  const float* vals;
  const float* sq;
  float* alpha;
  double* v;
  const double* y;
  double lam;
  const int32_t* seq;
  const int64_t* work_prefix;
  int32_t* status;
} syscd_exact_args;

int syscd_exact_logistic_round(const syscd_exact_args* e, void* stream);

/* ------------------------------------------------------------------------
 * Wild (asynchronous) epoch: run_wild_parallel_scd's worker loop
 * (solvers.py:214-286).  Worker w < P walks chunk w of np.array_split(perm,
 * P) with exact updates on the live shared vector v = v0 + dv: lin =
 * x_j . (u + gamma dv) with u = grad f(v0) (exact for the quadratic f of
 * ridge / lasso / svm-dual / logistic-dual; primal logistic goes through
 * syscd_exact_logistic_round).  dv (fp32, zero at the epoch start) is read
 * through L2 and updated with unsynchronised atomics, so results depend on
 * the hardware interleaving exactly as the reference's threads do.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t kind;
  int64_t d;
  int64_t lda;            /* dense store (A != NULL) */
  const float* A;
  const int64_t* col_ptr; /* CSC store (A == NULL) */
  const int32_t* row_idx;
  const float* vals;
  const float* sq;
  float* alpha;
  const float* u;
  float* dv;
  const int32_t* perm;    /* n store-column ids, this epoch's permutation */
  int64_t n;
  int32_t P;
  double gamma;
  double lam;
  double n_coords;
  int32_t* status;
} syscd_wild_epoch_args;

int syscd_wild_epoch(const syscd_wild_epoch_args* e, void* stream);

/* ------------------------------------------------------------------------
 * Reduction + epilogue (reduce_replicas solvers.py:112-125 at node/global
 * level, solvers.py:393,423; then grad_f objective.py:105-110 for the next
 * round, solvers.py:412).
 *   dv[i]  = sum_{w < n_workers} partials[w*part_ld + i]   (ascending w)
 *   if v:  v[i] += dv[i]  (fp64)  and  u[i] = grad f(v)[i]
 * v == NULL: only dv is produced (the multi-GPU path all-reduces dv first).
 * ------------------------------------------------------------------------ */
int syscd_reduce_partials(const float* partials, int64_t part_ld, int32_t n_workers, int64_t d,
                          float* dv, void* stream);
int syscd_apply_dv(int32_t kind, int64_t d, const float* dv, double* v, const double* y,
                   double lam, double n_coords, float* u, void* stream);
/* u = grad f(v) + drift * (v_node - v)   (solvers.py:379-382 for T2 > 1) */
int syscd_grad(int32_t kind, int64_t d, const double* v, const double* y, double lam,
               double n_coords, const double* v_node, double drift, float* u, void* stream);
/* T2 > 1 node rounds (solvers.py:384-393,423): acc = (first ? 0 : acc) +
 * (v_node - v) over the local nodes in ascending order, then v += acc. */
int syscd_node_delta(int64_t d, const double* v_node, const double* v, double* acc,
                     int32_t first, void* stream);
int syscd_vec_add(int64_t d, double* v, const double* acc, void* stream);
/* fp64 certificate point for the duality gap: primal kinds w = grad f(v),
 * dual kinds w = v / (lam n). */
int syscd_dual_point(int32_t kind, int64_t d, const double* v, const double* y, double lam,
                     double n_coords, double* w, void* stream);

/* ------------------------------------------------------------------------
 * Metrics (fresh shared vector, fp64 accumulation): full_objective
 * (objective.py:95-102) = matvec (dataset.py:100-110) + loss/penalty values;
 * rmatvec (dataset.py:112-116) for the duality gap; column norms
 * (compute_stats dataset.py:307).
 * ------------------------------------------------------------------------ */
int syscd_dense_matvec(int64_t d, int64_t n, int64_t lda, const float* A, const float* x,
                       double* out, double* work, int64_t work_bytes, void* stream);
int syscd_dense_rmatvec(int64_t d, int64_t n, int64_t lda, const float* A, const double* w,
                        double* out, void* stream);
int syscd_dense_col_sq_norms(int64_t d, int64_t n, int64_t lda, const float* A, float* out,
                             void* stream);
int syscd_sparse_matvec(int64_t d, int64_t n, const int64_t* col_ptr, const int32_t* row_idx,
                        const float* vals, const float* x, double* out, void* stream);
int syscd_sparse_rmatvec(int64_t n, const int64_t* col_ptr, const int32_t* row_idx,
                         const float* vals, const double* w, double* out, void* stream);
int syscd_sparse_col_sq_norms(int64_t n, const int64_t* col_ptr, const float* vals, float* out,
                              void* stream);

/* Objective / gap terms (fp64).  out[0..7] (see paper_1911_07722_b200/metrics.py):
 *   mode 0: out[0] = f(v), out[1] = sum_j g(alpha_j)
 *   mode 1: dual-certificate terms for the gap given atw = A^T w.      */
int syscd_objective_terms(int32_t kind, int64_t d, int64_t n, const double* v, const double* y,
                          const float* alpha, double lam, double n_coords, double* out,
                          double* work, void* stream);
int syscd_gap_terms(int32_t kind, int64_t d, int64_t n, const double* v, const double* y,
                    const double* atw, double lam, double n_coords, double scale, double* out,
                    double* work, void* stream);

/* ---------------------------------------------------------------------------
 * LIBSVM text ingest (host code; replaces the line loop of load_libsvm,
 * pkg/src/syscd/dataset.py:169-233).  Two calls over the same byte buffer:
 * scan validates every line and counts examples / nonzeros, fill writes the
 * example-major arrays (example e owns entries ex_ptr[e] .. ex_ptr[e+1],
 * 0-based feature indices ascending).  Lines follow Python's universal
 * newlines (\n, \r, \r\n); blank lines are skipped but counted; labels and
 * values follow Python float() and indices Python int() (base 10,
 * underscores between digits).  The first bad line (lowest line number) is
 * reported through info->err, exactly as the reference's ValueErrors:
 *   1 bad label, 2 bad entry, 3 index not 1-based, 4 indices not ascending,
 *   5 index beyond int32 (this store's limit).                            */
typedef struct {
  int64_t n_examples;  /* non-blank lines */
  int64_t nnz;
  int64_t max_feature; /* largest 1-based index (0 if none) */
  int32_t err;         /* 0 = ok, else the code above */
  int32_t pad_;
  int64_t err_line;    /* 1-based line of the first error */
  int64_t err_tok_off; /* offending token: byte offset and length in buf */
  int64_t err_tok_len;
  int64_t err_index;   /* the parsed index for codes 3 and 5 */
} syscd_libsvm_info;

int syscd_libsvm_scan(const char* buf, int64_t len, int32_t n_threads, syscd_libsvm_info* info);
int syscd_libsvm_fill(const char* buf, int64_t len, int32_t n_threads, double* labels,
                      int64_t* ex_ptr, int32_t* feat_idx, double* vals);
/* CSR -> CSC transpose on the host (stable: rows stay ascending per column). */
int syscd_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t* ptr, const int32_t* idx,
                        const double* vals, int64_t* t_ptr, int32_t* t_idx, double* t_vals);

/* ------------------------------------------------------------------------
 * Synthetic workload generation (no reference counterpart: the reference
 * draws its synthetic data with numpy on the host, dataset.py:262-273).
 * Counter-based (Philox4x32-10): value = f(seed, tag, column id, row), so
 * every rank generates exactly its own shard's columns in HBM (SURVEY 8(d)
 * column-block keys) and a sharded job sees the one-GPU matrix.
 * ------------------------------------------------------------------------ */
/* out[s*lda + i] = N(0,1) of column cols[s] (cols NULL: s), row i < d; rows
 * d..lda-1 zero.  lda % 4 == 0. */
int syscd_gen_normal_cols(uint64_t seed, uint32_t tag, const int64_t* cols, int64_t n_cols,
                          int64_t d, int64_t lda, float* out, void* stream);
/* out[t] = N(0,1) (uniform = 0) or U(0,1) (uniform = 1) of id ids[t] (NULL: t) */
int syscd_gen_ids(uint64_t seed, uint32_t tag, const int64_t* ids, int64_t n, int32_t uniform,
                  double* out, void* stream);
/* rows[s*nnz ...] = nnz distinct rows of column cols[s] drawn by inverse CDF
 * from cdf[0..d) (first nnz distinct draws), sorted ascending; *failed is set
 * if a column could not collect nnz distinct rows. */
int syscd_gen_zipf_onehot(uint64_t seed, uint32_t tag, const int64_t* cols, int64_t n_cols,
                          int64_t d, int32_t nnz, const double* cdf, int32_t* rows,
                          int32_t* failed, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SYSCD_B200_H_ */
