/*
 * ht_b200.h -- C ABI of the B200-native hierarchical-Tucker (HT) engine.
 *
 * The reference (arXiv 1708.03340, /root/reference/pkg/src/htucker) is a
 * pure-Python package with no FFI; this header is the binding a
 * ctypes/cffi/pybind shim would use to put the reference's HT tensor API on
 * the GPU.  Every entry point names the reference function it replaces.
 *
 * Conventions
 *  - float64 everywhere; all array pointers are DEVICE pointers unless noted.
 *  - A tensor is described by its dimension d (the tree is the reference's
 *    balanced dimension tree, tree.py:55-101: BFS node ids, root 0, 2d-1
 *    nodes), leaf sizes, per-node ranks and one device pointer per node.
 *    Node arrays are C-order exactly as in the reference HTensor
 *    (format.py:50-132): root (k_s1 x k_s2), inner (k_t x k_s1 x k_s2),
 *    leaf (n x k).
 *  - Functions are asynchronous on `stream` unless documented otherwise; no
 *    allocation happens inside -- callers pass a workspace sized by the
 *    matching *_workspace_size query.  Inputs are never modified.
 *  - Return value: HT_OK or an HT_ERR_* code; ht_last_error() gives the text
 *    (thread-local).  Python maps codes to the reference exceptions
 *    (ValueError for shape / orthogonality / symmetry errors).
 */
#ifndef HT_B200_H
#define HT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* ht_stream_t; /* cudaStream_t */

enum {
  HT_OK = 0,
  HT_ERR_SHAPE = 1,           /* arith.py:398-402, format.py:101-119 */
  HT_ERR_NOT_ORTHOGONAL = 2,  /* arith.py:306-307 */
  HT_ERR_NONCONVERGED = 3,
  HT_ERR_CUDA = 4,
  HT_ERR_NOT_SYMMETRIC = 5,   /* kernels.py:47-50 */
  HT_ERR_ARGUMENT = 6,        /* arith.py:47-51 */
  HT_ERR_UNSUPPORTED = 7
};

struct ht_kron_src;
struct ht_sum_src;
typedef struct ht_tensor {
  int32_t d;              /* tensor dimension, >= 2 */
  const int64_t* n;       /* [d] host: leaf sizes by mode (mode mu -> n[mu-1]) */
  const int64_t* rank;    /* [2d-1] host: rank per node id, rank[0] == 1 */
  double* const* node;    /* [2d-1] host array of device pointers, BFS node id order */
  int32_t orthogonal;     /* HTensor.orthogonal (format.py:76) */
  /* NULL for an ordinary tensor.  Otherwise the tensor is y = apply_operator(op, x)
   * (arith.py:378-395) whose transfer tensors and root matrix F_t = H_t (x) B_t
   * (arith.py:204-213) are NOT materialised: node[t] is NULL for every inner node and
   * the root (leaf frames are ordinary device arrays), and rank[t] = op.rank[t] *
   * x.rank[t].  Accepted by the truncation entry points only (ht_truncate*), whose
   * orthogonalisation sweep consumes H_t and B_t in place. */
  const struct ht_kron_src* kron;
  /* NULL for an ordinary tensor.  Otherwise the tensor is the block-form sum
   * y = sum_q alpha[q] * term[q] (arith.py:173-192: leaf frames concatenated, transfer
   * tensors and root block-diagonal, alpha on the root blocks) whose block-diagonal
   * transfer tensors and root are NOT materialised: node[t] is NULL for every inner
   * node and the root, the leaf frames [U_1 .. U_p] are ordinary device arrays, and
   * rank[t] = sum_q term[q].rank[t].  Accepted by the truncation entry points only:
   * the orthogonalisation sweep's mode products run on the diagonal blocks (SURVEY
   * K9 / 7.4.7: 1 - 1/p^2 of an inner node is structural zeros). */
  const struct ht_sum_src* sum;
} ht_tensor;

/* TruncationControl (arith.py:32-66). eps <= 0 means "no accuracy bound";
 * max_rank <= 0 and max_rank_per_node == NULL means "no cap". */
typedef struct {
  double eps;
  int64_t max_rank;
  const int64_t* max_rank_per_node; /* [2d-1] host or NULL (dict form of max_rank) */
  int32_t flags;                    /* HT_CTL_* bits (0: truncation only) */
} ht_trunc_ctl;

/* The caller reads the hierarchical singular values themselves (every sigma to
 * relative accuracy, also the tiny ones of graded spectra): nodes with graded
 * Gramians go to the Jacobi eigensolver.  Without it, truncation needs only the kept
 * eigenpairs and the tail sums, which the tridiagonal path delivers to the
 * reference's (LAPACK dsyevd) absolute accuracy. */
#define HT_CTL_RELATIVE_SIGMA 1
/* eps is RELATIVE to the norm of the tensor being truncated: the per-node budget is
 * (eps ||x||)^2 / (2d-2) with ||x|| = ||B_D||_F of the orthogonalised root, taken on
 * the device after the orthogonalisation sweep -- the C3 / C4 controls "rel. tol of
 * every truncate's own input" without a separate inner product (and without
 * materialising a Kronecker-form input).  Not available in ht_truncate_sharded. */
#define HT_CTL_RELATIVE_EPS 2

/* GeneralizedMatrix (format.py:135-180). kind: 0 dense (row-major rows x cols),
 * 1 diagonal (values[rows]), 2 CSR (int32 indptr[rows+1], indices[nnz]). */
typedef struct {
  int32_t kind;
  int64_t rows, cols, nnz;
  const double* values;
  const int32_t* indptr;
  const int32_t* indices;
} ht_gmat;

/* HTOperator (format.py:183-250): leaf node t carries rank[t] columns
 * leaf_cols[t][0..rank[t]-1]; transfer/root arrays as for ht_tensor. */
typedef struct {
  int32_t d;
  const int64_t* rank;            /* [2d-1] host */
  const ht_gmat* const* leaf_cols;/* [2d-1] host (NULL entries for non-leaves) */
  double* const* node;            /* [2d-1] device pointers (leaf entries unused) */
} ht_operator;

/* The terms of an unmaterialised block-form sum (see ht_tensor.sum). */
typedef struct ht_sum_src {
  int32_t count;                   /* p >= 2 terms */
  const ht_tensor* const* term;    /* [p] ordinary tensors (kron == sum == NULL), same d and n */
  const double* alpha;             /* [p] host: coefficient of each term (applied to its root block) */
} ht_sum_src;

/* The factors of an unmaterialised y = apply_operator(op, x) (see ht_tensor.kron). */
typedef struct ht_kron_src {
  const ht_operator* op;
  const ht_tensor* x;     /* ordinary tensor (x->kron == NULL) */
} ht_kron_src;

const char* ht_last_error(void);
const char* ht_version(void);

/* ---- tree-level operations (arith.py drivers) ------------------------- */

/* truncate (arith.py:325-352).  Two-phase form for data-dependent ranks:
 *  1. ht_truncate_ranks: orthogonalize (if needed) + reduced Gramians + batched
 *     eigendecomposition + select_rank; SYNCHRONISES the stream and returns the
 *     kept ranks in out_rank[2d-1] (host);
 *  2. ht_truncate_project: projection into `out` (allocated with out_rank),
 *     reusing the state phase 1 left in `ws`.
 * ht_truncate does both without a rank read-back when the ranks are fixed by
 * the shapes (ht_truncate_static_ranks returns 1); see ht_set_qr_mode for the
 * one synchronisation of the Cholesky-QR2 check. */
int ht_truncate_workspace_size(const ht_tensor* x, size_t* bytes);
int ht_truncate_static_ranks(const ht_tensor* x, const ht_trunc_ctl* ctl, int64_t* out_rank);
int ht_truncate_ranks(const ht_tensor* x, const ht_trunc_ctl* ctl, void* ws, size_t ws_bytes,
                      int64_t* out_rank, ht_stream_t stream);
int ht_truncate_project(const ht_tensor* x, const ht_trunc_ctl* ctl, void* ws, size_t ws_bytes,
                        const ht_tensor* out, ht_stream_t stream);
int ht_truncate(const ht_tensor* x, const ht_trunc_ctl* ctl, void* ws, size_t ws_bytes,
                const ht_tensor* out, ht_stream_t stream);
/* CUDA-graph replay of repeated fixed-rank truncations (process-wide, default on;
 * env HT_GRAPHS=0 turns it off at start-up).  The second ht_truncate call with the
 * same shapes, control and kernel policies captures the truncation as two graphs
 * (ORTH; GRAM + EIG + PROJECT) and later calls with the same input / output /
 * workspace addresses replay them; a new address combination runs eagerly once and gets
 * its own graph when it is seen again (up to eight per shape), unless relocation is
 * switched on (below).  Results are identical to the eager launches (same kernels, same
 * arguments). */
int ht_set_graph_mode(int on);
int ht_graph_stats(int64_t* captures, int64_t* replays);
int64_t ht_graph_relocations(void);
/* Relocation of cached graphs to moved buffers: off by default (a new address
 * combination runs eagerly once and is captured when seen again); HT_RELOC=1 or
 * ht_set_graph_relocation(1) turns it on. */
int ht_set_graph_relocation(int on);

/* Sticky error word of the queued (not host-checked) truncations on the current
 * device: fixed-rank ht_truncate, graph replays and the sharded phases OR their
 * eigensolver status into it.  Reads it behind `stream` (synchronising that stream),
 * optionally clears it, and returns HT_ERR_NOT_SYMMETRIC (kernels.py:47-50) or
 * HT_ERR_NONCONVERGED (non-finite Gramian / no convergence) when set.  The Python
 * layer calls it at every host synchronisation point (to_numpy, inner_product,
 * evaluate_entry, synchronize). */
int ht_status(int32_t clear, int32_t* status, ht_stream_t stream);

/* Sharded truncation (the paper's tree-parallel protocol, one subtree per GPU):
 * runs one phase restricted to the nodes with mask[t] != 0 (host array [2d-1]).
 *   phase 0 ORTH   : QR sweep of the masked nodes (R factors of unmasked sons must
 *                    already sit in their workspace slots -- received from the
 *                    shard owning them)
 *   phase 1 GRAM   : reduced Gramians of the sons of masked inner nodes / root
 *   phase 2 EIG    : eigendecomposition + rank choice of masked non-root nodes
 *   phase 3 PROJECT: projection of masked nodes into `out` (unmasked sons' eigen-
 *                    vectors must be in their slots)
 * `owned` (host [2d-1], or NULL = every node) is the node set this shard owns for the
 * whole truncation: the workspace then holds the orthogonalised arrays, R factors,
 * Gramians and eigenpairs of the owned nodes and of their sons (the message slots)
 * only, and phase scratch sized for the owned nodes -- ht_truncate_workspace_size_
 * sharded gives its size (C5, d = 256 on 8 GPUs: ~1/8 of the whole-tree plan).  Every
 * phase mask must lie inside `owned`; the same `owned` must be passed to every phase
 * and slot query of one truncation.
 * Node arrays of unowned nodes are never touched (any non-null pointer).
 * Replaces the node-worker protocol of dist.py:239-333 (_cmd_orth / _cmd_truncate). */
int ht_truncate_workspace_size_sharded(const ht_tensor* x, const uint8_t* owned, size_t* bytes);
int ht_truncate_sharded(const ht_tensor* x, const ht_trunc_ctl* ctl, void* ws, size_t ws_bytes, int32_t phase,
                        const uint8_t* mask, const uint8_t* owned, const ht_tensor* out, ht_stream_t stream);
/* Device pointer + element count of a per-node workspace slot of the truncation:
 * kind 0 R factor, 1 Gramian, 2 eigenvectors, 3 eigenvalues, 4 ranks (int32,
 * all nodes + status word), 5 orthogonalised node array.  Host-only query; with
 * `owned`, only owned nodes and their sons have slots. */
int ht_truncate_slot(const ht_tensor* x, void* ws, const uint8_t* owned, int32_t kind, int32_t node, void** ptr,
                     int64_t* count);

/* Hierarchical singular values: after ht_truncate_ranks, copy the descending,
 * clamped eigenvalues lambda_t of every non-root node's reduced Gramian
 * (sigma_t = sqrt(lambda_t)) into lam (device, concatenated in node-id order). */
int ht_truncate_eigenvalues(const ht_tensor* x, void* ws, size_t ws_bytes, double* lam, ht_stream_t stream);

/* orthogonalize (arith.py:273-296): out has the orthogonalised ranks
 * (ht_orth_ranks) and orthogonal = 1. */
int ht_orth_ranks(const ht_tensor* x, int64_t* out_rank);
int ht_orthogonalize_workspace_size(const ht_tensor* x, size_t* bytes);
int ht_orthogonalize(const ht_tensor* x, void* ws, size_t ws_bytes, const ht_tensor* out, ht_stream_t stream);

/* compute_bhat (arith.py:299-322): reduced Gramian of every non-root node t
 * (rank[t] x rank[t], row-major) at bhat[t]; x must be orthogonal. */
int ht_gramians_workspace_size(const ht_tensor* x, size_t* bytes);
int ht_gramians(const ht_tensor* x, void* ws, size_t ws_bytes, double* const* bhat, ht_stream_t stream);

/* add (arith.py:355-365) and subtract (arith.py:374-375, alpha_c = -1):
 * out ranks are a.rank + c.rank node by node (root 1). No FLOPs (Lemma 3). */
int ht_add(const ht_tensor* a, const ht_tensor* c, double alpha_c, const ht_tensor* out, ht_stream_t stream);
/* Sharded add: only nodes with mask[t] != 0 are read or written (the other node
 * pointers may be placeholders).  Add needs no communication (dist.py add protocol). */
int ht_add_sharded(const ht_tensor* a, const ht_tensor* c, double alpha_c, const uint8_t* mask,
                   const ht_tensor* out, ht_stream_t stream);

/* scale (arith.py:368-371): y = alpha * x elementwise (used on the root). */
int ht_scale(const double* x, double* y, int64_t count, double alpha, ht_stream_t stream);

/* inner_product (arith.py:246-265).  Result written to result_dev (device);
 * if result_host != NULL the stream is synchronised and the value copied. */
int ht_inner_product_workspace_size(const ht_tensor* a, const ht_tensor* c, size_t* bytes);
int ht_inner_product(const ht_tensor* a, const ht_tensor* c, void* ws, size_t ws_bytes,
                     double* result_dev, double* result_host, ht_stream_t stream);
/* Sharded inner product (reference dist.py:239-254 GRAM_UP wave, 516-524): the Phi
 * recursion of the nodes with mask[t] != 0 only (levels bottom-up); Phi of unmasked
 * sons must already sit in their slots (received from the shard that owns them).
 * If the root is masked the result lands in result_dev.  Same workspace size as
 * ht_inner_product; ht_inner_product_slot gives Phi_t's slot (k_a x k_c, row-major). */
int ht_inner_product_sharded(const ht_tensor* a, const ht_tensor* c, const uint8_t* mask, void* ws, size_t ws_bytes,
                             double* result_dev, ht_stream_t stream);
int ht_inner_product_slot(const ht_tensor* a, const ht_tensor* c, void* ws, int32_t node, void** ptr, int64_t* count);

/* apply_operator (arith.py:378-395): out ranks are op.rank * x.rank. */
/* Entry evaluation (reference arith.py:221-243, evaluate_entry): out[b] = X[idx[b, :]]
 * for `count` 0-based multi-indices idx (device int64, count x d, row-major; the
 * caller checks the bounds); one upward pass through the tree per entry. */
int ht_evaluate_entries(const ht_tensor* x, const int64_t* idx, int64_t count, double* out, ht_stream_t stream);

/* Weighted contraction readouts (reference cookie.py:362-426, extract_solution and
 * parameter_mean): as ht_evaluate_entries, but whenever leaf_weights[mu] != NULL the
 * leaf of 0-based dimension mu contributes the row w_mu^T U_mu (w_mu: device, length
 * n_mu) and idx[b, mu] is ignored.  leaf_weights: host array of d device pointers, or
 * NULL (plain entry evaluation). */
int ht_evaluate_weighted(const ht_tensor* x, const double* const* leaf_weights, const int64_t* idx, int64_t count,
                         double* out, ht_stream_t stream);

int ht_apply_operator(const ht_operator* op, const ht_tensor* x, const ht_tensor* out, ht_stream_t stream);
/* apply_operator restricted to mask[t] != 0: node-local, so the sharded form
 * (reference dist.py:324-333 _cmd_apply, 557-566) needs no communication. */
int ht_apply_operator_sharded(const ht_operator* op, const ht_tensor* x, const uint8_t* mask, const ht_tensor* out,
                              ht_stream_t stream);

/* ---- node kernels (kernels.py primitives, batched) ------------------- */

/* reduced_qr (kernels.py:24-32) on `nodes` m x K matrices A(row,col) =
 * A[node*a_node + row*a_r + col*a_c]; Q is m x min(m,K), R is min(m,K) x K
 * row-major (ld r_ld), diag(R) >= 0. */
int ht_qr_workspace_size(int64_t m, int64_t K, int64_t nodes, size_t* bytes);
int ht_qr_batched(int64_t m, int64_t K, int64_t nodes, const double* A, int64_t a_r, int64_t a_c, int64_t a_node,
                  double* Q, int64_t q_r, int64_t q_c, int64_t q_node, double* R, int64_t r_ld, int64_t r_node,
                  void* ws, size_t ws_bytes, ht_stream_t stream);

/* sym_eig_desc (kernels.py:35-54) on `nodes` K x K row-major matrices (K <= 512):
 * eigenvectors V (row-major, columns = eigenvectors), lam descending clamped, by
 * parallel cyclic Jacobi (relative accuracy on graded matrices; K > 112 keeps the
 * matrices in a temporary global scratch).  Synchronises to report
 * HT_ERR_NOT_SYMMETRIC like the reference. */
int ht_syev_batched(int64_t K, int64_t nodes, const double* S, double* V, double* lam, ht_stream_t stream);

/* Strided batched GEMM C = alpha*A*B + beta*C (the mode_multiply / tensordot
 * contractions, kernels.py:92-104). */
int ht_gemm_strided(int64_t M, int64_t N, int64_t K, int64_t batch, double alpha, const double* A, int64_t a_m,
                    int64_t a_k, int64_t a_b, const double* B, int64_t b_k, int64_t b_n, int64_t b_b, double beta,
                    double* C, int64_t c_m, int64_t c_n, int64_t c_b, ht_stream_t stream);

/* QR policy of the orthogonalisation sweep (process-wide).
 *   0 (default): Cholesky-QR on DMMA GEMMs for frames with m >= 2K, K <= 128,
 *      with the second (re-orthogonalisation) pass decided on the device per node
 *      (power-iteration estimate of kappa(R) > 20); the sweep then synchronises
 *      the stream ONCE to read a device red flag (pivot loss > 10 digits,
 *      non-finite values, or Q1^T Q1 not within 0.1 of I) and, if set, recomputes
 *      the whole sweep with Householder QR;
 *   1: Householder tree-TSQR only (no synchronisation);
 *   2: as 0 but both Cholesky-QR passes always run (CholeskyQR2).
 * Both give the unique QR with diag(R) >= 0 of kernels.py:24-32 up to rounding. */
int ht_set_qr_mode(int mode);
/* Implicit Q in truncation (process-wide; default 1, env HT_IMPLICIT_Q).  With 1 the
 * Cholesky-QR sweep of a truncation does not form the orthogonal transfer tensors
 * Q_t = M23(Bp_t) R_t^{-1}: it keeps the absorbed tensor Bp_t and R_t^{-1}, and the
 * Gramian and projection phases fold R_t^{-1} into their small operands
 * (G~ = R^-1 G R^-T, R^-1 Q_t).  Mathematically identical to reference
 * arith.py:325-352; 0 forms Q explicitly (A/B comparisons, tests). */
int ht_set_implicit_q(int on);
/* Number of Cholesky-QR2 sweeps that were re-run with Householder QR. */
int64_t ht_qr_fallback_count(void);
/* Graph replays re-run a flagged Cholesky-QR sweep on the Householder path through a
 * device-side conditional node (no host round trip): 1 when in use, 0 when the
 * driver lacks conditional nodes (host-side flag check), -1 before the first capture. */
int ht_graph_device_fallback(void);

/* Eigensolver policy of the truncation (process-wide).
 *   0 (default): Householder tridiagonalisation + multisection bisection +
 *      twisted-factorisation eigenvectors of the kept eigenpairs; nodes with a
 *      graded spectrum (min|lambda| < 1e-6 max|lambda|) or near-degenerate kept
 *      eigenvalues are redone by the Jacobi kernel in the same stream (no sync);
 *   1: parallel cyclic Jacobi for every node.
 * Both return dsyevd's eigenpairs (kernels.py:35-54) up to rounding / eigenvector
 * sign.  (ht_syev_batched always uses Jacobi.) */
int ht_set_eig_mode(int mode);

/* ---- instrumentation -------------------------------------------------- */

/* Total kernel launches issued by this library since load (always counted). */
int64_t ht_launch_count(void);
/* Bit 0: record a CUDA event pair on the launching stream around every kernel
 * launch and attribute algorithmic flops/bytes per kernel; bit 1: keep a
 * launch-order log of kernel tags (no events; for matching ncu launch lists);
 * bit 2 (with bit 0): one report entry per launch, keyed "tag#seq".
 * Clears the tally and the log. */
int ht_profile_enable(int on);
/* The launch-order log as JSON [["tag", flops, bytes], ...]; returns its length. */
int ht_profile_log(char* buf, size_t len);
/* Writes {"kernel": {"ms", "launches", "flops", "bytes"}, ...} JSON into buf
 * (synchronises the recorded events); returns the full JSON length. */
int ht_profile_report(char* buf, size_t len);

#ifdef __cplusplus
}
#endif

#endif /* HT_B200_H */
