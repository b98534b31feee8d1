/*
 * f2c_dcp.h -- C ABI of libf2c_dcp.so, the B200 (sm_100a) implementation of the
 * Dynamic Class Pool (DCP) head of F2C (arXiv 2105.10375).
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; Dn = reading n of
 * DESIGN.md section 3 (where the paper is silent or ambiguous).
 *
 * Conventions (every entry point):
 *   - Pointers are DEVICE pointers unless marked (host).  Device buffers are owned
 *     by the caller (allocated by torch); the library never allocates device
 *     memory.  It owns only host bookkeeping and, for world > 1, an NCCL
 *     communicator.
 *   - `stream` is a cudaStream_t passed as void*.  Every call validates its
 *     arguments on the host, enqueues work on `stream` and returns without
 *     synchronising (except the *_state / row_stats / check debug calls).
 *   - Return value: F2C_OK (0) or an f2c_status code; f2c_last_error() returns a
 *     thread-local message for the last failure on the calling thread.
 *   - Errors that only the device can see (negative labels in device buffers,
 *     pairing mismatches, zero-norm rows, non-finite loss, softmax underflow that
 *     the kernels could not absorb) are latched in a device error word.  The
 *     kernel that latches one also writes it to a mapped pinned host word of the
 *     handle, and every later f2c_dcp_enqueue / f2c_dcp_loss_fwd_bwd call reads
 *     that word before launching anything (no synchronisation, no copy): the first
 *     such call made after the error became visible to the host returns it
 *     (F2C_EPAIRING / F2C_EDEVICE, message via f2c_last_error) and launches
 *     nothing, and so does every later call until f2c_dcp_check() clears the
 *     latch.  Calls issued while the latching kernel is still queued or running
 *     cannot see it yet; f2c_dcp_check() synchronises and always reports it.
 *   - dtype: F2C_BF16 (pool and features bf16, fp32 accumulation) or F2C_F32
 *     (fp32 pool, features, x and dx; BJ:7's c0, reading D21): the logits are
 *     tf32 tensor-core products of the fp32 values (fp32 accumulation) and the
 *     P x pool product reads a bf16 shadow of the pool kept by the enqueue; the
 *     F2C_F32 loss call needs d <= 256 (x_hat lives in TMEM as fp32), F2C_EINVAL
 *     otherwise.  Feature dimension d: multiple of 128, <= 512.
 *   - No CPU fallback: on a host without a usable sm_100 device every entry point
 *     that launches work returns F2C_ECUDA.
 */
#ifndef F2C_DCP_H
#define F2C_DCP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct f2c_dcp f2c_dcp; /* opaque handle, one per rank (or one per emulated world) */

enum f2c_dtype { F2C_BF16 = 0, F2C_F32 = 1 };

enum f2c_status {
    F2C_OK = 0,
    F2C_EINVAL = 1,    /* bad configuration argument                        */
    F2C_ESHAPE = 2,    /* size / shape mismatch                      */
    F2C_ECAPACITY = 3, /* block larger than the pool, B_id > C              */
    F2C_EPAIRING = 4,  /* pairing[i] does not name row i's target (D13)             */
    F2C_ECUDA = 5,     /* CUDA runtime / driver failure or no sm_100 device         */
    F2C_ENCCL = 6,     /* NCCL failure (world > 1)                                  */
    F2C_EDEVICE = 7    /* latched device error: bad label, zero-norm row, non-finite
                          loss, unabsorbed softmax underflow                */
};

/* Bytes of the caller-owned device state buffer for one rank: this rank's pool
 * shard (rows [floor(r*C/W), floor((r+1)*C/W)) of the C slots, dtype, row-major
 * [C_loc][d]) plus labels and all per-step scratch for batches of up to
 * n_local_max rows and enqueue blocks of up to m_local_max rows per rank.
 * rank = -1 sizes an EMULATED world: all W shards on one device in one handle.
 * Returns 0 on invalid arguments. */
size_t f2c_dcp_state_bytes(int64_t C, int32_t d, int32_t dtype, int32_t world, int32_t rank,
                           int64_t n_local_max, int64_t m_local_max);

/* Create the DCP of capacity C ("a tensor T with size C x K x D", K = 1 (D1)).
 * The pool starts EMPTY: occupied slots are exactly [0, min(E, C)) where E counts
 * rows ever enqueued, so the paper's Gaussian initialisation is
 * unobservable and not materialised (D9).
 * world, rank: slot-range sharding over `world` processes (one per GPU); for
 *   world > 1 the call is collective and nccl_uid (host, 128 bytes, an
 *   ncclUniqueId from rank 0, broadcast by the caller) is required; NULL iff
 *   world == 1.  rank = -1 with world >= 1 creates an emulated world (all shards
 *   in this process on the current device; collectives become device copies) --
 *   a test vehicle with exactly the multi-rank arithmetic.
 * state_buf: device buffer of at least f2c_dcp_state_bytes(...) bytes, 256-byte
 *   aligned, owned by the caller and kept alive until f2c_dcp_destroy.  The
 *   library zeroes it (synchronously) during create.
 * out (host): receives the handle. */
int f2c_dcp_create(int64_t C, int32_t d, int32_t dtype, int32_t world, int32_t rank,
                   const void *nccl_uid, void *state_buf, size_t state_bytes,
                   int64_t n_local_max, int64_t m_local_max, f2c_dcp **out);

/* K features per slot (NEXT-1; the paper's default K = 2): the pool is
 * T [C][K][d] bf16.  Eq. 8's logits use T_bar_c = (1/K) sum_k T[c,k]; for K >= 2
 * L_cos uses the true cosine <x_hat, T_bar_c>/||T_bar_c|| (reading R4; a zero
 * center contributes 0).  Enqueue then takes g_feats [m_local][K][d] (k-fill mode;
 * the paper-literal mode duplicates one feature over K on the caller's side);
 * get_state / set_state exchange [C_loc][K][d].  K in [1, 8]; K > 1 requires bf16.
 * f2c_dcp_create / f2c_dcp_state_bytes are these with K = 1. */
size_t f2c_dcp_state_bytes_k(int64_t C, int32_t K, int32_t d, int32_t dtype, int32_t world,
                             int32_t rank, int64_t n_local_max, int64_t m_local_max);
int f2c_dcp_create_k(int64_t C, int32_t K, int32_t d, int32_t dtype, int32_t world, int32_t rank,
                     const void *nccl_uid, void *state_buf, size_t state_bytes,
                     int64_t n_local_max, int64_t m_local_max, f2c_dcp **out);

/* NEXT-3 variants of the L_cos term, applied by every later loss call on this handle.
 * The paper names phi only as "calculating the cosine similarity" between the out-of-pool
 * features and T and sums L_ce + L_cos unweighted; SPEC leaves the
 * reduction over the pool and a hinge open.
 *   phi_mode 0 = mean over the occupied centers (default, D10), 1 = sum, 2 = max (hardest
 *            negative; the first slot wins ties);
 *   hinge    1 replaces cos by max(0, cos) (only positive similarity is penalised);
 *   lambda   L = L_ce + lambda L_cos (default 1).
 * Cosines are the true cosines for K >= 2 (R4); zero centers are skipped.  Modes
 * other than (mean or sum, no hinge) run the out-of-pool rows through the fused kernel
 * too (their GEMM cost is the in-pool rows').  Errors: F2C_EINVAL for out-of-range values. */
int f2c_dcp_set_lcos(f2c_dcp *h, int32_t phi_mode, int32_t hinge, double lambda);

/* NEXT-3 variant of Eq. 9's denominator for pools holding several slots with one label
 * (possible under pure Eq. 7, D7).  The paper sums over every slot j = 1..C, so by
 * default (exclude_stale = 0, reading D8) an in-pool row's OLDER slots of its own label stay
 * in the softmax as ordinary, unmargined negatives.  exclude_stale = 1 drops them from the
 * row's softmax (and hence from p and dx): the row is then scored as if those stale slots
 * had been deleted.  The target is still the newest slot (D8); out-of-pool rows and L_cos are
 * unaffected.  Applies to every later loss call on this handle.  Cost: two extra passes over
 * the shard's slot labels per loss call.  Errors: F2C_EINVAL unless exclude_stale is 0 or 1. */
int f2c_dcp_set_dup_mode(f2c_dcp *h, int32_t exclude_stale);

/* NEXT-3 enqueue variant: SPEC's refresh-in-place insert ("If an id is
 * already resident, its features are overwritten in place and its queue position is
 * unchanged"; reading R7 in DESIGN.md).  With refresh_in_place = 1, later enqueues on this
 * handle do, for the global block (rows j, labels y_j):
 *   - y_j must be pairwise distinct (a duplicate latches F2C_EDEVICE) and >= 0;
 *   - sigma_j = write index of the newest occupied slot with label y_j (D8), if any;
 *   - n = the smallest n >= n0 (rows with no resident slot) with
 *     n = n0 + #{j : sigma_j exists, sigma_j < E + n - C}: the resident rows whose slot the
 *     appends overwrite are appended too, so every block id is resident afterwards;
 *   - appended rows go, in block order, to slots (E + k) mod C, k < n; the other rows
 *     overwrite the features of their resident slot (label and age unchanged); E += n.
 * The pairing check of the next loss call follows each row's actual slot.  Because n is
 * data-dependent, a refresh enqueue synchronises `stream` before it returns (the host
 * bookkeeping needs E).  refresh_in_place = 0 restores pure Eq. 7 (D7).
 * Errors: F2C_EINVAL unless refresh_in_place is 0 or 1; F2C_ECUDA if pinned memory fails. */
int f2c_dcp_set_enqueue_mode(f2c_dcp *h, int32_t refresh_in_place);

/* Enqueue one identity block (Eq. 7 + Algorithm 1):
 * the global block is the concatenation of every rank's g_feats in rank order
 * (emulated world: g_feats already holds the concatenation, world*m_local rows).
 * Global block row j is written to slot (E + j) mod C with its label; then E +=
 * world * m_local.  While E < C this is the sequential fill of Algorithm 1; after
 * that it overwrites the oldest rows, i.e. Eq. 7's shift up to relabelling (D6).
 * A resident identity is not refreshed in place: duplicates may coexist (D7).
 * g_feats: [m_local, d] dtype row-major; labels: [m_local] int64, each >= 0
 *   (checked on the device; -1 is reserved for empty slots).
 * Requires 1 <= world*m_local <= C and m_local <= m_local_max.  Collective for
 * world > 1 (the rows are routed to the owners of their slots). */
int f2c_dcp_enqueue(f2c_dcp *h, const void *g_feats, const int64_t *labels, int64_t m_local,
                    void *stream);

/* Loss forward + backward of the DCP head (Eq. 6 split P:124-133, Eq. 8 logits
 * P:155-159 with K = 1, Eq. 9 CE P:160-164, L_cos P:165-169, L_total P:170):
 *   for every row i of the global batch X (rank-ordered concatenation of every
 *   rank's x; emulated world: x is already the concatenation):
 *     x_hat_i = x_i / ||x_i||;  cos_ic = <x_hat_i, T_c> for occupied slots c;
 *     t_i = the occupied slot with label y_i and the newest write (D8), if any.
 *   In-pool rows (t_i exists, count N_pos = I):
 *     z_ic = s cos_ic, z_it = s (cos_it - m)  (cosine margin, D3);
 *     L_ce = (1/N_pos) sum_i [logsumexp_c z_ic - z_it].
 *   Out-of-pool rows (count N_neg = M - I):
 *     L_cos = (1/N_neg) sum_i mean_c cos_ic  (mean reduction of phi, D10).
 *   loss = L_ce + L_cos (empty sets contribute 0, D11);  dx = dL/dx for the raw
 *   local rows including the normalisation Jacobian (D12).  The pool takes no
 *   gradient.
 * x: [n_local, d] dtype; labels: [n_local] int64 >= 0;
 * pairing: [n_local] int32 or NULL: pairing[i] = j >= 0 asserts that row i's
 *   target is row j of the most recent global enqueue block (checked on the
 *   device, F2C_EPAIRING); -1 marks an instance row (D13);
 * s > 0 (logit scale), m finite (cosine margin).  The softmax runs against a per-row reference
 *   2^b_r, b_r = max(target logit, bound - 100) in log2 units (R1), exact up to s ~ 69
 *   with unit-norm features; for s > 68 a refinement pass lowers the reference of any row whose
 *   terms fell far below it to that row's exact maximum and re-runs the fused kernel (its CTAs
 *   exit at once when no row needs it).  A row still underflowing latches F2C_EDEVICE;
 * loss: device fp32 scalar (global-batch loss, identical on every rank);
 * dx: [n_local, d] dtype, must not alias x.  For world > 1, dx is the gradient of
 *   the GLOBAL loss w.r.t. this rank's rows: backbone gradients must be summed,
 *   not averaged, across ranks.
 * Every rank must pass the same n_local, s and m. */
int f2c_dcp_loss_fwd_bwd(f2c_dcp *h, const void *x, const int64_t *labels, const int32_t *pairing,
                         int64_t n_local, float s, float m, float *loss, void *dx, void *stream);

/* G-Net moving-average update ("inherits parameters from P-Net in a moving
 * average manner"): g_k <- m*g_k + (1-m)*p_k for k < n, evaluated in
 * fp64 exactly in that order and rounded to nearest-even fp32 (D17).  p, g: fp32,
 * 16-byte aligned, may not overlap; 0 <= momentum <= 1. */
int f2c_gnet_ema(const float *p, float *g, int64_t n, double momentum, void *stream);

/* ---- support: parity, checkpoint/resume, debugging (all synchronous) ------- */

/* Copy this handle's pool out: feats_host [C_loc, d] dtype (emulated world: all C
 * slots in global order), labels_host [C_loc] (-1 = empty), *enq_count_host = E. */
int f2c_dcp_get_state(f2c_dcp *h, void *feats_host, int64_t *labels_host, int64_t *enq_count_host);

/* Restore a pool (same layout as get_state).  Slots >= min(E, C) must be empty
 * (label -1); their features are ignored and stored as zeros.  The next enqueue
 * writes at E mod C.  The derived state is rebuilt from the restored slots: the
 * running norm bound (R1), T_bar and w_c for K >= 2 (R5), an fp32 pool's bf16 shadow
 * (D21), the label index of target resolution (label -> newest write index, DESIGN.md
 * section 6), and the pool sum mu of the L_cos gradient (R3; the enqueue keeps it as an
 * exact fixed-point running sum, so a restored handle continues bit-identically). */
int f2c_dcp_set_state(f2c_dcp *h, const void *feats_host, const int64_t *labels_host,
                      int64_t enq_count);

/* Per-row results of the last loss call, global-batch order, host arrays of
 * n_global entries each (any may be NULL): lse (natural log-sum-exp with the
 * margin, 0 for out-of-pool rows), target_seq (global write index of the target
 * slot, -1 = out of pool), cos_t (cosine to the target), phi (mean cosine for
 * out-of-pool rows), ell (per-row CE term), counts (host int64[3] = N_pos, N_neg,
 * C_occ).  n_global = world * n_local of that call. */
int f2c_dcp_row_stats(f2c_dcp *h, float *lse, int64_t *target_seq, float *cos_t, float *phi,
                      float *ell, int64_t *counts);

/* Synchronise the last stream used with the handle and return the latched device
 * error (F2C_OK, F2C_EPAIRING or F2C_EDEVICE, or F2C_ENCCL for an asynchronous
 * NCCL error); clears the latch (device word and host mirror). */
int f2c_dcp_check(f2c_dcp *h);

/* Thread-local message for the last non-OK return on this thread. */
const char *f2c_last_error(void);

/* Number of kernel launches issued by the last enqueue / loss / ema call on this
 * thread (for the bench's gpu_launches accounting). */
int f2c_last_launch_count(void);

/* Kernel timing for the bench (CUDA events recorded on the launching stream around
 * the fused loss kernel of every loss call while enabled).  enable=1 starts (and
 * resets) accumulation, enable=0 stops.  f2c_dcp_profile_read synchronises and
 * returns the summed device time of the fused kernel (ms), the number of timed
 * launches, and the sum of N_pos over those calls. */
int f2c_dcp_profile(f2c_dcp *h, int enable);
int f2c_dcp_profile_read(f2c_dcp *h, double *main_ms, int64_t *launches, int64_t *n_pos_sum);

/* Which fused loss kernel a loss call with n_global global rows runs on this handle (the
 * choice depends on the variant, K, d and F2C_KERNEL): *kind = 0
 * dcp_pc_kernel (CTA pairs, 128-row groups), 1 dcp_tp64_kernel, 2 dcp_pc4_kernel
 * (cta_group::2 SM pairs, 256-row groups); *ctas = its persistent grid (CTAs).  Host only. */
int f2c_dcp_fused_kernel(f2c_dcp *h, int64_t n_global, int32_t *kind, int32_t *ctas);

/* C5 routing plan of a pure Eq. 7 enqueue across `world` ranks (SURVEY 8(e) stage 0, P:143-151;
 * host only: no handle, no device).  The global block is every rank's m_local rows in rank order,
 * block row j goes to slot (E + j) mod C (Eq. 7 on the ring, D6), and slot p belongs to rank q
 * with floor(qC/W) <= p < floor((q+1)C/W).  Writes pieces[4 i .. 4 i + 3] = (source rank,
 * destination rank, first global block row, rows): every run of block rows of one sender whose
 * slots are contiguous inside one destination shard, ordered by source rank then block row -- the
 * order in which both ends issue their sends and receives.  At most 2 world + 1 pieces.
 * Returns the piece count, or -1 for invalid arguments or max_pieces too small. */
int64_t f2c_c5_plan(int64_t C, int32_t world, int64_t E, int64_t m_local, int64_t *pieces, int64_t max_pieces);

/* Release host resources and the NCCL communicator.  The caller frees state_buf. */
void f2c_dcp_destroy(f2c_dcp *h);

#ifdef __cplusplus
}
#endif
#endif /* F2C_DCP_H */
