/*
 * sparsemlp_b200.h -- C ABI of the B200 (sm_100a) static-sparse MLP training path.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `sparsemlp` (arxiv 2407.17437, "Nerva"): the four CSR kernels of
 * pkg/src/sparsemlp/_kernels.py, the validated operators of tensor_core.py that
 * wrap them, and the per-step glue of nn.py / train.py that runs between them
 * (bias, ReLU, softmax cross-entropy, optimizer arithmetic, batch gather,
 * Xavier init).  The reference binds its kernels by name from Python
 * (nn.py:16-23 imports spmm/spmm_transposed/sddmm/sparse_combine from
 * tensor_core); a maintainer would bind these symbols with ctypes instead
 * (see INTEGRATION.md).
 *
 * Conventions (all entry points):
 *   - every pointer is a DEVICE pointer unless documented otherwise; the caller
 *     owns all buffers (the library never allocates on the hot path);
 *   - dense operands are row-major [rows x ld] with the logical width `n`
 *     (the reference's feature-major [features, batch] layout, nn.py:3-8);
 *   - `dtype` is SMB_F32 or SMB_F64 (CsrMatrix accepts both,
 *     tensor_core.py:170-171); engine-only ops are float32;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *   - calls are stream-ordered, never synchronise, and are reentrant on
 *     disjoint outputs;
 *   - return value: SMB_OK, or an SMB_ERR_* code with a message available from
 *     smb_last_error() (thread-local).  The Python layer maps
 *     SMB_ERR_INVALID -> InvalidArgumentError and SMB_ERR_STATE -> StateError
 *     (errors.py:4-9).
 *
 * Rounding contract ("exact" kernels): every output element is accumulated in
 * ascending source index with multiply and add rounded separately (no FMA
 * contraction), exactly as the numba kernels do with fastmath off
 * (_kernels.py:1-6).  spmm, spmm_t, sddmm, axpby, the fused optimizer update,
 * row_sums (numpy pairwise order) and relu/relu_backward are therefore
 * bit-identical to the reference given identical inputs.
 */
#ifndef SPARSEMLP_B200_H
#define SPARSEMLP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SMB_API __attribute__((visibility("default")))
#else
#define SMB_API
#endif

#define SMB_ABI_VERSION 1

/* status codes */
#define SMB_OK 0
#define SMB_ERR_INVALID 1 /* InvalidArgumentError (errors.py:4) */
#define SMB_ERR_STATE 2   /* StateError (errors.py:8) */
#define SMB_ERR_CUDA 3    /* CUDA launch / runtime failure */

/* value dtypes */
#define SMB_F32 0
#define SMB_F64 1

/* epilogues of smb_spmm */
#define SMB_EPI_NONE 0
#define SMB_EPI_RELU 1 /* y = max(y, 0) as np.maximum (nn.py:86-87) */

/* optimizer kinds (nn.py:42-72, SparseLinearLayer.optimize nn.py:187-198) */
#define SMB_OPT_NONE 0     /* gradient only, no update */
#define SMB_OPT_GD 1       /* w += f(-eta) * g                                   nn.py:196-197 */
#define SMB_OPT_MOMENTUM 2 /* v = f(mu) v + g;  w += f(-eta) * v                 nn.py:190,194-195 */
#define SMB_OPT_NESTEROV 3 /* v = f(mu) v + g;  w += f(-eta*mu) v;  w += f(-eta) g  nn.py:190-193 */

/* ---- library info -------------------------------------------------------- */

SMB_API int smb_abi_version(void);
/* Thread-local message of the last failing call on this thread ("" if none). */
SMB_API const char* smb_last_error(void);
/* Number of kernels this library has launched in this process (all threads). */
SMB_API uint64_t smb_launch_count(void);

/* ---- the four reference kernels ------------------------------------------ */

/* out[i,:] = sum_{p in row i, ascending} values[p] * dense[col_idx[p], :]
 *            (+ bias[i]) (then ReLU if epilogue == SMB_EPI_RELU).
 * Replaces _kernels.spmm_kernel (_kernels.py:25-37) via tensor_core.spmm
 * (tensor_core.py:227-240), fused with the bias add of
 * SparseLinearLayer.forward (nn.py:173) and ReLU.forward (nn.py:86-87).
 * Rows without nonzeros produce bias (or 0). m x k CSR, dense k x n, out m x n. */
SMB_API int smb_spmm(int dtype, const int32_t* row_ptr, const int32_t* col_idx, const void* values,
             int64_t m, int64_t k, const void* dense, int64_t ld_dense, int64_t n,
             const void* bias, int epilogue, void* out, int64_t ld_out, void* stream);

/* ---- SparsityPattern handle (tensor_core.py:97-152) -------------------------
 * The static CSR structure shared by a layer's weights, gradient and velocity
 * (nn.py:148-158), plus the indices derived from it once per layer:
 * a CSC transpose index (col_ptr[k+1], row_idx[nnz] ascending inside each
 * column, perm[nnz] = CSC slot -> CSR value index), which replaces the
 * O(nblocks*nnz) rescan of _kernels.spmm_t_kernel (_kernels.py:40-59), and the
 * SDDMM tile index.  row_ptr / col_idx are BORROWED device arrays and must
 * outlive the handle; the pattern is immutable (tensor_core.py:128-133).
 * With validate != 0 the structure is checked on the device like
 * tensor_core._validate_structure (tensor_core.py:78-94) and a violation
 * returns SMB_ERR_INVALID with the reference's message.  Setup-time call: it
 * allocates and synchronises `stream`. */
typedef struct smb_pattern smb_pattern;
SMB_API int smb_pattern_create(const int32_t* row_ptr, const int32_t* col_idx, int64_t m, int64_t k,
                       int64_t nnz, int validate, void* stream, smb_pattern** out);
SMB_API int smb_pattern_destroy(smb_pattern* pattern);
/* copy the CSC index into caller-owned device buffers (col_ptr[k+1],
 * row_idx[nnz], perm[nnz]; any may be NULL), stream-ordered. */
SMB_API int smb_pattern_csc(const smb_pattern* pattern, int32_t* col_ptr, int32_t* row_idx,
                            int32_t* perm, void* stream);

/* smb_spmm through a pattern handle: the same product, order and epilogue
 * (tensor_core.spmm, tensor_core.py:227-240; nn.py:169-176, 86-87); the
 * handle's nonzero count selects the lane width (short rows: 2 x 16 bytes
 * per lane, long rows: 16 bytes). */
SMB_API int smb_spmm_p(int dtype, const smb_pattern* pattern, const void* values,
                       const void* dense, int64_t ld_dense, int64_t n, const void* bias,
                       int epilogue, void* out, int64_t ld_out, void* stream);

/* out[c,:] = sum_{i ascending} values[perm[q]] * dense[i,:] over the column-c
 * slots q of the CSC index, then out *= (mask[c,:] > 0) when mask != NULL.
 * Replaces _kernels.spmm_t_kernel (_kernels.py:40-59) via
 * tensor_core.spmm_transposed (tensor_core.py:243-255), fused with
 * ReLU.backward of the layer below (nn.py:89-91: d * (x_cached > 0); the
 * post-activation A satisfies A > 0 <=> x_cached > 0).  `values` are in CSR
 * order.  dense m x n, out k x n. */
SMB_API int smb_spmm_t(int dtype, const smb_pattern* pattern, const void* values, const void* dense,
               int64_t ld_dense, int64_t n, const void* mask, int64_t ld_mask, void* out,
               int64_t ld_out, void* stream);

/* smb_spmm_t with the values already in CSC slot order (values_csc[q] =
 * values[perm[q]], see smb_values_to_csc): the same sums bit for bit without
 * the per-nonzero indirection through perm.  The training step keeps such a
 * copy next to each layer's value buffer (refreshed after every update on
 * the update's own stream): config-4 hidden layer 149 -> 132 us, config-5
 * 608 -> 503 us (scripts/probe_spmm_t_cost.py). */
SMB_API int smb_spmm_t_csc(int dtype, const smb_pattern* pattern, const void* values_csc,
                           const void* dense, int64_t ld_dense, int64_t n, const void* mask,
                           int64_t ld_mask, void* out, int64_t ld_out, void* stream);

/* values_csc[q] = values[perm[q]] for the nnz CSC slots q of the pattern
 * (the CSR -> CSC permutation of a value array; no reference counterpart:
 * the reference's spmm_t_kernel indexes values in CSR order). */
SMB_API int smb_values_to_csc(int dtype, const smb_pattern* pattern, const void* values,
                              void* values_csc, void* stream);

/* smb_spmm_t plus the bias side of the layer BELOW, fused into the epilogue:
 * grad_bias[c] = row_sums(out[c, :]) in numpy's pairwise order (nn.py:184,
 * tensor_core.py:353-356) and the optimizer update of bias / velocity_bias
 * (_step_vector, nn.py:118-131) -- out is that layer's output gradient
 * d_out, so this is the exact bias arithmetic of its backward + optimize.
 * opt_kind == SMB_OPT_NONE only writes grad_bias_out (data-parallel path). */
SMB_API int smb_spmm_t_bias(int dtype, const smb_pattern* pattern, const void* values,
                            const void* dense, int64_t ld_dense, int64_t n, const void* mask,
                            int64_t ld_mask, void* out, int64_t ld_out, void* bias,
                            void* velocity_bias, void* grad_bias_out, int opt_kind, double mu,
                            double eta, void* stream);

/* out_values[p] = a[i,0]*b[j,0] + a[i,1]*b[j,1] + ... (sequential over the
 * n columns) for the p-th stored (i, j).  n == 0 gives zeros.
 * Replaces _kernels.sddmm_kernel (_kernels.py:62-75) via tensor_core.sddmm
 * (tensor_core.py:258-288).  a m x n, b k x n. */
SMB_API int smb_sddmm(int dtype, const smb_pattern* pattern, const void* a, int64_t lda, const void* b,
              int64_t ldb, int64_t n, void* out_values, void* stream);

/* s[p] = T(alpha) * s[p] + T(beta) * t[p]   (alpha/beta pre-cast to the value
 * dtype as tensor_core.py:304-305).  Replaces _kernels.axpby_kernel
 * (_kernels.py:78-83) via tensor_core.sparse_combine (tensor_core.py:291-306). */
SMB_API int smb_axpby(int dtype, double alpha, void* s, double beta, const void* t, int64_t count,
              void* stream);

/* ---- fused training-step ops ---------------------------------------------- */

/* One launch for the whole weight side of SparseLinearLayer.backward+optimize
 * (nn.py:178-198): grad = sddmm(pattern, d_out, x) (nn.py:183),
 * grad_bias = row_sums(d_out) (nn.py:184, numpy pairwise order), then the
 * optimizer update of values/velocity (the sparse_combine sequence
 * nn.py:189-197) and of bias/velocity_bias (_step_vector, nn.py:118-131).
 * With opt_kind == SMB_OPT_NONE nothing is updated and grad_out /
 * grad_bias_out receive the gradients (data-parallel path: allreduce, then
 * smb_optimizer_step).  grad_out / grad_bias_out may be NULL otherwise.
 * velocity / velocity_bias may be NULL for SMB_OPT_GD and SMB_OPT_NONE.
 * bias / velocity_bias / grad_bias_out may all be NULL (no bias).
 * NOTE: spmm_t of this layer must run BEFORE this call (it reads pre-update
 * values, train.py:400-401). */
SMB_API int smb_sddmm_update(int dtype, const smb_pattern* pattern, const void* d_out, int64_t ld_dout,
                     const void* x, int64_t ld_x, int64_t n, void* values, void* velocity,
                     void* grad_out, void* bias, void* velocity_bias, void* grad_bias_out,
                     int opt_kind, double mu, double eta, void* stream);

/* smb_sddmm_update with the pre-update values read from `values` and the
 * updated values written to `values_out` (may equal `values`).  Lets the
 * training step keep two value buffers so the transposed SpMM of the same
 * layer (which must see the pre-update weights, train.py:400-401) can run
 * concurrently with the update on another stream.
 * opt_kind may carry SMB_HINT_CONCURRENT (OR-ed in): the launch shares the
 * GPU with other kernels, so small layers on the general cp.async kernel take
 * the staging ring with the smallest shared-memory footprint (same results
 * bit for bit; the lean one-warp kernel's ring was chosen inside the step and
 * ignores the hint). */
#define SMB_HINT_CONCURRENT 0x100
SMB_API int smb_sddmm_update_into(int dtype, const smb_pattern* pattern, const void* d_out,
                                  int64_t ld_dout, const void* x, int64_t ld_x, int64_t n,
                                  const void* values, void* values_out, void* velocity,
                                  void* grad_out, void* bias, void* velocity_bias,
                                  void* grad_bias_out, int opt_kind, double mu, double eta,
                                  void* stream);

/* grad_bias = row_sums(d_out) (numpy pairwise order) and the bias optimizer
 * update; one warp per row (nn.py:184, 118-131).  Dense layers and any
 * layer whose output gradient was not produced by smb_spmm_t_bias. */
SMB_API int smb_bias_grad_update(int dtype, const void* d_out, int64_t ld, int64_t m, int64_t n,
                                 void* bias, void* velocity_bias, void* grad_bias_out,
                                 int opt_kind, double mu, double eta, void* stream);

/* param/velocity update from a gradient segment with the exact
 * sparse_combine / _step_vector rounding (nn.py:118-131, 187-198). */
SMB_API int smb_optimizer_step(int dtype, void* param, void* velocity, const void* grad, int64_t count,
                       int opt_kind, double mu, double eta, void* stream);

/* The data-parallel update pass in one launch: `segments` is a DEVICE array of
 * n_segments (<= 32) records {void* param; void* velocity; const void* grad;
 * const void* mask; int64_t start;} -- element e of the concatenation
 * (start[i] <= e < start[i+1], the last segment ends at `total`) is updated
 * exactly like smb_optimizer_step (mask == NULL) or
 * smb_masked_optimizer_step (nn.py:118-131, 187-198, 255-263). */
SMB_API int smb_optimizer_step_multi(int dtype, const void* segments, int n_segments,
                                     int64_t total, int opt_kind, double mu, double eta,
                                     void* stream);

/* Masked-dense baseline update, DenseLinearLayer.optimize with a mask
 * (nn.py:258-264, gradient masked as in backward nn.py:255-256):
 * g' = grad*mask, velocity *= mask, _step_vector(param, g', velocity),
 * param *= mask -- one pass over count elements. */
SMB_API int smb_masked_optimizer_step(int dtype, void* param, void* velocity, const void* grad,
                                      const void* mask, int64_t count, int opt_kind, double mu,
                                      double eta, void* stream);

/* out[i] = sum_t dense[i, t] in numpy's pairwise order (tensor_core.row_sums,
 * tensor_core.py:353-356). */
SMB_API int smb_row_sums(int dtype, const void* dense, int64_t m, int64_t n, int64_t ld, void* out,
                 void* stream);

/* d_y = (softmax_columns(y) - t) / divisor   (nn.py:385-389, 411-417 and the
 * "/ batch_size" of train.py:399).  y, t, d_y are classes x n.  If loss_out
 * (device double[1]) is not NULL it receives softmax_ce_loss(y, t)
 * (nn.py:397-408, summed over the batch, not divided).  exp is the
 * full-accuracy expf (<= 2 ulp; numpy's float32 exp is not correctly rounded
 * either), so this op is tolerance-exact, not bit-exact. */
SMB_API int smb_softmax_ce_grad(int dtype, const void* y, int64_t ld_y, const void* t, int64_t ld_t,
                        int64_t classes, int64_t n, double divisor, void* d_y, int64_t ld_dy,
                        double* loss_out, void* stream);

/* The loss step of the fused training step: smb_softmax_ce_grad over
 * ceil(n/256) CTAs, whose last CTA additionally (a) reduces the batch loss in
 * a fixed order into loss_out, (b) applies the last layer's bias side
 * (row sums of d_y + update, as smb_bias_grad_update) and (c) advances
 * *step_counter modulo `modulo` (CUDA-graph replays of the step).  Any of
 * loss_out / bias / grad_bias_out / step_counter may be NULL.  `workspace`
 * (device, smb_softmax_ce_workspace_bytes(n) bytes, zeroed once before first
 * use) holds the CTA ticket and the per-CTA loss partials. */
SMB_API size_t smb_softmax_ce_workspace_bytes(int64_t n);
SMB_API int smb_softmax_ce_step(int dtype, const void* y, int64_t ld_y, const void* t,
                                int64_t ld_t, int64_t classes, int64_t n, double divisor,
                                void* d_y, int64_t ld_dy, double* loss_out, void* bias,
                                void* velocity_bias, void* grad_bias_out, int opt_kind, double mu,
                                double eta, int32_t* step_counter, int32_t modulo,
                                void* workspace, void* stream);

/* d_x = W^T d_out for a dense layer of m <= 32 output rows (the
 * ER-saturated output layer; DenseLinearLayer.backward, nn.py:241-255),
 * each element summed over ascending i with separately rounded multiply /
 * add, then d_x *= (mask > 0) when mask != NULL (ReLU.backward of the layer
 * below, nn.py:89-91).  W is [m, ld_w] row-major, d_out [m, ld_d], mask /
 * d_x [k, ld].  One HBM pass over mask and d_x (the cuBLAS product plus a
 * separate mask kernel make three). */
SMB_API int smb_dense_backward_input(int dtype, const void* w, int64_t ld_w, int64_t m, int64_t k,
                                     const void* d_out, int64_t ld_d, int64_t n,
                                     const void* mask, int64_t ld_mask, void* d_x,
                                     int64_t ld_dx, void* stream);

/* Weight side of a dense layer of m <= 32 output rows (the ER-saturated
 * output layer; DenseLinearLayer.backward + optimize, nn.py:241-264):
 *   grad[i, c] = sum_t d_out[i, t] * x[c, t]   (one sequential chain per
 *   element over ascending t, multiply and add rounded separately -- the
 *   SDDMM chain of _kernels.py:62-75 over a full pattern; the reference's
 *   d @ x.T is numpy BLAS, so parity is tolerance-exact)
 * then the optimizer update of w[i, c] / velocity[i, c] (_step_vector,
 * nn.py:118-131) in the same launch.  opt_kind == SMB_OPT_NONE writes the
 * gradient to grad_out ([m, k] contiguous; data-parallel path) and updates
 * nothing; grad_out may be NULL otherwise.  d_out [m, ld_d], x [k, ld_x],
 * w / velocity [m, ld_w]. */
SMB_API int smb_dense_grad_update(int dtype, const void* d_out, int64_t ld_d, int64_t m,
                                  const void* x, int64_t ld_x, int64_t k, int64_t n, void* w,
                                  int64_t ld_w, void* velocity, void* grad_out, int opt_kind,
                                  double mu, double eta, void* stream);

/* y = W x + bias for a dense layer of m <= 32 output rows (the ER-saturated
 * output layer; DenseLinearLayer.forward, nn.py:241-255 -- numpy BLAS there,
 * so tolerance parity): a deterministic split-K pass (each K slice summed in
 * ascending order with fused multiply-add, the slices then summed in
 * ascending order, then bias).  W [m, ld_w], x [k, ld_x], y [m, ld_y];
 * `workspace` holds smb_dense_forward_workspace_bytes(m, k, n) bytes. */
SMB_API size_t smb_dense_forward_workspace_bytes(int64_t m, int64_t k, int64_t n);
SMB_API int smb_dense_forward_small(int dtype, const void* w, int64_t ld_w, int64_t m, int64_t k,
                                    const void* x, int64_t ld_x, int64_t n, const void* bias,
                                    void* y, int64_t ld_y, void* workspace, void* stream);

/* y = max(x, 0) (nn.py:86-87) and out = d_out * (x_cached > 0) (nn.py:89-91). */
SMB_API int smb_relu(int dtype, const void* x, int64_t ld_x, int64_t m, int64_t n, void* y, int64_t ld_y,
             void* stream);
SMB_API int smb_relu_backward(int dtype, const void* d_out, int64_t ld_d, const void* x_cached,
                      int64_t ld_x, int64_t m, int64_t n, void* out, int64_t ld_out,
                      void* stream);

/* dst[f, j] = src[perm[base + j], f] for f < features, j < batch, where
 * base = (*step_counter) * batch when step_counter != NULL, else `base`.
 * `src` is the device-resident training set stored sample-major
 * [n_samples x features]; dst is feature-major [features x ld_dst].
 * Replaces the host gather Xtrain[:, batch] of sgd_train (train.py:390-396). */
SMB_API int smb_gather_columns(int dtype, const void* src, int64_t n_samples, int64_t features,
                       const int32_t* perm, const int32_t* step_counter, int64_t base,
                       int64_t batch, void* dst, int64_t ld_dst, void* stream);

/* The same gather for the batch `step_offset` steps ahead of the device step
 * counter: batch index ((*step_counter + step_offset) mod modulo) (modulo 0:
 * no wrap).  Lets the next batch be gathered while the current step runs. */
SMB_API int smb_gather_columns_ahead(int dtype, const void* src, int64_t n_samples,
                                     int64_t features, const int32_t* perm,
                                     const int32_t* step_counter, int32_t step_offset,
                                     int32_t modulo, int64_t batch, void* dst, int64_t ld_dst,
                                     void* stream);

/* *counter = (*counter + 1) % modulo  (device-side step index for CUDA-graph
 * replays of the training step). */
SMB_API int smb_step_counter_advance(int32_t* counter, int32_t modulo, void* stream);

/* ---- initialisation ------------------------------------------------------- */

/* out[p] = T(-a + 2a * u_{offset+p}) for p < count, where u_i = (x_i >> 11) * 2^-53
 * and x_i is the (i+1)-th 64-bit output of numpy's PCG64 (XSL-RR 128/64)
 * started at (state, inc).  Bit-identical to xavier_init
 * (sparsity.py:223-237: rng.uniform(-a, a, size).astype(dtype)) for the
 * Generator whose bit_generator.state is (state, inc); every thread jumps
 * ahead independently (O(log n) LCG jump). */
SMB_API int smb_xavier_pcg64(int dtype, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                     uint64_t inc_lo, uint64_t offset, int64_t count, double limit, void* out,
                     void* stream);

/* Scale-mode pattern sampler (the device counterpart of the reference's
 * sample_pattern, sparsity.py:183-216 -- same distribution, a uniform
 * size-nnz subset of the m x k grid, not the same numpy stream):
 * candidates pos_i = floor(Philox4x32-10(seed, counter (i, stream_id)) * m*k
 * / 2^64), the pattern = the first nnz distinct candidates (or, for
 * nnz > m*k/2, every position but the first m*k - nnz distinct ones), written
 * as CSR into row_ptr[m+1] / col_idx[nnz] (device, caller-owned).
 * Deterministic in (m, k, nnz, seed, stream_id).  Setup-time call: allocates
 * scratch and synchronises `stream`. */
SMB_API int smb_sample_pattern(int64_t m, int64_t k, int64_t nnz, uint64_t seed,
                               uint64_t stream_id, int32_t* row_ptr, int32_t* col_idx,
                               void* stream);
/* The sampler's 64-bit Philox draw i (host-callable, for checking). */
SMB_API uint64_t smb_philox_u64(uint64_t seed, uint64_t stream_id, uint64_t i);

/* Column-chain step (B200 addition, no single reference counterpart): the
 * batch-column-parallel middle of one training step in one cluster launch --
 * the forward products of layers 1..L-1 with bias / ReLU (nn.py:169-176,
 * 86-87), the softmax cross-entropy gradient and loss (nn.py:385-417,
 * train.py:399), and the input gradients d_{l-1} = (W_l^T d_l) * (a_{l-1} > 0)
 * for l = L-1..1 (nn.py:178-185, 89-91; train.py:216-220) -- with the same
 * arithmetic, bit for bit, as smb_spmm_p / smb_softmax_ce_step /
 * smb_spmm_t_csc.  Layer 0's forward product and all weight-side work
 * (SDDMM, updates, bias row sums) stay separate launches.
 *
 * smb_chain_plan_create: setup-time (synchronises the device); patterns[l]
 * of the L sparse layers (W_0 first), relu[l] = activation after layer l
 * (relu[L-1] must be 0), batch width n, leading dimension ld (multiple of 4).
 * The plan owns quad-padded copies of layers 1..L-1 (CSR and CSC order; a
 * pad is an exact no-op: value -0.0 times a zero operand row).  Returns
 * SMB_ERR_INVALID with a "chain: unsupported" message when the model does not
 * fit the kernel (more than 16 classes, operands over shared memory, ...);
 * the caller then runs the separate kernels.
 * smb_chain_refresh: re-derive the plan's padded value copies of layer
 * `layer` (1..L-1) from its values (CSR order); call after every change of
 * the values, stream-ordered before the next smb_chain_run.
 * smb_chain_plan_info: info4 = {CTAs per cluster, column groups, shared
 * memory bytes, layers}.
 * smb_chain_run: host arrays of L device pointers each (index = layer;
 * entry 0 of bias is not read): bias, acts[l] = a_l [m_l x ld] (acts[0] is
 * read, acts[1..] written), dys[l] = d_l (written); t the one-hot targets
 * [classes x ld_t]; loss_out (device float64, may be NULL) needs workspace
 * (smb_chain_workspace_bytes(n) bytes, zeroed once). */
typedef struct smb_chain_plan smb_chain_plan;
SMB_API int smb_chain_plan_create(int nlayers, const smb_pattern* const* patterns,
                                  const int* relu, int64_t n, int64_t ld, smb_chain_plan** out);
SMB_API int smb_chain_plan_destroy(smb_chain_plan* plan);
SMB_API int smb_chain_plan_info(const smb_chain_plan* plan, int64_t* info4);
/* Diagnostics: later runs of the plan record SM clock (clock64) stamps of their
 * phases (thread 0 of every CTA, 32 slots per CTA) into `stamps` (device,
 * uint64[CTAs x 32]); NULL turns it off. */
SMB_API int smb_chain_plan_profile(smb_chain_plan* plan, void* stamps);
SMB_API int smb_chain_refresh(const smb_chain_plan* plan, int layer, const void* values,
                              void* stream);
SMB_API size_t smb_chain_workspace_bytes(int64_t n);
SMB_API int smb_chain_run(const smb_chain_plan* plan, const void* const* bias, void* const* acts,
                          void* const* dys, const void* t, int64_t ld_t, double divisor,
                          double* loss_out, void* workspace, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPARSEMLP_B200_H */
