/*
 * ppmoe_capi.h — C-ABI of the B200-native PPMoE (Pipeline MoE, arXiv 2304.11414)
 * MoE-layer hot path.  Built as paper_2304_11414_b200/lib/libppmoe.so.
 *
 * The reference (`moesim` 0.1.0, pure Python/numpy) has no FFI for this path; its
 * boundary is the Python API in pkg/src/moesim/moe.py.  Each entry point below
 * replaces one step of that API and cites the reference code it reproduces.
 * The Python package paper_2304_11414_b200 binds these symbols with ctypes
 * and mirrors the reference's Python signatures on top.
 *
 * Conventions
 *  - All pointers are DEVICE pointers owned by the caller (PyTorch caching
 *    allocator).  The library never allocates or frees device memory (except the
 *    explicit ppmoe_ipc_* helpers) and never synchronises the host: every call only
 *    enqueues kernels / async copies on `stream` (a cudaStream_t passed as void*).
 *    Its only state: the thread-local GEMM SM budget (ppmoe_set_gemm_sm_budget) and
 *    GEMM mode, the thread-local error string, and one 4-byte module-scope device
 *    word per device (the grouped GEMM's wave-synchronisation counter, reset on the
 *    launch stream before each long-K GEMM; PPMOE_KSYNC=0 disables it).  Long-K
 *    GEMMs of one device must therefore be stream-ordered (they are, in this path).
 *  - Return value 0 = success; negative = error, message via ppmoe_last_error()
 *    (thread-local).  -1/-3 map to ValueError, -2/-4 to RuntimeError.
 *  - dtype: 0 = bf16 (activations/expert weights bf16, fp32 accumulation),
 *           1 = fp32 (reference-precision mode, CUDA-core GEMM).
 *    The gate weight Wg and all routing scores/weights are always fp32; routing
 *    logits and softmax are evaluated in fp64.
 *  - Layouts are row-major.  Token-major activations [N x H] (moe.py: b*s rows).
 *    Gate weight Wg [H x E] (GateParams.wg, moe.py:30-53).  Expert weights of the
 *    El local experts are stacked: up [El x H x F], down [El x F x H],
 *    bias_up [El x F], bias_down [El x H] (ExpertFfn, moe.py:80-110).
 *  - Dispatch plan ("padded segments"): the sorted-pair buffer holds, for every
 *    expert e, its kept token rows in ascending token id starting at seg[e]; each
 *    segment is padded to a multiple of 128 rows with tok = -1.  A rank owning
 *    experts [r*El, (r+1)*El) passes `seg + r*El` (El+1 entries) to the expert
 *    calls; local row = seg[g] - seg[0] + m.  rows_cap bounds local rows.
 */
#ifndef PPMOE_CAPI_H
#define PPMOE_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Library identity / errors ------------------------------------------------ */
int ppmoe_version(void);
const char* ppmoe_last_error(void);
/* Number of SMs of the current device (grid sizing of the persistent kernels). */
int ppmoe_num_sms(void);
/* Persistent-GEMM grid budget for the calling host thread: 0 = one CTA per SM (default);
 * n > 0 = at most n CTAs, leaving SMs free for a collective that runs concurrently. */
int ppmoe_set_gemm_sm_budget(int sms);
/* Grouped-GEMM kernel selection for the calling host thread: 0 = automatic (CTA pair,
 * 1-CTA for long-K token GEMMs; PPMOE_GEMM env overrides), 1 = 1-CTA, 2 = CTA pair. */
int ppmoe_set_gemm_mode(int mode);
/* Diagnostic counter: kernels this library has launched in this process (all threads). */
unsigned long long ppmoe_kernel_launches(void);

/* Routing: gate GEMV + fp64 softmax + top-k + aux loss ---------------------
 * Replaces gate_top1 (moe.py:196-208), aux_loss (moe.py:211-223) and the
 * route_override path (moe.py:199-205); top-k > 1 extends the reference
 * (repeated argmax, lowest expert id wins ties, raw softmax weights, aux-loss
 * fractions from the top-1 choice).
 *   X        [N x H] dtype
 *   Wg       [H x E] fp32
 *   override [N x K] int32 or NULL; ids already validated to lie in [0, E)
 *   idx      [N x K] int32   out: chosen experts per token (slot-major per token)
 *   w        [N x K] fp32    out: softmax score of each chosen expert
 *   scores   [N x E] fp32    out: full softmax scores
 *   l_aux    [2] fp64        out: {l_aux, sum_e frac_e (== 1)}
 *   counts_top1 [E] int32    out: tokens whose slot-0 expert is e (or NULL)
 *   score_sums  [E] fp64     out: sum over the N tokens of each expert's score (or NULL);
 *                            with counts_top1 it lets token slices be combined across ranks
 *   ws       workspace of ppmoe_route_workspace_bytes(N, E, K) bytes
 */
size_t ppmoe_route_workspace_bytes(int N, int E, int K);
int ppmoe_route(const void* X, int dtype, const float* Wg, int N, int H, int E, int K, const int* route_override,
                int* idx, float* w, float* scores, double* l_aux, int* counts_top1, double* score_sums, void* ws,
                size_t ws_bytes, void* stream);

/* Dispatch plan with capacity: replaces build_dispatch_plan (moe.py:226-235)
 * and _capacity_mask (moe.py:345-360).  Stable counting sort of the (token,
 * slot) pairs by expert; capacity keeps the first `capacity` pairs per expert in
 * (slot, token id) priority order (== ascending global token id at K=1).
 *   idx         [N x K] expert ids in [0, E) (validated by the caller)
 *   w           [N x K] gate weights or NULL (then w_sorted may be NULL)
 *   capacity    max kept pairs per expert (INT32_MAX = unlimited)
 *   rank_offset [K x E] or NULL: pairs of higher priority held by other ranks (the
 *               all-to-all comparator's global token order, moe.py:352-359)
 *   counts      [E]    out: routed pairs per expert before capacity
 *   kept        [E]    out: kept pairs per expert
 *   seg         [E+1]  out: padded segment starts (multiples of 128)
 *   tok_sorted  [rows_cap_global] out: token id per sorted row (-1 = padding)
 *   w_sorted    [rows_cap_global] out: gate weight per sorted row
 *   pair_pos    [N x K] out: sorted row of every pair, -1 if dropped
 *   rows_cap_global >= N*K + 128*E
 */
/* Sliced routing (T ranks each routed N/T tokens with ppmoe_route, score_sums + counts_top1
 * written into their record of stats): stats [T x 4E] int32 words per rank = E fp64 score
 * sums, E int32 top-1 counts, E words of padding (16-byte records), all-gathered.  Sums the records in rank order and writes
 * l_aux [2] (value, sum of fractions) and the global counts_top1 [E] (moe.py:211-223).   */
/* Workspace of ppmoe_route including the tensor-core router's prepared Wg pieces (needs H):
 * a workspace of at least this size enables that router (bf16, E <= 16, H % 128 == 0, no
 * route override); ppmoe_route_workspace_bytes(N, E, K) alone selects the fp64 routers.   */
size_t ppmoe_route_workspace_bytes_h(int N, int H, int E, int K);
int ppmoe_route_combine_stats(const int* stats, int T, int N, int E, double* l_aux, int* counts_top1, void* stream);
size_t ppmoe_dispatch_workspace_bytes(int N, int E, int K);
int ppmoe_dispatch_plan(const int* idx, const float* w, int N, int E, int K, int capacity, const int* rank_offset,
                        int* counts, int* kept, int* seg, int* tok_sorted, float* w_sorted, int* pair_pos,
                        int rows_cap_global, void* ws, size_t ws_bytes, void* stream);

/* Index-slice gather ("tensor index slicing"; index_select,
 * tensor.py:226-241): Xs[row] = X[tok_sorted[seg[0]+row]] for the local rows,
 * zero for padding rows, staged through shared memory with bulk-TMA copies.
 * Also emits the local token id / gate weight per row.                       */
int ppmoe_gather(const void* X, int dtype, int N, int H, const int* seg, int El, const int* tok_sorted,
                 const float* w_sorted, int rows_cap, void* Xs, int* tok_local, float* w_local, void* stream);

/* Token-chunk row ranges: for chunk c of C (tokens [c*N/C, (c+1)*N/C)) and local
 * expert g, row_lo/row_hi[c*El+g] = local rows of that expert's segment holding the
 * chunk's tokens (segments are ascending in token id).  kept = plan kept counts of the
 * El local experts; row_lo/row_hi hold (C+1)*El entries, the last El being each segment's
 * padding rows.  Used to pipeline the forward combine all-reduce by token chunk.        */
int ppmoe_chunk_rows(const int* tok_local, const int* seg, const int* kept, int El, int N, int C, int* row_lo,
                     int* row_hi, void* stream);

/* Expert FFN forward, first GEMM: a = Xs*up_g + bias_up, Act = GeLU(a), and
 * GeluGrad = GeLU'(a) saved for the backward (ExpertFfn.forward, moe.py:100-104;
 * gelu backward tensor.py:204-207).  bias_up may be NULL.  row_lo/row_hi [El]
 * (both NULL = whole segments) restrict each expert to a row range.           */
int ppmoe_expert_fc1_fwd(int dtype, const void* Xs, const void* up, const void* bias_up, const int* seg, int El,
                         int H, int F, int rows_cap, const int* row_lo, const int* row_hi, void* GeluGrad, void* Act,
                         void* stream);

/* Expert FFN forward, second GEMM fused with the gate-weighted combine:
 * Y = Dropout(Act*down_g + bias_down) (stored, pre-scale), out_acc[tok] += w*Y
 * (moe.py:104-107, scale_rows tensor.py:184-196, index_assign 244-272, dropout
 * tensor.py:315-330 drawn from the reference's Philox stream: drop_stream = the
 * descriptor of ppmoe_dropout_stream, required when dropout_p > 0, else may be NULL).
 * out_acc [N x H] fp32 must be zeroed by the caller; NULL = store Y only (for ppmoe_combine).
 * Y2 (optional) receives a second copy of Y (the peer-visible rows of ppmoe_nvl_owner_gather). */
int ppmoe_expert_fc2_fwd(int dtype, const void* Act, const void* down, const void* bias_down, const int* seg,
                         int El, int H, int F, int rows_cap, const int* row_lo, const int* row_hi,
                         const int* tok_local, const float* w_local, int weight_scaling, float dropout_p,
                         const unsigned long long* drop_stream, void* Y, void* Y2, float* out_acc, void* stream);

/* Gather-combine over this rank's pairs, in slot order (deterministic):
 *   out[t] = sum_s w[t,s] * R[pair_pos[t,s] - seg[0]]  (+ dL[t,:] . Wg^T when dL != NULL)
 * summing the slots whose sorted row lies in this rank's rows [seg[0], seg[El]); w NULL = 1.
 * Forward: R = the fc2 outputs Y (ppmoe_expert_fc2_fwd with out_acc NULL), the top-k
 * combine (scale_rows + index_assign, tensor.py:184-272).  The optional gate term takes
 * dL [N x E] fp32 and Wg [H x E] fp32 (see ppmoe_input_grads).  out [N x H] in dtype.  */
int ppmoe_combine(int dtype, const void* R, const int* seg, int El, const int* pair_pos, const float* w, int N, int K,
                  int H, const float* dL, const float* Wg, int E, void* out, void* stream);

/* The layer's input gradients in one pass over the tokens (index_select + gate matmul
 * backward, tensor.py:134-138, 235-239):
 *   dX[t] = sum_s dXs[pair_pos[t,s] - seg[0]] + dL[t,:] . Wg^T     (dtype; NULL = skip)
 *   dWg   = X^T dL                                                   (fp32 [H x E]; NULL = skip)
 * dXs = the per-row dX of ppmoe_expert_fc1_dgrad; pair sums in slot order, dWg partials
 * reduced in a fixed order (deterministic).  ws of ppmoe_input_grads_workspace_bytes.  */
size_t ppmoe_input_grads_workspace_bytes(int dtype, int N, int H, int E);
int ppmoe_input_grads(int dtype, const void* dXs, const int* seg, int El, const int* pair_pos, int N, int K, int H,
                      const void* X, const float* dL, const float* Wg, int E, void* dX, float* dWg, void* ws,
                      size_t ws_bytes, void* stream);

/* out = out_acc cast to dtype (the replicated [N x H] layer output before or
 * after the TP all-reduce, collectives.py:135-153).                         */
int ppmoe_cast_out(const float* acc, int n, void* out, int dtype, void* stream);

/* Dropout stream descriptor (device, 3 + El uint64) of the reference's tensor.dropout draws
 * (tensor.py:315-330, moesim Rng = numpy Philox4x64-10 keyed (key0, key1)): the experts
 * draw one [kept rows x H] uniform block each in ascending id starting at draw first_draw
 * of the stream; this rank's experts are [e0, e0+El); kept [E] device counts of every
 * expert (kept pairs, i.e. rows).  threshold = ceil(p * 2^53): draw w is kept iff
 * (w >> 11) >= threshold, i.e. its uniform (w >> 11) * 2^-53 >= p.                    */
int ppmoe_dropout_stream(const int* kept, int E, int e0, int El, int H, unsigned long long key0,
                         unsigned long long key1, unsigned long long threshold, unsigned long long first_draw,
                         unsigned long long* desc, void* stream);

/* Backward of scale_rows + index_assign + dropout (tensor.py:190-194, 264-270, 326-328):
 * dY[row] = w*dOut[tok] (times the forward's dropout mask / (1-p)),
 * dw[row] = <dOut[tok], Y[row]>; zero for padding.  dy_colsum_part (optional, bf16 and
 * H % 256 == 0): [rows/32 x H] fp32 per-32-row-block column sums of dY, consumed by
 * ppmoe_expert_fc2_wgrad for the bias_down gradient.                        */
int ppmoe_bwd_dy(int dtype, const void* dOut, const void* Y, const int* seg, int El, int H, int rows_cap,
                 const int* tok_local, const float* w_local, int weight_scaling, float dropout_p,
                 const unsigned long long* drop_stream, void* dY, float* dw, float* dy_colsum_part, void* stream);

/* dH = (dY*down_g^T) .* GeluGrad   (matmul/gelu backward, tensor.py:134-138, 204-207).
 * dh_colsum_part (optional, bf16 path): [rows/32 x F] fp32 column sums of dH per 32-row
 * block, produced in the epilogue for ppmoe_expert_fc1_wgrad's bias_up gradient.      */
int ppmoe_expert_fc2_dgrad(int dtype, const void* dY, const void* down, const void* GeluGrad, const int* seg, int El,
                           int H, int F, int rows_cap, void* dH, float* dh_colsum_part, void* stream);

/* dDown_g = Act_g^T * dY_g  [El x F x H]; dbias_down_g = colsum(dY_g) (may be NULL), reduced
 * from dy_colsum_part when given (else by a pass over dY).                              */
int ppmoe_expert_fc2_wgrad(int dtype, const void* Act, const void* dY, const int* seg, int El, int H, int F,
                           int rows_cap, void* dDown, void* dBiasDown, const float* dy_colsum_part, void* stream);

/* dH*up_g^T per local row: scatter-added into dx_acc[tok] (fp32, index_select backward
 * tensor.py:235-239) or stored per row into dXs [rows x H] (dtype) for the deterministic
 * gather-combine in ppmoe_gate_grads.  Exactly one of dx_acc / dXs.                   */
int ppmoe_expert_fc1_dgrad(int dtype, const void* dH, const void* up, const int* seg, int El, int H, int F,
                           int rows_cap, const int* tok_local, float* dx_acc, void* dXs, void* stream);

/* dUp_g = Xs_g^T * dH_g  [El x H x F]; dbias_up_g = colsum(dH_g) (may be NULL), reduced from
 * dh_colsum_part when given.                                                            */
int ppmoe_expert_fc1_wgrad(int dtype, const void* Xs, const void* dH, const int* seg, int El, int H, int F,
                           int rows_cap, void* dUp, void* dBiasUp, const float* dh_colsum_part, void* stream);

/* Gate backward (gather_rowwise, softmax and aux_loss backward, tensor.py:218-221,
 * 287-291, moe.py:211-223): dL[t,e] = s*(dS - sum(dS*s)) with
 * dS[t, idx[t,k]] += dw[pair] for pairs in sorted rows [seg[0], seg[El]) and
 * dS[t,e] += aux_grad[0] * E/N * frac_e; aux_grad is a device scalar (the upstream
 * gradient of l_aux) or NULL — pass it on exactly one rank of the TP group.   */
int ppmoe_gate_bwd(const float* scores, const int* idx, const int* pair_pos, const float* dw, const int* seg, int El,
                   const int* counts_top1, int N, int E, int K, const float* aux_grad, float* dL, void* stream);

/* dX = dx_acc + dL*Wg^T (cast to dtype) and the per-chunk partials of
 * dWg = X^T*dL, reduced deterministically into dWg [H x E] fp32.  Either of
 * dX / dWg may be NULL (with dXs rows, dX comes from ppmoe_combine instead).
 * ws of ppmoe_gate_grad_workspace_bytes(N,H,E).                            */
size_t ppmoe_gate_grad_workspace_bytes(int N, int H, int E);
int ppmoe_gate_grads(const float* dx_acc, const void* X, int dtype, const float* dL, const float* Wg, int N, int H,
                     int E, void* dX, float* dWg, void* ws, size_t ws_bytes, void* stream);

/* All-to-all expert-parallel comparator (dpmoe_forward, moe.py:363-469) ------------ */
/* Compact expert-major layout of this rank's kept pairs (the dispatch send buffer order,
 * moe.py:405-414): cstart [E+1], tok_c/w_c per compact row, pair_pos_c [N*K] = compact
 * row of every pair (-1 dropped).  w_sorted/w_c may be NULL.                          */
int ppmoe_a2a_compact(const int* tok_sorted, const float* w_sorted, const int* seg, const int* kept, int E,
                      const int* idx, const int* pair_pos, int NK, int* cstart, int* tok_c, float* w_c,
                      int* pair_pos_c, void* stream);
/* Owner-side regrouping of received rows (source-major) into expert-major padded
 * segments with sources in rank order: seg_out [El+1], map[owner row] = receive row
 * (-1 padding).  recv_counts [T x El] rows per (source, local expert).             */
int ppmoe_a2a_owner_layout(const int* recv_counts, int T, int El, int rows_cap, int* seg_out, int* map,
                           void* stream);
/* dst[map[o]] = src[o] for o < rows with map[o] >= 0 (rows of H values in dtype, 16-byte
 * multiples): the owner's expert-major rows back to all-to-all receive order.        */
int ppmoe_a2a_permute_rows(const void* src, int dtype, int H, int rows, const int* map, void* dst, void* stream);
/* dst[tok[r]] += w[r]*src[r] (fp32 dst, src in dtype) for r < nrows[0] (device scalar),
 * tok < 0 skipped, w NULL = 1 (index_assign back to token order, moe.py:461-467).   */
int ppmoe_scatter_rows(const void* src, int dtype, int H, const int* nrows, const int* tok, const float* w, float* dst,
                       void* stream);

/* Tensor-parallel exchange over NVLink peer memory (replaces the [N x H] all-reduces of
 * reduce_from_tensor_parallel_region moe.py:307 and tp_region backward
 * collectives.py:205-228, whose partials are k/T-sparse by token) ------------------ */
/* CUDA IPC: device buffer + handle (ppmoe_ipc_handle_bytes() bytes), open a peer's handle. */
size_t ppmoe_ipc_handle_bytes(void);
int ppmoe_ipc_alloc(size_t bytes, void** ptr, void* handle);
int ppmoe_ipc_open(const void* handle, void** ptr);
int ppmoe_ipc_close(void* ptr);
int ppmoe_ipc_free(void* ptr);
/* Pointer sets (pads, rows, push, srcs) are HOST arrays of T device pointers (passed to
 * the kernels by value; T <= 8), entry q = rank q's buffer as mapped in this process.
 * Barrier of T ranks on channel ch (0 <= ch < 16): writes `epoch` (release, system scope) into every
 * peer's signal pad (ppmoe_nvl_pad_bytes() each),
 * then waits until all T flags of this rank's pad reach `epoch`.  A spin longer than
 * timeout_cycles stores 1 to *err (plain store + system fence, so err may be pinned
 * host memory mapped into the device: the host reads it without a sync) and returns
 * instead of hanging; the caller must treat the exchange as failed.                  */
size_t ppmoe_nvl_pad_bytes(void);
int ppmoe_nvl_barrier(void* const* pads, int T, int rank, int ch, unsigned int epoch, int* err,
                      long long timeout_cycles, void* stream);
/* Owner gather for this rank's tokens [t0, t1) = [rank*N/T, (rank+1)*N/T):
 *   out[t] = sum_s w[t,s] * rows[q][pair_pos[t,s] - seg[q*El]]   q = idx[t,s] / El
 *            (+ dl[t - t0, :] . Wg^T when dl != NULL)
 * in slot order; rows = the T ranks' row buffers (bf16 [rows x H]; Y forward, per-row dX
 * backward), dl = this rank's summed dL rows [t1-t0 x E] fp32 (from ppmoe_nvl_sum_rows;
 * E <= 128).  Writes the owned rows of out (local [N x H]) and either of out_sym (this
 * rank's peer-visible copy, push NULL: peers pull; may be NULL) or of every rank's
 * exchange buffer push[q] (P2P stores, then a local pull).  sym_mc = 1: out_sym is an
 * NVLS multicast address (multimem.st: one store reaches every rank's buffer, then a
 * local copy).  With T = 1 it is the single-GPU top-k combine / input-gradient gather.  */
int ppmoe_nvl_owner_gather(const void* const* rows, const int* seg, int El, const int* idx, const int* pair_pos,
                           const float* w, int N, int K, int H, int T, int rank, const float* dl, const float* Wg,
                           int E, void* out, void* out_sym, void* const* push, int sym_mc, void* stream);
/* out [t1-t0 x C] = sum over q (rank order) of srcs[q] rows [t0, t1) (fp32 [N x C]): the
 * owned rows of the ranks' partial gate-logit gradients.                               */
int ppmoe_nvl_sum_rows(const void* const* srcs, int T, int rank, int N, int C, float* out, void* stream);
/* out [count] = sum over q (rank order) of srcs[q][0, count) (fp32): the all-reduce of the
 * gate-weight gradient over the tensor group (replaces collectives.py:135-153 all_reduce_sum
 * in sync_gate_gradients, moe.py:311-313), called after a barrier that published srcs.    */
int ppmoe_nvl_sum_all(const void* const* srcs, int T, int count, float* out, void* stream);
/* Sliced routing over peer memory (the all-gather of moe.py:288-291's replicated gate
 * outputs): recs = the T ranks' records of their nr-token slices, 32-bit words
 * [stats 4E (ppmoe_route's score_sums fp64 | counts_top1 | pad) | idx nr*K | w nr*K |
 * scores nr*E]; writes the full idx [T*nr x K], w, scores [T*nr x E] and stats [T x 4E]
 * (the input of ppmoe_route_combine_stats).  Call after a barrier that published recs. */
int ppmoe_nvl_route_gather(const void* const* recs, int T, int nr, int K, int E, int* idx, float* w, float* scores,
                           int* stats, void* stream);
/* Fused forward variant: ppmoe_expert_fc2_fwd_owner's epilogue scatter-adds w*Y of every
 * row straight into the fp32 accumulator of the rank that owns the row's token (owner_acc
 * = DEVICE array of T peer pointers, each [owner_rows x H], token t owned by t / owner_rows,
 * red.global.add over NVLink while the GEMM runs; k <= 2 keeps it order-independent).
 * After a barrier, ppmoe_nvl_cast_owned turns this rank's accumulator rows into bf16
 * (out rows and the exchange copy) and zeroes them for the next pass.               */
/* Owner-slot variant (owner_slots instead of owner_acc): w*Y is stored in bf16 with plain
 * P2P stores into slot s of the owner's [owner_rows x K x H] buffer (s = the pair's top-k
 * slot from pair_pos [N x K], K <= 2), and ppmoe_nvl_sum_slots sums the valid slots.   */
int ppmoe_expert_fc2_fwd_owner(int dtype, const void* Act, const void* down, const void* bias_down, const int* seg,
                               int El, int H, int F, int rows_cap, const int* tok_local, const float* w_local,
                               int weight_scaling, float dropout_p, const unsigned long long* drop_stream, void* Y,
                               float* const* owner_acc, void* const* owner_slots, const int* pair_pos, int K,
                               int owner_rows, void* stream);
int ppmoe_nvl_cast_owned(float* acc, int rows, int H, void* out_rows, void* xch_rows, void* stream);
int ppmoe_nvl_sum_slots(const void* slots, int rows, int K, int H, int t0, const int* pair_pos, void* out_rows,
                        void* xch_rows, void* stream);
/* All-gather by pull: out rows of every other owner q's block from srcs[q] (its out_sym),
 * by SM loads (_blocks) or by copy-engine transfers, one per peer block (_blocks_ce).  */
int ppmoe_nvl_pull_blocks(const void* const* srcs, int T, int rank, int N, int H, void* out, void* stream);
int ppmoe_nvl_pull_blocks_ce(const void* const* srcs, int T, int rank, int N, int H, void* out, void* stream);
/* Copy-engine pull of the blocks of owners [q_lo, q_hi) only (token-chunked exchange). */
int ppmoe_nvl_pull_range_ce(const void* const* srcs, int T, int rank, int N, int H, int q_lo, int q_hi, void* out,
                            void* stream);

/* Self-test entry: plain grouped GEMM D_g = A_g * B_g through the tcgen05 path
 * (use_tc=1 default, 2 1-CTA, 3 CTA pair 256x256, 4 CTA pair 256x512, 5 CTA pair 256x128) or the
 * CUDA-core path (use_tc=0).  mode 0: A [rows x K] K-major
 * per segment, B [G*K x N] MN-major, D [rows x N]; mode 1: K from segments,
 * A [rows x M] MN-major, B [rows x N] MN-major, D [G x M x N];
 * mode 2: A K-major segments, B [G*N x K] K-major, D [rows x N].           */
/* Thread-local tile choice of the long-K token GEMMs (fc2 fwd, fc1 dgrad): 1 = the narrow
 * 256 x 128 CTA-pair tile (twice the tiles: a fuller last wave when few expert rows sit on
 * a GPU), 0 = the 256 x 256 tile, -1 = PPMOE_NARROW / default (256 x 256).             */
int ppmoe_set_gemm_narrow(int narrow);
int ppmoe_gemm_selftest(int mode, int use_tc, int dtype, const void* A, const void* B, const int* seg, int G, int M,
                        int N, int K, int rows_cap, void* D, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PPMOE_CAPI_H */
