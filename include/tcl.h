/*
 * tcl.h -- C ABI of libtcl.so, the B200 (sm_100a) batched scorer of TCL's Mamba cost model.
 *
 * The operation (§3.2): an auto-tuning round proposes candidate tensor
 * programs; the cost model predicts each one's performance and the best K are selected for
 * measurement on the hardware.  Each candidate is a sequence of schedule-primitive feature
 * vectors, L x D with D = 22 on CPU targets (§5.1), padded at the tail to
 * `max_len`, plus its real length T.  The model is the Mamba-based cost
 * model of PAPER.md §5.2 (lines 429-451, Fig. 5): encoder (3 linears) -> norm -> Mamba
 * block(s) -> norm -> masked mean over the T real tokens -> decoder (3 linears) -> one score.
 * Higher score = better predicted performance.  The readings where the
 * paper is silent are listed in DESIGN.md §3 (R1-R20).
 *
 * Conventions
 *   - Every function returns tcl_status (0 = TCL_OK); nothing throws across the ABI.
 *   - "_dev" pointers are CUDA device pointers on the model's device; "_host" pointers are host
 *     memory (pinned or pageable).  The caller owns every pointer it passes in.
 *   - Compute calls enqueue work on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *     default stream) and return after host-side validation; outputs are valid once the stream
 *     has synchronised.  The *_host variants synchronise before returning.
 *   - Host-detectable errors return immediately (TCL_EINVAL, TCL_ESHAPE); a per-thread message
 *     is available from tcl_last_error().
 *   - Device-detected errors are sticky: a candidate length outside [1, max_len] produces a NaN
 *     score for that candidate, sets a device flag, and is reported as TCL_ELEN by
 *     tcl_sync_error() (or by the next *_host call).
 *   - Padded slots (t >= T_i) are ignored whatever they contain, including NaN/Inf.
 *   - A model is not thread-safe: one host thread (one stream) per model at a time.  Create one
 *     model per stream for concurrent scoring (weights are only ~4 MB).
 */
#ifndef TCL_H_
#define TCL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TCL_OK = 0,
    TCL_EINVAL = -1, /* null pointer, n < 0, k <= 0, n_passes < 1, dropout_p not in [0,1) ...  */
    TCL_ESHAPE = -2, /* inconsistent dims (e.g. enc_dims[2] != d_model), unsupported size      */
    TCL_ELEN = -3,   /* a candidate length outside [1, max_len] was seen on the device          */
    TCL_ECUDA = -4,  /* CUDA runtime/driver error                                               */
    TCL_ENOMEM = -5, /* device allocation failed                                                */
    TCL_ENCCL = -6,  /* NCCL error                                                              */
    TCL_ESTATE = -7  /* call out of order (e.g. tcl_topk_global before tcl_comm_init)           */
} tcl_status;

/* Arithmetic of the projections (in_proj, out_proj, encoder linears 2-3).
 *   FP32:      every GEMM in fp32 on the CUDA cores (FFMA); score within 1e-4*max(1,|ref|).
 *   BF16_PROJ: bf16 operands on the tcgen05 tensor cores with fp32 accumulation (TMEM); the
 *              activations between kernels are bf16 (features, encoder hidden states, LN
 *              outputs, x and SiLU(z), the gated scan output), SiLU / tanh / exp use the MUFU
 *              approximations; the residual stream, norm statistics, conv, scan state and head
 *              stay fp32; score within 2e-2*max(1,|ref|). */
typedef enum { TCL_PREC_FP32 = 0, TCL_PREC_BF16_PROJ = 1 } tcl_precision;

/* Discretisation of B ("a discretization method", reading R5):
 *   ZOH:     Abar = exp(Delta*A), Bbar = (exp(Delta*A) - 1)/A * B   (default)
 *   EULER_B: Abar = exp(Delta*A), Bbar = Delta*B                      (Mamba's reference code) */
typedef enum { TCL_DISC_ZOH = 0, TCL_DISC_EULER_B = 1 } tcl_disc;

/* Model dimensions.  Paper model ([n_layer,d_state,expand,d_conv] = [1,8,1,4], PAPER.md:586;
 * encoder 64,128,128 / decoder 64,32,1) is d_model = 128, enc_dims = {64,128,128},
 * dec_dims = {64,32,1}, dt_rank = 8, d_in = 22.
 * Supported by this build: d_in <= 32; d_model, enc_dims in {multiples of 32} <= 256;
 * d_inner = expand*d_model <= 512 (multiple of 32); d_state in {8, 16}; dt_rank <= 32;
 * d_conv <= 8; dec_dims[0..1] multiples of 4 <= 256, dec_dims[2] == 1; max_len <= 256.
 * BF16_PROJ additionally needs d_model, d_inner in {64, 128, 256}, enc_dims[0..1] <= 256,
 * d_conv == 4. */
typedef struct {
    int32_t d_in;        /* feature width D per token (22 on CPU targets)          */
    int32_t max_len;     /* L: padded sequence length of the feature tensor                       */
    int32_t d_model;     /* residual width                                                        */
    int32_t n_layer;     /* number of Mamba blocks (pre-norm residual, reading R3)                */
    int32_t d_state;     /* N: SSM state size per channel                          */
    int32_t d_conv;      /* depthwise causal conv width                            */
    int32_t expand;      /* d_inner = expand * d_model                              */
    int32_t dt_rank;     /* R: rank of the Delta projection (reading R7: ceil(d_model/16))         */
    int32_t enc_dims[3]; /* encoder output widths; enc_dims[2] == d_model                         */
    int32_t dec_dims[3]; /* decoder output widths; dec_dims[2] == 1                               */
    float ln_eps;        /* LayerNorm epsilon (reading R2: 1e-5, biased variance)                 */
    float dropout_p;     /* inverted-dropout rate, used only by tcl_score_mc (reading R17)        */
    int32_t precision;   /* tcl_precision                                                          */
    int32_t disc;        /* tcl_disc                                                               */
} tcl_dims;

typedef struct tcl_model tcl_model;

/* Number of fp32 values in the canonical weight blob for `dims` (0 if dims are invalid).
 * Blob order (fp32 little-endian, PyTorch [out][in] row-major):
 *   enc: W1[e1][d_in] b1[e1] W2[e2][e1] b2[e2] W3[dm][e2] b3[dm]
 *   per layer: ln_w[dm] ln_b[dm] W_in[2di][dm] (rows 0..di-1 -> x, di.. -> z)
 *              w_conv[di][d_conv] (tap d_conv-1 = current token) b_conv[di]
 *              W_x[R+2N][di] (rows: dt_r, then B, then C) W_dt[di][R] b_dt[di]
 *              A_log[di][N] (A = -exp(A_log), reading R8) Dv[di] W_out[dm][di]
 *   lnf_w[dm] lnf_b[dm]
 *   dec: W1[h1][dm] b1[h1] W2[h2][h1] b2[h2] W3[1][h2] b3[1]                               */
size_t tcl_weights_count(const tcl_dims* dims);

/* Validate dims, copy the weights to `cuda_device` (converting/pre-splitting for the chosen
 * precision and pre-scaling A by log2(e)), allocate the workspace lazily.  The host buffer may be
 * freed on return.  *out receives the model handle. */
tcl_status tcl_model_create(const float* weights_host, size_t n_floats, const tcl_dims* dims,
                            int cuda_device, tcl_model** out);
tcl_status tcl_model_destroy(tcl_model* model);

/* Optional pre-allocation of the workspace for batches of up to n_max candidates (no allocation
 * happens in later calls with n <= n_max, or, for tcl_score_mc, n <= n_max and n_passes <=
 * mc_passes_max: the MC passes run batched, n_passes x n virtual candidates per forward). */
tcl_status tcl_reserve(tcl_model* model, int64_t n_max, int32_t mc_passes_max);

/* Score n candidates.
 *   feats_dev  [n][max_len][d_in] fp32 row-major (padded slots ignored)
 *   lens_dev   [n] int32, each in [1, max_len]
 *   scores_dev [n] fp32 output.
 * n == 0 is a no-op.  Scores are batch-invariant: a candidate's score does not depend on n, on
 * its position in the batch, or on the other candidates (bit-identical). */
tcl_status tcl_score(tcl_model* model, const float* feats_dev, const int32_t* lens_dev, int64_t n,
                     float* scores_dev, void* stream);

/* MC-dropout uncertainty (north-star addition for the RDU sampler; the paper's
 * own uncertainty is Eqs. 2-3): n_passes forward passes with inverted dropout (rate
 * dims.dropout_p) after the SiLU of encoder layers 1-2 and decoder layers 1-2; mask bits from
 * Philox4x32-10 keyed by `seed`, counter (unit>>2, token<<2|site, pass, index_base+i) (reading
 * R17).  mean_dev/var_dev [n] fp32: mean and population variance (divide by n_passes). */
tcl_status tcl_score_mc(tcl_model* model, const float* feats_dev, const int32_t* lens_dev, int64_t n,
                        int32_t n_passes, uint64_t seed, int64_t index_base, float* mean_dev,
                        float* var_dev, void* stream);

/* Top-k ("selects the best K"): the k largest scores under the total order
 * (score desc, index asc), NaN treated as -inf.  idx_dev [k] int64 receives index_base + i,
 * topscore_dev [k] fp32 the scores.  If k > n, slots >= n get idx -1 and score -inf.
 * Requires index_base + n <= 2^32 - 1.  1 <= k <= 4096. */
tcl_status tcl_topk(tcl_model* model, const float* scores_dev, int64_t n, int32_t k,
                    int64_t index_base, int64_t* idx_dev, float* topscore_dev, void* stream);

/* Multi-GPU (one process per GPU).  Rank 0 calls tcl_comm_unique_id, broadcasts the 128 bytes
 * (e.g. through torch.distributed), every rank calls tcl_comm_init (collective). */
tcl_status tcl_comm_unique_id(uint8_t id_out[128]);
tcl_status tcl_comm_init(tcl_model* model, const uint8_t id[128], int32_t nranks, int32_t rank);

/* Global top-k across ranks: local top-k of this rank's n_local scores (indices index_base + i),
 * ncclAllGather of the k packed (score, index) keys over NVLink, merge -> the identical
 * (idx, score)[k] on every rank.  Collective: every rank must call it with the same k. */
tcl_status tcl_topk_global(tcl_model* model, const float* local_scores_dev, int64_t n_local,
                           int64_t index_base, int32_t k, int64_t* idx_dev, float* topscore_dev,
                           void* stream);

/* The two device halves of tcl_topk_global, for callers that run the exchange themselves (another
 * transport, or tests with several processes or virtual shards on one GPU):
 *   tcl_topk_local_keys: this shard's best k as packed keys (tcl_topk_key), sorted descending,
 *     0-padded when k > n_local -> keys_dev [k] (uint64, device).  n_local == 0 gives k zeros.
 *   tcl_topk_merge_keys: the best k of `count` gathered keys (any order, 0 = padding) decoded to
 *     (idx, score) [k]; slots beyond the real keys get idx -1, score -inf.
 * tcl_topk_global is exactly local_keys -> ncclAllGather -> merge_keys. */
tcl_status tcl_topk_local_keys(tcl_model* model, const float* local_scores_dev, int64_t n_local, int64_t index_base,
                               int32_t k, uint64_t* keys_dev, void* stream);
tcl_status tcl_topk_merge_keys(tcl_model* model, const uint64_t* keys_dev, int64_t count, int32_t k, int64_t* idx_dev,
                               float* topscore_dev, void* stream);

/* Host-side pieces of the multi-GPU protocol; no device needed.
 *   tcl_shard_range: rank's contiguous shard of n_global candidates: start = rank * ceil(n / nranks),
 *     count = min(n, start + ceil(n / nranks)) - start (clamped to 0); global index = start + i.
 *   tcl_topk_key: the packed (score desc, index asc) key the device kernels compute:
 *     orderable_u32(score) << 32 | (0xFFFFFFFF - global_index), NaN = -inf, -0 = +0. */
tcl_status tcl_shard_range(int64_t n_global, int32_t nranks, int32_t rank, int64_t* start, int64_t* count);
uint64_t tcl_topk_key(float score, int64_t global_index);

/* End-to-end host variant (the call a user without device buffers makes): copies feats/lens
 * host->device (pipelined in sub-chunks with the scoring on a second stream), scores, selects the
 * top-k (k > 0) and copies the results device->host.  Candidate i gets index index_base + i.  If
 * tcl_comm_init was called with nranks > 1 the top-k is the global one (tcl_topk_global, a
 * collective: every rank must call).  Synchronises; returns TCL_ELEN if a length was invalid.
 * idx_host/topscore_host may be NULL when k == 0. */
tcl_status tcl_score_host(tcl_model* model, const float* feats_host, const int32_t* lens_host,
                          int64_t n, int64_t index_base, float* scores_host, int32_t k,
                          int64_t* idx_host, float* topscore_host, void* stream);

/* KB + AC two-column model (§6, Eq. 7; reading R23):
 * the model TCL deploys on a target after continual knowledge distillation.  Both columns share
 * `dims` (canonical blobs of tcl_weights_count(dims) floats each).  The AC's layer i output is
 *   h_i = act(W_i h_{i-1} + alpha_i (.) U_i SiLU(V_i h^KB_{i-1} + c_i) + b_i)
 * at the three encoder linears, after every Mamba block (act = identity: added to the residual
 * stream) and at the two hidden decoder layers; h^KB_{i-1} is the KB's input to its own layer i
 * (the features for encoder layer 1).  Adapter blob (adapters_host, tcl_adapters_count floats),
 * per site in the order enc1, enc2, enc3, layer 0..n_layer-1, dec1, dec2:
 *   V [a][in], c [a], U [out][a], alpha [out]   (a = adapter_rank, 1..64).
 * The returned handle is used with tcl_score / tcl_score_mc / tcl_score_host / tcl_topk like a
 * one-column model; the score is the AC column's output; MC dropout applies to the AC column only
 * (the KB is frozen).  TCL_PREC_FP32 only (TCL_ESHAPE otherwise).  Host buffers are copied. */
size_t tcl_adapters_count(const tcl_dims* dims, int32_t adapter_rank);
tcl_status tcl_model_create_kbac(const float* kb_weights_host, const float* ac_weights_host, size_t n_floats,
                                 const float* adapters_host, size_t n_adapter_floats, int32_t adapter_rank,
                                 const tcl_dims* dims, int cuda_device, tcl_model** out);

/* Training (§5.3 Eq. 6, §7.1.3; reading R24), fp32 one-column
 * models only (TCL_ESHAPE otherwise).  tcl_train_init allocates the training state for batches of
 * up to n_max candidates (gradients, Adam moments (zero), saved activations) and sets Adam's lr,
 * beta1, beta2, eps (paper: Adam, lr 7e-4) and the LambdaRank scale sigma_rank (1).
 * tcl_train_step runs one step on a batch already on the device: feats/lens as tcl_score,
 * latency_dev [n] the measured latencies (> 0), group_offsets_dev [n_groups+1] int64 CSR groups
 * (one tuning task each; 1 <= members <= max_group, 2 <= max_group <= 4096; a single-member group
 * has no pairs and contributes 0; a group outside that range, or outside [0, n), contributes nothing and makes tcl_sync_error return TCL_ESHAPE; candidates outside every
 * group get a zero score gradient), the loss
 *   L = mean_g sum_{y_i > y_j} |G_i - G_j| |1/D_i - 1/D_j| log2(1 + e^{-sigma (s_i - s_j)}),
 *   y = min latency of the group / latency, G = (2^y - 1) / maxDCG, D = log2(1 + predicted rank)
 * (fp32) goes to loss_dev [1] (may be NULL), the gradient of every weight (canonical blob layout)
 * is computed by the backward pass, and apply_update != 0 applies one Adam step to the model's
 * weights (scoring calls then use the updated model).  No dropout during training.
 * tcl_train_read copies (synchronising) what = 0: weights [tcl_weights_count], 1: last gradients
 * [tcl_weights_count], 2: last dL/dscore [n], 3: last training scores [n] to host memory. */
tcl_status tcl_train_init(tcl_model* model, int64_t n_max, float lr, float beta1, float beta2, float eps,
                          float sigma_rank);
tcl_status tcl_train_step(tcl_model* model, const float* feats_dev, const int32_t* lens_dev, int64_t n,
                          const float* latency_dev, const int64_t* group_offsets_dev, int64_t n_groups,
                          int32_t max_group, int32_t apply_update, float* loss_dev, void* stream);
tcl_status tcl_train_read(tcl_model* model, int32_t what, float* host, int64_t count);

/* Top-k score, Eq. 12 (§7.1.2; reading R22):
 *   Top-k = sum_t minlat_t w_t / sum_t min{latency of task t's k best-predicted candidates} w_t
 * Tasks (one per subgraph of a model) are CSR segments: candidates task_offsets_dev[t] ..
 * task_offsets_dev[t+1]-1 (int64, [n_tasks+1], offsets into scores_dev / latency_dev) with
 * predicted scores (larger = better; ties: lower index first; NaN = -inf, R15), true latencies
 * (positive, finite) and a task weight task_weights_dev [n_tasks] (occurrence frequency).  k values
 * come from ks_host [n_k] (1 <= n_k <= 16, each k >= 1; k > task size clamps to the task size).
 * result_dev [3 * n_k] fp64 receives Top-k score[j], numerator[j], denominator[j].  Every task
 * must hold 1 .. max_task_len candidates (max_task_len <= 16384); a task outside that range makes
 * its terms NaN and tcl_sync_error return TCL_ESHAPE.  Integer ranking (exact); fp64 sums in a
 * fixed order (deterministic).  Device pointers; asynchronous on `stream`. */
tcl_status tcl_topk_score(tcl_model* model, const float* scores_dev, const float* latency_dev,
                          const int64_t* task_offsets_dev, const float* task_weights_dev, int64_t n_tasks,
                          int32_t max_task_len, const int32_t* ks_host, int32_t n_k, double* result_dev,
                          void* stream);

/* RDU acquisition, one selection round (Algorithm 1 lines 16-31,
 * Eqs. 1-3; reading R21 in DESIGN.md).  Given the model's predictions for the unlabeled pool
 * (pool_scores_dev [n_pool], with operator types pool_ops_dev [n_pool] in [0, n_ops)) and for the
 * current labeled set (labeled_scores_dev [n_labeled]), greedily picks up to budget_total pool
 * candidates by the total score t_s = f^ d_s + u_s (f^ min-max normalised over pool and labeled,
 * d_s = distance to the nearest labeled score, u_s = variance of the labeled set plus the
 * candidate), ties broken by higher f^ then lower index, skipping operator types whose budget
 * budget_total * count(op) / n_pool is exhausted; each pick joins the labeled set before the next.
 * selected_idx_dev [budget_total] receives the picks in order, n_selected_dev [1] their number.
 * Requires 1 <= n_ops <= 256 and n_pool <= 4096 * (SM count).  Non-finite scores take no part
 * (never selected, not in the labeled set nor the min/max; their op still counts in the budget
 * shares); pool entries with op outside [0, n_ops) are never selected.  Scores are evaluated in
 * fp32 with a fixed operation order (bit-reproducible, identical picks to oracle/).  Device
 * pointers; no allocation after the first call per model; asynchronous on `stream`. */
tcl_status tcl_rdu_select(tcl_model* model, const float* pool_scores_dev, const int32_t* pool_ops_dev,
                          int64_t n_pool, const float* labeled_scores_dev, int64_t n_labeled, int32_t n_ops,
                          int32_t budget_total, int64_t* selected_idx_dev, int32_t* n_selected_dev,
                          void* stream);

/* Per-model options.
 *   TCL_OPT_GRAPHS (default 1): replay the launch sequence of a repeated call (same pointers,
 *     sizes, seeds and stream-independent arguments: tcl_score, tcl_score_mc, tcl_topk,
 *     tcl_train_step) from a CUDA graph captured on its second occurrence; 0 launches every
 *     kernel directly.  Results are bit-identical either way (tested); graphs only remove the
 *     host launch cost and the inter-kernel gaps of the small, launch-bound configurations.
 *   TCL_OPT_SCAN (default 0 = auto): how the fp32 path runs the mixer's recurrence.  1 = sequential
 *     (one thread per (candidate-range, channel) walking the tokens: work-efficient);
 *     2 = chunked (one CTA per candidate, warp-shuffle chunked scan ACROSS L with the associative
 *     operator (a1, b1) o (a2, b2) = (a1 a2, a2 b1 + b2), lanes = tokens; for max_len <= 32 and
 *     d_inner <= 128).  The choice is per model, never per n, so scores stay batch-invariant;
 *     auto = sequential (measured faster at every BASELINE configuration: the chunked scan does
 *     ~4-8x the instructions for 32x the parallelism).  The two modes round differently (both
 *     within the fp32 parity bound).
 * Returns TCL_EINVAL for an unknown option or value. */
typedef enum { TCL_OPT_GRAPHS = 1, TCL_OPT_SCAN = 2 } tcl_option;
tcl_status tcl_set_option(tcl_model* model, int32_t option, int64_t value);

/* Synchronise `stream`, then return (and clear) the sticky device error of the model. */
tcl_status tcl_sync_error(tcl_model* model, void* stream);

/* Number of kernels this model launched so far (instrumentation for bench.py). */
int64_t tcl_launch_count(const tcl_model* model);

/* Per-stage device-time instrumentation: when enabled, every launch is bracketed by CUDA events
 * recorded on the launching stream.  tcl_profile_read synchronises the device, adds the elapsed
 * times per stage kind into ms_out[TCL_PROF_NKINDS] and launch counts into launches_out, and
 * clears the record list if reset != 0. */
typedef enum {
    TCL_PROF_PACK = 0, TCL_PROF_ENCODER, TCL_PROF_LAYERNORM, TCL_PROF_IN_PROJ, TCL_PROF_CONV,
    TCL_PROF_X_PROJ, TCL_PROF_DT_PROJ, TCL_PROF_SCAN, TCL_PROF_OUT_PROJ, TCL_PROF_HEAD,
    TCL_PROF_TOPK, TCL_PROF_MIXER, TCL_PROF_ALLGATHER, TCL_PROF_MC, TCL_PROF_LATERAL, TCL_PROF_XDT,
    TCL_PROF_NKINDS
} tcl_prof_kind;
tcl_status tcl_profile_enable(tcl_model* model, int enable);
tcl_status tcl_profile_read(tcl_model* model, double* ms_out, int64_t* launches_out, int reset);
const char* tcl_profile_name(int kind);

/* Debugging aid (per-stage parity tests): copy the current contents of a workspace buffer, as
 * fp32, to host memory.  name: "H" (residual stream [P][d_model]), "A" (LayerNorm output
 * [P][d_model]), "XZ" (in_proj output [P][2 d_inner]; bf16 path: [x | SiLU(z)]), "G" (gated
 * scan output [P][d_inner]), "U" (conv + SiLU output [P][d_inner]), "DELTA" ([P][d_inner]), "BC"
 * (bf16 path: x_proj's B and C [P][2 d_state]).  Rows are the packed tokens of the
 * last chunk scored; buffers hold the values of the LAST kernel that wrote them (bf16 path with
 * d_model >= 128: the last layer writes LN_f(H) into "A" and does not write "H").  Synchronises. */
tcl_status tcl_debug_read(tcl_model* model, const char* name, float* host_out, int64_t rows, int64_t cols);

/* Thread-local message describing the last error returned on this thread ("" if none). */
const char* tcl_last_error(void);

/* Build information (compile target, version). */
const char* tcl_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* TCL_H_ */
