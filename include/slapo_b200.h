/*
 * slapo_b200.h — C ABI of the B200-native executor for Slapo's scheduled
 * forward+backward step (libslapo_b200.so).
 *
 * Conventions: every function returns 0 on success, 1 on error, 2 on a
 * schedule rule violation (R1..R5, proj/include/slapo/schedule.hpp:27-35);
 * sb_last_error() returns the thread-local message. Never throws. Handles are
 * opaque. Host buffers are plain double arrays (the reference's TensorValue
 * payload); device entry points take device pointers, sizes and an explicit
 * cudaStream_t (passed as void*) and only enqueue.
 *
 * Each entry point names the reference interface it replaces.
 */
#ifndef SLAPO_B200_H
#define SLAPO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sb_model sb_model;       /* slapo::ModuleDef                    */
typedef struct sb_schedule sb_schedule; /* slapo::Schedule (a path handle)     */
typedef struct sb_pipeline sb_pipeline; /* slapo::PipelineStagePlan             */
typedef struct sb_executor sb_executor; /* slapo::Executor                     */

const char* sb_last_error(void);
int sb_version(void);

/* ---------------------------------------------------------------- models */
/* toy_bert / tp_two_linear / fig3c_exact / ffn_stack — proj/tests/support/fixtures.hpp:21-38 */
int sb_model_toy_bert(int layers, int64_t hidden, int64_t heads, int64_t vocab, int64_t batch, int64_t seq,
                      double dropout_p, sb_model** out);
int sb_model_tp_two_linear(int64_t hidden, int64_t inner, int64_t batch, sb_model** out);
/* f2: T5-style encoder-decoder (BASELINE.json configs[4]): pre-LN encoder, pre-LN decoder with causal
   self-attention + cross-attention over the encoder output, ReLU MLPs, shared embedding, untied head;
   two id inputs (B, enc_seq) and (B, dec_seq) (csrc/host/model_io.cpp t5) */
int sb_model_t5(int enc_layers, int dec_layers, int64_t hidden, int64_t heads, int64_t vocab, int64_t batch,
                int64_t enc_seq, int64_t dec_seq, double dropout_p, sb_model** out);
/* tie_embeddings = 0: separate encoder / decoder tables (enc_embed, dec_embed) — a tied table
   cannot be cut by pipeline_split (used by two segments) */
int sb_model_t5_ex(int enc_layers, int dec_layers, int64_t hidden, int64_t heads, int64_t vocab, int64_t batch,
                   int64_t enc_seq, int64_t dec_seq, double dropout_p, int tie_embeddings, sb_model** out);
/* f2 (no reference fixture): GPT-Neo-style pre-LN causal decoder in the reference's module
   vocabulary (csrc/host/model_io.cpp gpt_neo); its oracle is the documented extension
   oracle/causal_ext.py (a `causal` attr on softmax, proj/src/executor.cpp:907-916) */
int sb_model_gpt_neo(int layers, int64_t hidden, int64_t heads, int64_t vocab, int64_t batch, int64_t seq,
                     double dropout_p, sb_model** out);
int sb_model_fig3c(sb_model** out);
int sb_model_ffn_stack(int n, int64_t hidden, int64_t batch, sb_model** out);
/* load_model / save_model — proj/include/slapo/model_io.hpp:16-23 */
int sb_model_from_json(const char* text, sb_model** out);
int sb_model_to_json(const sb_model* m, char* buf, size_t cap, size_t* needed);
/* f32 storage for every param and input (proj/tests/combos_test.cpp:90-100) */
int sb_model_to_f32(sb_model* m);
/* modules_structurally_equal — proj/include/slapo/module.hpp:127 */
int sb_model_equal(const sb_model* a, const sb_model* b, int* equal);
/* Analytical step-time / memory estimate (slapo::estimate, proj/include/slapo/costmodel.hpp:52;
 * proj/src/costmodel.cpp:258-266). constants: {device_flops_per_s, link_bytes_per_s,
 * kernel_launch_overhead_s, optimizer_state_multiplier} or NULL for the reference defaults.
 * ints[8]: flops, recompute_flops, launches, collective_bytes, param_bytes, activation_bytes,
 * peak_memory_bytes, oom; reals[2]: step_time_s, throughput_samples_per_s; text: CostReport::to_text. */
int sb_estimate(const sb_model* m, int64_t batch, int world_size, int64_t device_memory_bytes, const double* constants,
                int64_t* ints, double* reals, char* text, size_t cap, size_t* needed);
/* Flag the first floor(ratio * L) children of `container` as checkpointed
 * (slapo::apply_checkpoint_ratio, costmodel.hpp:59; costmodel.cpp:310-324). */
int sb_model_apply_checkpoint_ratio(sb_model* m, const char* container, double ratio, int* count);
int sb_model_free(sb_model* m);
/* declared_input_specs — proj/include/slapo/shape_inference.hpp:37 */
int sb_model_num_inputs(const sb_model* m, int* n);
int sb_model_input_shape(const sb_model* m, int idx, int64_t* dims, int* ndims /* in: cap, out: rank */);
/* random_tensor(spec, seed, stream) — proj/include/slapo/executor.hpp:85 */
int sb_model_random_input(const sb_model* m, int idx, uint64_t seed, uint64_t stream, double* out, size_t cap,
                          size_t* n);
/* init_param_rank(param at dotted path, rank) — proj/include/slapo/module.hpp:147 */
int sb_model_param_values(const sb_model* m, const char* dotted, int rank, double* out, size_t cap, size_t* n);

/* -------------------------------------------------------------- schedule */
/* create_schedule / Schedule::at — proj/include/slapo/schedule.hpp:65-111 */
int sb_schedule_create(const sb_model* m, int world_size, sb_schedule** out);
int sb_schedule_at(const sb_schedule* s, const char* path, sb_schedule** out);
int sb_schedule_trace(sb_schedule* s, int flatten, const char* leaves_csv);
int sb_schedule_replace(sb_schedule* s, const char* library, const char* pattern /* NULL: whole module */);
int sb_schedule_shard(sb_schedule* s, const char* params_csv, int axis);
int sb_schedule_sync(sb_schedule* s, const char* type /* forward|backward|both */);
int sb_schedule_checkpoint(sb_schedule* s, const char* pattern /* NULL: whole module */);
int sb_schedule_define_pattern(sb_schedule* s, const char* name, const char* graph_json);
int sb_schedule_fuse(sb_schedule* s, const char* pattern, const char* backend /* composed | sm100 */);
int sb_schedule_pipeline_split(sb_schedule* s, const char* after_child);
int sb_schedule_find(sb_schedule* s, const char* glob, int* count);
/* load_schedule_script — proj/include/slapo/script.hpp:17 */
int sb_schedule_load_script(sb_schedule* s, const char* text);
int sb_schedule_num_warnings(const sb_schedule* s, int* n);
/* Schedule::apply — proj/src/schedule.cpp:719-746 */
int sb_schedule_apply(const sb_schedule* s, sb_model** out);
/* Schedule::apply with pipeline_split annotations: the stage plan
 * (ApplyResult::stages, proj/include/slapo/schedule.hpp:54-57; build_pipeline_plan,
 * proj/src/pipeline.cpp:343-420). Stage i's module is returned as a fresh sb_model;
 * stage_io: which 0 = consumes, 1 = produces (i < 0: the plan's model inputs / outputs),
 * newline-terminated names. */
int sb_schedule_apply_pipeline(const sb_schedule* s, sb_pipeline** out);
int sb_pipeline_num_stages(const sb_pipeline* p, int* n);
int sb_pipeline_stage(const sb_pipeline* p, int i, sb_model** out);
int sb_pipeline_stage_io(const sb_pipeline* p, int i, int which, char* buf, size_t cap, size_t* needed);
int sb_pipeline_free(sb_pipeline* p);
/* Pipeline-parallel training step over the stages of a pipeline_split plan (f1): GPipe with
   re-materialisation, one Executor per stage on its own device (devices: one per stage, NULL:
   the current device), stage-boundary values stashed per micro-batch (peer copies between
   devices), backward seeded with the consumers' input gradients, parameter gradients summed
   over micro-batches. Extends run_pipeline (proj/src/executor.cpp:1531-1579; forward only in
   the reference) to a training step; per-micro-batch semantics as run_pipeline. */
typedef struct sb_pipeline_executor sb_pipeline_executor;
int sb_pipeline_executor_create(const sb_pipeline* p, int micro_batches, int train, uint64_t seed, int dtype,
                                const int* devices, int fused, sb_pipeline_executor** out);
/* tp > 1: each stage's (sharded) module runs on tp lockstep ranks of its device; the gradient
   functions below then take a slot = stage * tp + rank */
int sb_pipeline_executor_create_tp(const sb_pipeline* p, int micro_batches, int tp, int train, uint64_t seed,
                                   int dtype, const int* devices, int fused, sb_pipeline_executor** out);
/* one process per (stage, tp rank): rank = stage * tp + tp_rank of world = stages * tp; stage I/O by
   ncclSend / ncclRecv over a pipeline communicator (pp_uid, broadcast from rank 0), the stage's own TP
   over an NCCL communicator of its tp ranks (tp_uid, one per stage; NULL when tp == 1). forward returns
   only the model outputs this rank's stage produces (others: empty); gradients: this rank's only. */
int sb_pipeline_executor_create_dist(const sb_pipeline* p, int micro_batches, int tp, int train, uint64_t seed,
                                     int dtype, int fused, int rank, int world, const void* pp_uid128,
                                     const void* tp_uid128, sb_pipeline_executor** out);
/* the transfer program of one rank (lines "kind m idx peer value numel", kind in fwd_recv / fwd_run /
   fwd_send / bwd_recv / bwd_run / bwd_send): what a distributed rank executes, for host-side checks */
int sb_pipeline_program(const sb_pipeline* p, int micro_batches, int tp, int rank, char* buf, size_t cap,
                        size_t* needed);
int sb_pipeline_executor_forward(sb_pipeline_executor* e, const double* const* inputs, int n);
int sb_pipeline_executor_num_outputs(sb_pipeline_executor* e, int* n);
int sb_pipeline_executor_output(sb_pipeline_executor* e, int idx, double* out, size_t cap, size_t* n, int64_t* dims,
                                int* ndims);
int sb_pipeline_executor_backward(sb_pipeline_executor* e);
int sb_pipeline_executor_num_grads(sb_pipeline_executor* e, int stage, int* n);
int sb_pipeline_executor_grad_name(sb_pipeline_executor* e, int stage, int idx, char* buf, size_t cap);
int sb_pipeline_executor_grad(sb_pipeline_executor* e, int stage, const char* dotted, double* out, size_t cap,
                              size_t* n);
int sb_pipeline_executor_num_input_grads(sb_pipeline_executor* e, int stage, int* n);
int sb_pipeline_executor_input_grad(sb_pipeline_executor* e, int stage, int idx, double* out, size_t cap, size_t* n);
int sb_pipeline_executor_time_steps(sb_pipeline_executor* e, int steps, float* ms); /* CUDA graph replay */
int sb_pipeline_executor_time_steps_ex(sb_pipeline_executor* e, int steps, int use_graph, float* ms);
int sb_pipeline_executor_free(sb_pipeline_executor* e);
int sb_schedule_free(sb_schedule* s);

/* -------------------------------------------------------------- executor */
/* Executor(root, mode, seed, world) — proj/include/slapo/executor.hpp:37-63.
 * dtype: 0 = fp32, 1 = bf16 (fp32 accumulate). fused: 1 lowers fused regions and
 * EfficientAttention to fused kernels, 0 runs them op-by-op. All `world` ranks
 * live on the current device (the reference's lockstep simulator, with device
 * collectives). */
int sb_executor_create(const sb_model* m, int train, uint64_t seed, int world, int dtype, int fused, sb_executor** out);
/* One process per GPU: this process is `rank` of `world`; collectives via NCCL. */
int sb_nccl_unique_id(void* out128);
int sb_executor_create_nccl(const sb_model* m, int train, uint64_t seed, int world, int rank, const void* unique_id128,
                            int dtype, int fused, sb_executor** out);
int sb_executor_free(sb_executor* e);
/* Host-only lowering of `rank`'s device plan (no GPU needed): JSON with op
 * kinds, checkpoint regions, the activation ledger (ActivationLedger rule,
 * proj/include/slapo/executor.hpp:20-25) and forward collective count. */
int sb_plan_describe(const sb_model* m, int train, uint64_t seed, int world, int rank, int dtype, int fused, char* buf,
                     size_t cap);
int sb_executor_set_nan_guard(sb_executor* e, int on);
/* Executor::forward (inputs replicated to every rank) */
int sb_executor_forward(sb_executor* e, const double* const* inputs, int n_inputs);
/* Executor::outputs_of_rank */
int sb_executor_num_outputs(sb_executor* e, int rank, int* n);
int sb_executor_output(sb_executor* e, int rank, int idx, double* out, size_t cap, size_t* n, int64_t* dims,
                       int* ndims);
/* Executor::backward_all_ranks (loss = sum of outputs) */
int sb_executor_backward(sb_executor* e);
int sb_executor_num_grads(sb_executor* e, int rank, int* n);
int sb_executor_grad_name(sb_executor* e, int rank, int idx, char* buf, size_t cap);
int sb_executor_grad(sb_executor* e, int rank, const char* dotted, double* out, size_t cap, size_t* n);
int sb_executor_input_grad(sb_executor* e, int rank, int idx, double* out, size_t cap, size_t* n);
/* Executor::ledger / collective_invocations */
int sb_executor_ledger(sb_executor* e, int64_t* bytes);
int sb_executor_collectives(sb_executor* e, int64_t* count);
/* device-resident stepping for benchmarks: H2D of inputs (pinned host ok),
 * one fwd+bwd (optionally through a captured CUDA graph), loss to host. */
int sb_executor_upload_inputs(sb_executor* e, const double* const* inputs, int n_inputs);
int sb_executor_step(sb_executor* e, int use_graph);
int sb_executor_step_loss(sb_executor* e, int use_graph, float* loss_host);
int sb_executor_synchronize(sb_executor* e);
/* device time (CUDA events on the executor stream) of `steps` back-to-back steps */
int sb_executor_time_steps(sb_executor* e, int steps, int use_graph, float* ms);
/* end-to-end: per step H2D of the host inputs, fwd+bwd, D2H of the loss (sum of outputs) */
int sb_executor_time_e2e(sb_executor* e, int steps, const double* const* inputs, int n_inputs, int use_graph,
                         float* ms, float* loss);
/* kernel nodes in the captured fwd+bwd CUDA graph (after a graph step) */
int sb_executor_kernels_per_step(sb_executor* e, int* n);
int sb_executor_stream(sb_executor* e, void** stream);
int sb_executor_describe(sb_executor* e, char* buf, size_t cap);
int sb_executor_profile(sb_executor* e, char* buf, size_t cap); /* per-op-kind ms of one step, JSON */
int sb_executor_device_bytes(sb_executor* e, int64_t* bytes);

/* ------------------------------------------------------- device kernels */
/* dtype codes: 0 f32, 1 bf16, 2 f64. */
/* linear_fwd / linear_dx / linear_dw / matmul_fwd — proj/src/executor.cpp:38-133.
 * epilogue: 0 none; 1 C = gelu(v), aux = v (pre-activation); 2 C = gelu'(aux) * v (dgrad into a
 * GeLU input); 3 C = max(v, 0); 4 C = v * (aux > 0) (dgrad through a ReLU whose output is aux);
 * v = alpha * A B + bias. aux shares C's row stride. */
int sb_gemm(const void* A, int ta, int64_t sAb, int64_t sAm, int64_t sAk, const void* B, int tb, int64_t sBb,
            int64_t sBk, int64_t sBn, void* C, int tc, int64_t sCb, int64_t sCm, int64_t sCn, int64_t batch, int64_t M,
            int64_t N, int64_t K, float alpha, int accumulate, const void* bias, int epilogue, void* aux, void* stream);
int sb_gemm_engine(void);                /* engine of the last sb_gemm: 0 SIMT, 1 tcgen05 1-SM, 2 tcgen05 2-SM */
int sb_gemm_force_simt(int on);
/* engine cap: 0 best available (2-SM > 1-SM tcgen05 > SIMT), 1 at most the 1-SM kernel, 2 SIMT */
int sb_gemm_set_engine(int max_engine);
/* 2-SM kernel cluster tile N: 0 default (256), 128 or 256 forced (tests) */
int sb_gemm_set_tile_n(int bn);
/* experiments: grid size of the keep-bit generator (0 = one warp per 32x32 block) */
int sb_set_mask_blocks(int n);
/* attention engine cap: 0 best available (tcgen05 > mma.sync > SIMT), 1 at most mma.sync, 2 SIMT;
 * sb_attn_engine(bwd) = engine of the last forward (0) / backward (1) call: 3 tcgen05, 2 mma.sync, 1 SIMT */
int sb_attn_set_engine(int max_engine);
int sb_attn_engine(int bwd);
/* scratch the tcgen05 path may use for deterministic split-K (wgrad) */
int sb_gemm_set_workspace(void* ws, size_t bytes);
/* dropout keep mask (apply_dropout, proj/src/executor.cpp:793-806): bit i of word i/32 =
 * uniform01(hash_combine(exec_seed, node_seed), 0xd0, i) >= p */
int sb_dropout_mask(uint32_t* bits, int64_t n, uint64_t exec_seed, uint64_t node_seed, double p, void* stream);
/* eval_layernorm_mod / backward_layernorm_mod — proj/src/executor.cpp:699-740,1158-1197 */
int sb_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int dtype,
                     int64_t rows, int64_t n, float eps, void* stream);
/* fused bias+dropout+residual+LayerNorm (the .fuse'd output block) */
int sb_bias_dropout_residual_ln_fwd(const void* partial, const void* bias, const void* residual, const void* gamma,
                                    const void* beta, void* sum, void* y, float* mean, float* rstd, int dtype,
                                    int64_t rows, int64_t n, float eps, uint64_t exec_seed, uint64_t node_seed,
                                    double p, void* stream);
/* backward_layernorm_mod (proj/src/executor.cpp:1158-1197): gx (+)= d LN / dx . g; dgamma/dbeta
 * overwritten with the column sums (fp32; may be NULL). workspace: sb_layernorm_bwd_workspace bytes */
int sb_layernorm_bwd(const void* x, const float* mean, const float* rstd, const void* gamma, const void* g, void* gx,
                     float* dgamma, float* dbeta, int dtype, int64_t rows, int64_t n, int gx_accumulate, void* workspace,
                     void* stream);
size_t sb_layernorm_bwd_workspace(int64_t rows, int64_t n);
/* backward of the fused bias+dropout+residual+LayerNorm block: g_res = g_sum (the LN input gradient),
 * g_partial = dropout_bwd(g_sum) (the Linear output gradient), dbias / dgamma / dbeta column sums */
int sb_bias_dropout_residual_ln_bwd(const void* sum, const float* mean, const float* rstd, const void* gamma,
                                    const void* g, void* g_res, void* g_partial, float* dbias, float* dgamma,
                                    float* dbeta, int dtype, int64_t rows, int64_t n, uint64_t exec_seed,
                                    uint64_t node_seed, double p, void* workspace, void* stream);
size_t sb_bias_dropout_residual_ln_bwd_workspace(int64_t rows, int64_t n);
/* the .fuse'd Linear->gelu region outside a GEMM (executor.cpp:901-906,1306-1312; the product folds it
 * into the tcgen05 GEMM epilogue, sb_gemm epilogue 1 / 2): pre = x + bias, y = gelu(pre);
 * backward gx = g * gelu'(pre), dbias = column sums of gx (fp32, may be NULL) */
int sb_bias_gelu_fwd(const void* x, const void* bias, void* y, void* pre, int dtype, int64_t rows, int64_t n,
                     void* stream);
int sb_bias_gelu_bwd(const void* pre, const void* g, void* gx, float* dbias, int dtype, int64_t rows, int64_t n,
                     void* workspace, void* stream);
size_t sb_bias_gelu_bwd_workspace(int64_t rows, int64_t n);
/* eval_embedding / backward (executor.cpp:749-784,1199-1219): row = llround(id) mod vocab; a
 * vocab-parallel shard owns rows [row0, row0 + local_rows) and writes zeros elsewhere; the backward is
 * a deterministic sorted scatter-add into the fp32 shard gradient */
int sb_embedding_fwd(const double* ids, int64_t n_ids, const void* table, int dtype, int64_t dim, int64_t vocab,
                     int64_t row0, int64_t local_rows, void* out, void* stream);
int sb_embedding_bwd(const double* ids, int64_t n_ids, const void* g, int dtype, int64_t dim, int64_t vocab,
                     int64_t row0, int64_t local_rows, float* gtable, void* workspace, void* stream);
size_t sb_embedding_bwd_workspace(int64_t n_ids, int64_t dim);
/* all_reduce (executor.cpp:812-820): rank-ascending sum of `ranks` device buffers on one device (the
 * lockstep simulator's semantics); sb_executor_allreduce: in place over an NCCL executor's ranks */
int sb_allreduce_local(const void* const* srcs, void* const* dsts, int ranks, int dtype, int64_t n, int accumulate,
                       void* stream);
int sb_executor_allreduce(sb_executor* e, void* buf, int64_t n, int dtype, void* stream);
/* attention keep bits in both layouts (S % 128 == 0): words [0, W) natural (bit e%32 of word e/32
 * for element e = ((b*nh + h)*S + i)*S + j, exactly sb_dropout_mask's bits), words [W, 2W)
 * transposed (element ((b*nh + h)*S + j)*S + i), W = B*nh*S*S/32 */
int sb_attn_dropout_mask(uint32_t* bits, int64_t B, int64_t S, int64_t nh, uint64_t exec_seed, uint64_t node_seed,
                         double p, void* stream);
/* EfficientAttention forward/backward (library.cpp:9-34 semantics). keep_bits: the
 * sb_attn_dropout_mask bits of the (B, nh, S, S) probabilities (required by the
 * tensor-core kernels when p > 0; the forward and the mma.sync backward read the
 * natural half, the tcgen05 backward the transposed half; NULL makes the portable
 * kernel hash in place). workspace: sb_attn_bwd_workspace() bytes of device scratch. acc_mask:
 * bit 0/1/2 = dq/dk/dv are accumulated into (+=), else overwritten. */
int sb_attn_fwd(const void* q, const void* k, const void* v, void* o, int64_t ld_qkv, int64_t ld_o, float* lse,
                int64_t B, int64_t S, int64_t nh, int64_t hd, float scale, uint64_t exec_seed, uint64_t node_seed,
                double p, int dtype, const uint32_t* keep_bits, void* stream);
size_t sb_attn_bwd_workspace(int64_t B, int64_t S, int64_t nh, int64_t hd);
int sb_attn_bwd(const void* q, const void* k, const void* v, const void* o, int64_t ld_qkv, int64_t ld_o,
                const float* lse, const void* dout, void* dq, void* dk, void* dv, void* workspace, int64_t B, int64_t S,
                int64_t nh, int64_t hd, float scale, uint64_t exec_seed, uint64_t node_seed, double p, int dtype,
                const uint32_t* keep_bits, int acc_mask, void* stream);

/* Causal attention core (SURVEY.md §8(f) f2 — C4's decoder blocks). Not in the reference's op set
 * (shape_inference.cpp:10-16 has no mask op), so this extends sb_attn_fwd / sb_attn_bwd rather than
 * replacing a reference interface: flags & SB_ATTN_CAUSAL masks key j > query i before the softmax
 * (the keep-bit indexing of dropout is unchanged). Causal forwards run on tcgen05 where the shape
 * fits (bf16, head_dim 64, S % 128 == 0), causal backwards on mma.sync (bf16, head_dim 64/128,
 * S % 64 == 0), anything else on the SIMT engine; other flag bits are an error. */
#define SB_ATTN_CAUSAL 1
int sb_attn_fwd_ex(const void* q, const void* k, const void* v, void* o, int64_t ld_qkv, int64_t ld_o, float* lse,
                   int64_t B, int64_t S, int64_t nh, int64_t hd, float scale, uint64_t exec_seed, uint64_t node_seed,
                   double p, int dtype, const uint32_t* keep_bits, int flags, void* stream);
int sb_attn_bwd_ex(const void* q, const void* k, const void* v, const void* o, int64_t ld_qkv, int64_t ld_o,
                   const float* lse, const void* dout, void* dq, void* dk, void* dv, void* workspace, int64_t B,
                   int64_t S, int64_t nh, int64_t hd, float scale, uint64_t exec_seed, uint64_t node_seed, double p,
                   int dtype, const uint32_t* keep_bits, int acc_mask, int flags, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SLAPO_B200_H */
