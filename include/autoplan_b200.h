/*
 * autoplan_b200.h — C-ABI of the B200 plan-exploration engine.
 *
 * The reference (`autoplan`, pure Python + numpy) has no FFI: its boundary
 * for this path is the in-process Python API.  Each entry point below states
 * the reference interface it replaces (file:line under /root/reference/pkg/src).
 * The Python host package `paper_2007_04069_b200` binds these symbols with
 * ctypes; nothing here uses torch types.
 *
 * Conventions
 *   - Every function returns 0 on success, a negative AP_ERR_* on failure;
 *     ap_last_error() gives a thread-local message for the last failure.
 *   - Pointers named *_dev are device pointers (cudaMalloc / torch CUDA
 *     tensors); everything else is host memory.  `stream` is a cudaStream_t
 *     passed as void* (0 = legacy default stream).  Launches are
 *     stream-ordered; no call synchronises the device unless it says so.
 *   - A handle is bound to the device that was current when it was created.
 *   - Sharding statuses are int8: 1 = PARTITIONED, 0 = REPLICATED,
 *     -1 = UNDECIDED (reference `sharding.py:36-41`).  Seed vectors use
 *     -1 = "no seed", 0/1 = seed R/P, 2 = a seed whose value is UNDECIDED
 *     (legal in the reference `run`, `sharding.py:221-229`).
 *   - Outcome codes: 0 = COMPLETE, 1 = INCOMPLETE, 2 = CONFLICT
 *     (reference `sharding.py:44-47`).
 */
#ifndef AUTOPLAN_B200_H
#define AUTOPLAN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AP_OK 0
#define AP_ERR_INVALID (-1)   /* bad argument or graph (reference: GraphValidationError / ValueError) */
#define AP_ERR_CUDA (-2)      /* CUDA runtime failure */
#define AP_ERR_UNSUPPORTED (-3) /* size beyond what the kernels were built for */
#define AP_ERR_INFEASIBLE (-4) /* reference: InfeasiblePlanError (pipecost.py:21) */

#define AP_OUTCOME_COMPLETE 0
#define AP_OUTCOME_INCOMPLETE 1
#define AP_OUTCOME_CONFLICT 2

/* Opcode numbering used in ap_graph_desc.opcode (reference vocabulary ir.py:33-68). */
enum ap_opcode {
  AP_OP_PARAMETER = 0, AP_OP_CONSTANT = 1, AP_OP_ADD = 2, AP_OP_SUBTRACT = 3,
  AP_OP_MULTIPLY = 4, AP_OP_DIVIDE = 5, AP_OP_EXP = 6, AP_OP_TANH = 7,
  AP_OP_DOT = 8, AP_OP_RESHAPE = 9, AP_OP_TRANSPOSE = 10, AP_OP_BROADCAST = 11,
  AP_OP_REDUCE = 12, AP_OP_TUPLE = 13, AP_OP_GET_TUPLE_ELEMENT = 14
};

typedef struct ap_graph* ap_graph_t;
typedef struct ap_decision* ap_decision_t;

/* A validated graph, instructions in ascending-id order ("positions").
 * Operands / gte_element are positions.  Mirrors HloGraph (ir.py:199-414);
 * validation itself stays on the host (the reference raises
 * GraphValidationError before any rule is compiled). */
typedef struct ap_graph_desc {
  int32_t num_instructions;
  const int32_t* opcode;          /* [N] enum ap_opcode */
  const int32_t* rank;            /* [N] */
  const int64_t* dims_offset;     /* [N+1] */
  const int64_t* dims;            /* [dims_offset[N]] extents */
  const int32_t* operand_offset;  /* [N+1] */
  const int32_t* operands;        /* [operand_offset[N]] positions */
  const int32_t* gte_element;     /* [N] position of the tuple element read, -1 otherwise */
} ap_graph_desc;

typedef struct ap_graph_info {
  int64_t num_slots;        /* |S| = sum of ranks; slot = dims_offset[pos] + dim */
  int32_t num_classes;      /* link-equivalence classes over slots */
  int32_t num_links;        /* equality links compiled from the rules */
  int64_t num_implications; /* class-level "P forces R" edges */
  int32_t num_forced;       /* distinct forced-replicated slots */
} ap_graph_info;

/* Replaces PropagationEngine.__init__/_build (sharding.py:148-202): compiles
 * the rule table into link classes, forced-R classes and implication lists
 * (host only; the tables are uploaded to the current device on first use,
 * and the handle stays bound to that device). */
int ap_graph_create(const ap_graph_desc* desc, ap_graph_t* out);
int ap_graph_destroy(ap_graph_t g);
int ap_graph_get_info(ap_graph_t g, ap_graph_info* info);
/* Host copies of the compiled tables, for tests / tooling (any pointer may be
 * NULL): class_of_slot [num_slots], class_forced [num_classes],
 * imp_offset [num_classes+1], imp_target [num_implications]. */
int ap_graph_export(ap_graph_t g, int32_t* class_of_slot, uint8_t* class_forced, int32_t* imp_offset,
                    int32_t* imp_target);

/* A decision set: the seed / candidate positions of a propagation batch.
 * Replaces the `candidates` list of PropagationEngine (sharding.py:148-153,
 * 204-208) plus any extra seeded dims.  slots[i] must be strictly
 * increasing (the reference applies seeds sorted by (id, dim),
 * sharding.py:221); is_candidate[i] != 0 marks the positions that count
 * toward newly_decided / outcome (sharding.py:240-247). */
int ap_decision_create(ap_graph_t g, const int64_t* slots, const uint8_t* is_candidate,
                       int32_t n, ap_decision_t* out);
int ap_decision_destroy(ap_decision_t d);

/* Batched sharding propagation — replaces PropagationEngine.run
 * (sharding.py:210-248), once per row of `seeds_dev`.
 *   seeds_dev    [batch, seed_stride] int8, first n columns used
 *   slots_dev    [batch, slots_stride] int8 or NULL: every slot's status
 *                (the reference `assignments`, flattened in slot order).
 *                For CONFLICT rows the reference snapshot is schedule
 *                dependent; this writes the closure with P winning and
 *                ap_propagate_trace gives the exact reference snapshot.
 *   cand_dev     [batch, cand_stride] int8 or NULL: status per decision
 *                position (all positions, candidate or not)
 *   outcome_dev  [batch] uint8 AP_OUTCOME_*
 *   counts_dev   [batch, 4] int32 or NULL: candidates decided P, decided R,
 *                newly P, newly R (newly = not seeded, sharding.py:240-245)
 */
int ap_propagate_batch(ap_graph_t g, ap_decision_t d, const int8_t* seeds_dev, int64_t batch,
                       int64_t seed_stride, int8_t* slots_dev, int64_t slots_stride,
                       int8_t* cand_dev, int64_t cand_stride, uint8_t* outcome_dev,
                       int32_t* counts_dev, void* stream);

/* ap_propagate_batch with the slot statuses emitted as 2-bit codes by K1
 * itself (code = status + 1; slot j in bits 2*(j%16) of little-endian 32-bit
 * word j/16 of its row, i.e. bits 2*(j%4) of byte j/4, codes past num_slots
 * 0) — the ap_pack_slots2 layout without the int8 round trip through HBM.
 *   packed_dev   [batch, packed_stride] uint8, packed_stride a multiple of 4
 *                and >= 4*ceil(num_slots/16)
 * Other arguments as ap_propagate_batch (same reference interface,
 * sharding.py:210-248).  Graphs outside the fast kernel's limits run the
 * generic kernel into a stream-ordered scratch and pack it. */
int ap_propagate_batch_packed(ap_graph_t g, ap_decision_t d, const int8_t* seeds_dev, int64_t batch,
                              int64_t seed_stride, uint8_t* packed_dev, int64_t packed_stride,
                              int8_t* cand_dev, int64_t cand_stride, uint8_t* outcome_dev,
                              int32_t* counts_dev, void* stream);

/* Exact replay of the reference sweep order for one seed row (one device
 * thread): the CONFLICT snapshot of `assignments` and `conflict_site`
 * (sharding.py:219-239, 250-265).  conflict_site_out gets the *position*
 * of the conflicting rule's instruction, or -1.  init_state_host (nullable,
 * [num_slots] int8) replaces the all-UNDECIDED start state, which is how
 * rule_for applies one opcode's rule to given specs (sharding.py:314-392).
 * Synchronises `stream`. */
int ap_propagate_trace(ap_graph_t g, ap_decision_t d, const int8_t* seeds_host,
                       const int8_t* init_state_host, int8_t* slots_host, int32_t* outcome_host,
                       int32_t* conflict_site_out, void* stream);

/* ---------------------------------------------------------------------------
 * Pipeline cost model (reference pipecost.py, topology.py, envs.py:276-404).
 * All fp64 arithmetic reproduces the reference's evaluation order bit for
 * bit: naive sequential stage sums (pipecost.py:99-102), CPython 3.12's
 * compensated sum() (pipecost.py:173-174, 225), left-to-right products and
 * quotients, first-wins max/min.
 * ------------------------------------------------------------------------- */

typedef struct ap_pipe* ap_pipe_t;

typedef struct ap_topology {
  int32_t num_servers;
  int32_t gpus_per_server;
  double intra_bw;   /* bytes/s inside a server (topology.py:18) */
  double inter_bw;   /* bytes/s between servers (topology.py:19) */
} ap_topology;

/* The forward instruction order of a graph (forward_subgraph, ir.py:464-470)
 * with what the cost model reads from it.  Positions index that order. */
typedef struct ap_pipe_desc {
  int32_t num_forward;
  const double* cost_ms;         /* [F] compute_cost_ms or 0.0 */
  const int64_t* out_bytes;      /* [F] output byte size */
  const int32_t* last_use;       /* [F] largest forward-consumer position, -1 if none */
  int32_t num_vars;
  const int32_t* var_anchor;     /* [V] first forward-consumer position, else own position, else -1 */
  const int64_t* var_bytes;      /* [V] in trainable_ids() order */
} ap_pipe_desc;

/* Replaces the per-graph work inside stage_metrics / candidate_pivots
 * (pipecost.py:72-141, 279-336): crossing-activation bytes per cut,
 * parameter-ownership prefixes, the naive cost prefix. */
int ap_pipe_create(const ap_pipe_desc* desc, ap_pipe_t* out);
int ap_pipe_destroy(ap_pipe_t p);

/* candidate_pivots pruning mask (pipecost.py:279-336) on the device:
 * allowed_dev [F-1] uint8 = position kept as a K-stage pivot candidate. */
int ap_pipe_candidates(ap_pipe_t p, const ap_topology* topo, int32_t num_stages, int32_t radius,
                       uint8_t* allowed_dev, void* stream);

/* Batched stage_metrics (pipecost.py:72-141): pivots_dev [B, P] strictly
 * increasing forward positions -> per stage (P+1 stages) compute_ms,
 * activation_bytes, param_bytes (fp64) and num_variables (int32). */
int ap_pipe_metrics(ap_pipe_t p, const int32_t* pivots_dev, int64_t batch, int32_t num_pivots,
                    double backward_multiplier, double* compute_dev, double* act_dev, double* param_dev,
                    int32_t* nvars_dev, void* stream);

/* ap_pipe_metrics for tuples of candidate positions of a list bound with
 * ap_pipe_train_table: stage sums are read from the bound table (tuples with
 * any other pivot fall back to the sweep; an unbound list is plain
 * ap_pipe_metrics).  Same outputs, bit for bit. */
int ap_pipe_metrics_bound(ap_pipe_t p, const int32_t* cand_pos_dev, int32_t num_cand, const int32_t* pivots_dev,
                          int64_t batch, int32_t num_pivots, double backward_multiplier, double* compute_dev,
                          double* act_dev, double* param_dev, int32_t* nvars_dev, void* stream);

/* Batched proportional_device_cuts + pipeline_length + memory_feasible
 * (pipecost.py:144-252) from per-stage metrics [B, K].  cuts_dev [B, K-1]:
 * if `given_cuts` is non-zero they are inputs, else they are written with
 * the proportional allocation.  mem_per_device < 0 disables the memory
 * check (feasible = 1); optimizer_multiplier is memory_feasible's (4.0).
 * python_floats != 0: the metrics are Python floats and builtin sum() is
 * CPython's compensated float sum; 0: they are numpy float64 scalars (as
 * PipeInferEnv.decode_metrics returns) and sum() is a naive left fold.
 * length_dev [B] fp64, feasible_dev [B] uint8 (nullable). */
int ap_pipe_length(const ap_topology* topo, int32_t num_stages, int32_t micro_batches, int64_t batch,
                   const double* compute_dev, const double* act_dev, const double* param_dev, int32_t* cuts_dev,
                   int32_t given_cuts, double mem_per_device, double optimizer_multiplier, int32_t python_floats,
                   double* length_dev, uint8_t* feasible_dev, void* stream);

/* PipeTrainEnv._state for `num_envs` states at once (envs.py:371-404): for
 * every allowed candidate pivot of each state, the slowest stage allreduce,
 * the slowest boundary transfer and the compute balance of the plan
 * applied + [candidate], block-normalised, plus the one-hot of the applied
 * picks.  cand_pos_dev [C] candidate positions (ascending); applied_dev
 * [E, max_applied] candidate *indices* (-1 padded); mask_dev [E, C];
 * state_dev [E, 4C] fp64. */
int ap_pipe_train_state(ap_pipe_t p, const ap_topology* topo, const int32_t* cand_pos_dev, int32_t num_cand,
                        const int32_t* applied_dev, int32_t max_applied, const uint8_t* mask_dev, int64_t num_envs,
                        double backward_multiplier, double* state_dev, void* stream);

/* ap_pipe_train_state that also writes the state as fp32 rows (the learner's
 * input) into state_f32 [E, >= 4C] (row stride ld_f32) and, when non-null, a
 * second copy state_f32_b: from the fused table kernel directly when the list
 * is bound, else by one conversion pass.  state_dev (fp64) is written as well. */
int ap_pipe_train_state_ex(ap_pipe_t p, const ap_topology* topo, const int32_t* cand_pos_dev, int32_t num_cand,
                           const int32_t* applied_dev, int32_t max_applied, const uint8_t* mask_dev, int64_t num_envs,
                           double backward_multiplier, double* state_dev, float* state_f32, int64_t ld_f32,
                           float* state_f32_b, int64_t ld_f32_b, void* stream);

/* generate_environment(distribution, n, seed) (dataproc.py:123-145) for many
 * seeds: kind 0 uniform (= ap_generate_uniform_envs), 1 normal (numpy's
 * ziggurat, N(0.5, 0.15) clipped to [0, 1]), 2 binomial (numpy's BTPE,
 * B(100, 0.5) / 100).  pcg_states as ap_generate_uniform_envs; arrays_out
 * [num_envs, 3, granularity] fp64, bit-identical to the host. */
int ap_generate_envs(int32_t kind, const uint64_t* pcg_states, int64_t num_envs, int32_t n, int32_t granularity,
                     double* arrays_out, void* stream);
/* Host run of the same per-environment code (tests): kinds 1 and 2 of ap_generate_envs. */
int ap_generate_envs_host(int32_t kind, const uint64_t* pcg_states, int64_t num_envs, int32_t n,
                          int32_t granularity, double* arrays_out);
/* Host run of the device samplers (tests): kind 0 Generator.standard_normal(),
 * kind 1 Generator.binomial(bin_n, bin_p); state6 as ap_pcg64_host_draws. */
int ap_np_samples_host(uint64_t* state6, int32_t kind, int64_t count, int64_t bin_n, double bin_p, double* out);

/* Host-consumer slot format (run_batch_host(want_slots="packed")): K1's int8
 * slot rows [batch, slots_stride] (-1 / 0 / 1, sharding.py:36-48) packed to
 * 2 bits per slot, code = status + 1, slot j in bits 2*(j%4) of byte j/4 of
 * its row; packed rows are packed_stride >= 4*ceil(num_slots/16) bytes and
 * codes past num_slots are 0.  Cuts the D2H of a full-contract plan 4x. */
int ap_pack_slots2(const int8_t* slots_dev, int64_t batch, int64_t slots_stride, int64_t num_slots, uint8_t* packed_dev,
                   int64_t packed_stride, void* stream);

/* PP-infer data plane: num_envs synthetic uniform
 * profiles at once, bit-identical to generate_environment("uniform", n, seed)
 * (dataproc.py:123-145 -> build_environment_arrays :99-120 -> coarsen :79-96).
 * pcg_states [E, 4] uint64 = each seed's PCG64 (state hi, state lo, inc hi,
 * inc lo) as numpy's default_rng(seed) initialises it; arrays_out [E, 3, G]
 * fp64 = the coarsened, jointly scaled C, A, W arrays.  n <= 8533. */
int ap_generate_uniform_envs(const uint64_t* pcg_states, int64_t num_envs, int32_t n, int32_t granularity,
                             double* arrays_out, void* stream);

/* Binds a candidate list to the handle: builds (once, outside stream capture)
 * the table of every stage sum a plan over these candidates can have --
 * the naive sum of cost[start .. end] for each pair of candidate boundaries,
 * (C+1)^2 + (C+1) fp64 owned by the handle.  Later ap_pipe_train_state calls
 * with the same (cand_pos_dev, num_cand) read stage sums from it instead of
 * re-summing the cost array per candidate (bit-identical: same additions,
 * same order).  The list's contents must not change while bound; calling
 * again rebuilds from the current contents.  AP_ERR_UNSUPPORTED when the
 * table would exceed 4 GiB (the per-candidate sweep is then used).
 * New in this library: the reference recomputes stage_metrics per candidate
 * (envs.py:378-397). */
int ap_pipe_train_table(ap_pipe_t p, const int32_t* cand_pos_dev, int32_t num_cand, void* stream);

/* PP-infer terminal evaluation on coarsened arrays (envs.py:593-616):
 * decode_metrics + pipeline_length on the normalised topology for B
 * (boundaries, cuts) points.  arrays_dev = [3 * G] fp64 (C*, A*, W*). */
int ap_infer_length(const double* arrays_dev, int32_t granularity, const ap_topology* topo_normalized,
                    int32_t num_stages, int32_t micro_batches, const int32_t* boundaries_dev,
                    const int32_t* cuts_dev, int64_t batch, double* length_dev, void* stream);

/* Exhaustive PP-infer search over per-slot bands (helpers.py:156-230 space,
 * env-path arithmetic): lexicographic first-wins argmin.  band_* are host
 * CSR lists of allowed values per pick (K-1 picks each).  Synchronises. */
int ap_infer_search(const double* arrays_dev, int32_t granularity, const ap_topology* topo_normalized,
                    int32_t num_stages, int32_t micro_batches, const int32_t* band_b, const int32_t* band_b_off,
                    const int32_t* band_c, const int32_t* band_c_off, int32_t* best_boundaries,
                    int32_t* best_cuts, double* best_length, int64_t* points_evaluated, void* stream);

/* ---------------------------------------------------------------------------
 * DQN (reference agent.py).  The Q-network's dense contractions run on the
 * tcgen05 tensor cores; everything else of the learner stays device-resident.
 * ------------------------------------------------------------------------- */

/* C[M,N] = op(A)[M,K] * op(B)[K,N] (+ bias[N]) (ReLU), fp32 in/out.
 * op(A)[m,k] = transA ? A[k*lda+m] : A[m*lda+k]; op(B)[k,n] = transB ?
 * B[n*ldb+k] : B[k*ldb+n].  precision 3 = 3xTF32 split (fp32-accurate),
 * 1 = plain TF32.  Replaces the numpy matmuls of QNetwork.forward_cached /
 * backward (agent.py:93-136). */
int ap_gemm_tf32(const float* A, int64_t lda, int32_t transA, const float* B, int64_t ldb, int32_t transB,
                 float* C, int64_t ldc, int32_t M, int32_t N, int32_t K, const float* bias, int32_t relu,
                 int32_t precision, void* stream);

/* Dueling combine Q = V + A - mean(A) from fused head outputs z = [V, A]
 * (agent.py:104-109).  z [B, 1+A] (row stride ldz), q [B, A]. */
int ap_dqn_dueling(const float* z, int64_t ldz, float* q, int64_t ldq, int32_t B, int32_t A, void* stream);

/* Masked argmax per row, ties to the lowest index (agent.py:147-152); with
 * epsilon > 0, epsilon-greedy with a counter-based RNG keyed by `seed`
 * (throughput mode; parity mode draws with numpy on the host). */
int ap_dqn_act(const float* q, int64_t ldq, const uint8_t* mask, int64_t ldm, int32_t E, int32_t A, float epsilon,
               uint64_t seed, int32_t* actions, void* stream);

/* Double-DQN TD error, per-row Huber loss contributions w*huber(td) (loss_rows
 * [B]; the loss is their mean) and the gradient w.r.t. z = [V, A]
 * (agent.py:258-299, 114-118). */
int ap_dqn_td(const float* q, const float* online_next, const float* target_next, int64_t ldq, const int32_t* actions,
              const float* rewards, const uint8_t* done, const uint8_t* next_mask, int64_t ldm, const float* weights,
              int32_t B, int32_t A, float gamma, float huber_delta, float* dz, int64_t ldz, float* td,
              float* loss_rows, void* stream);
/* ap_dqn_td reading actions / rewards / done / next masks straight from replay-ring
 * rows indices[b] (the sample gather of agent.py:207-223 fused in); dz_t
 * (nullable) also receives dz^T [1 + A, B]. */
int ap_dqn_td_ring(const float* q, const float* online_next, const float* target_next, int64_t ldq,
                   const int32_t* indices, const int32_t* ring_actions, const float* ring_rewards,
                   const uint8_t* ring_done, const uint8_t* ring_next_mask, int64_t ldm, const float* weights,
                   int32_t B, int32_t A, float gamma, float huber_delta, float* dz, int64_t ldz, float* dz_t,
                   int64_t ldzt, float* td, float* loss_rows, void* stream);
/* n <= 8 transposes in one launch: dst_i[c * ld_dst_i + r] = src_i[r * ld_src_i + c]
 * for r < rows_i, c < cols_i (descriptor arrays are host memory). Refreshes the
 * transposed weight copies the K-major tcgen05 GEMMs read. */
int ap_transpose_batch(int32_t n, const float* const* src, const int64_t* ld_src, float* const* dst,
                       const int64_t* ld_dst, const int32_t* rows, const int32_t* cols, void* stream);

/* Dueling head forward for 1 + A <= 8 outputs (agent.py:99-109): q = V + A - mean(A)
 * with [V, A] = h @ wh + bh; wh_t is wh transposed ([1 + A, H], row stride ldw).
 * AP_ERR_UNSUPPORTED for wider heads (GEMM + ap_dqn_dueling). */
int ap_dqn_head_forward(const float* h, int64_t ldh, const float* wh_t, int64_t ldw, const float* bh, int32_t B,
                        int32_t H, int32_t A1, float* q, int64_t ldq, void* stream);
/* ReLU backward in place on dh [B, H] (agent.py:132) that also writes dh^T [H, B]. */
int ap_dqn_relu_backward_t(float* dh, int64_t lddh, const float* h, int64_t ldh, int32_t B, int32_t H, float* dh_t,
                           int64_t ldt, void* stream);
/* dh[i] = 0 where h[i] <= 0 (ReLU backward, agent.py:132). */
int ap_dqn_relu_backward(float* dh, const float* h, int64_t n, void* stream);
/* out[c] = sum_r x[r*ld + c] (bias gradients, agent.py:118,134). */
int ap_dqn_colsum(const float* x, int64_t ld, int32_t rows, int32_t cols, float* out, void* stream);
/* Roofline probe (no reference counterpart): `blocks` x 256 threads each run 8
 * independent fp64 add chains of `iters` adds; time the launch to get the
 * FP64 add throughput that bounds the PP-train cost kernels.  scratch_dev:
 * one double, never written in practice. */
int ap_probe_fp64_add(int32_t blocks, int64_t iters, double* scratch_dev, void* stream);

/* Gradient into the last hidden layer from the (1 + A)-wide head (agent.py:120-132):
 * dh = relu'(h) * (dz @ wh^T), wh [H, A1] row-major; dh_t (nullable) gets dh^T [H, B]. */
int ap_dqn_head_backward(const float* dz, int64_t ldz, const float* wh, int64_t ldw, const float* h, int64_t ldh,
                         int32_t B, int32_t H, int32_t A1, float* dh, int64_t lddh, float* dh_t, int64_t ldt,
                         void* stream);
/* ap_dqn_head_backward for the dueling TD gradient the TD kernels write (dz[b] =
 * g_b (e_0 + e_{1+a_b}) - (g_b/A)[0, 1, .., 1]): dh[b, j] = relu'(h) (g_b wh[j,0] +
 * g_b wh[j,1+a_b] - (g_b/A) sum_k wh[j,1+k]) in O(B H) after one row-sum pass over
 * wh (rowsum_scratch [H]) instead of the O(B H A) product.  Same value up to fp32
 * rounding; the throughput learner uses it for wide heads. */
int ap_dqn_head_backward_dueling(const float* dz, int64_t ldz, const float* wh, int64_t ldw, const float* h,
                                 int64_t ldh, int32_t B, int32_t H, int32_t A1, float* rowsum_scratch, float* dh,
                                 int64_t lddh, float* dh_t, int64_t ldt, void* stream);
/* Adam over a flat parameter buffer (agent.py:240-250); correct1/2 = 1 - beta^t. */
int ap_dqn_adam(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1, float beta2,
                float eps, float correct1, float correct2, void* stream);

/* Prioritized replay sample for B caller-drawn uniforms (agent.py:207-223):
 * p**alpha, numpy pairwise sum, sequential cumsum / cdf[-1],
 * searchsorted(side='right'), IS weights (n*p)**-beta / max.  fp64.
 * scratch: 2*n + B doubles. */
int ap_per_sample(const double* priorities, int32_t n, double alpha, double beta, const double* uniforms, int32_t B,
                  double* scratch, int32_t* indices, float* weights, void* stream);
/* priorities[idx] = |td| + 1e-6, last duplicate wins (agent.py:225-226). */
int ap_per_update(double* priorities, const int32_t* indices, const float* td, int32_t B, void* stream);
/* dst[b, :] = src[idx[b], :] (replay minibatch gather). */
int ap_gather_rows(const float* src, int64_t lds, const int32_t* idx, int32_t B, int32_t cols, float* dst,
                   int64_t ldd, void* stream);
/* Two row gathers with the same indices in one launch: dst0[b] = src0[idx[b]],
 * dst1[b] = src1[idx[b]] (src1 nullable: a single gather). */
int ap_gather_rows_pair(const float* src0, int64_t lds0, float* dst0, int64_t ldd0, const float* src1, int64_t lds1,
                        float* dst1, int64_t ldd1, const int32_t* idx, int32_t B, int32_t cols, void* stream);

/* ---------------------------------------------------------------------------
 * Vectorised episode driver (device-resident train_partition, cli.py:193-248)
 * ------------------------------------------------------------------------- */

/* seeds[e, position[e]] = P (action 0) or R (action 1) (envs.py:137-144). */
int ap_vec_apply(int8_t* seeds, int64_t ld, const int32_t* position, const int32_t* actions, int32_t E, void* stream);

/* After ap_propagate_batch over the E seed rows: rewards (0.4 newP + 0.1 newR
 * or -1 on conflict), done flags, next decision positions (first undecided dim
 * in `order`), next states [E, n+1], next masks, episode bookkeeping and
 * auto-reset of finished envs (envs.py:103-177, 207-221).  order_index [n]
 * (nullable) is the inverse of `order`: the search for the first undecided
 * dim starts at the current position's rank (decided dims stay decided within
 * an episode, so nothing before it can be undecided). */
int ap_vec_post(int32_t E, int32_t n, int64_t ld, int8_t* seeds, const int8_t* status, const uint8_t* outcome,
                const int32_t* counts, int32_t* prev_counts, int32_t* position, const int32_t* order,
                const int32_t* order_index, float* cur_state,
                int64_t lds, float* next_state, float* rewards, uint8_t* done, uint8_t* next_mask, int32_t A,
                float* ep_return, float* finished_return, int32_t* finished_partitions, int32_t* episodes_done,
                void* stream);

/* Per-env best completed plan of the vectorised driver (cli.py:237-240):
 * replaces the incumbent iff (partitions, return) is strictly greater; records
 * the global episode id step_base + e and copies the per-candidate status row
 * into best_status [E, ld].  Cross-env / cross-rank selection keeps the
 * reference's first-wins by lowest episode id. */
int ap_vec_track_best(int32_t E, int32_t n, int64_t ld, const int8_t* status, const uint8_t* outcome,
                      const uint8_t* done, const int32_t* finished_partitions, const float* finished_return,
                      int64_t step_base, const int64_t* ctl, int32_t world, int32_t rank, int32_t* best_partitions,
                      float* best_return, int64_t* best_episode, int8_t* best_status, void* stream);

/* ---- graph-capturable driver: device control block --------------------------------
 * ctl = int64[4] in device memory: {vector_step, ring_slot, ring_size, train_steps}.
 * The *_ctl entry points read their step counters from it instead of by-value
 * arguments, so one captured CUDA graph of a whole vector step replays
 * correctly (cli.py:193-248 loop body).  With ctl, ap_vec_track_best uses
 * step_base = (ctl[0] * world + rank) * E. */

/* epsilon-greedy act (agent.py:50-55,147-170) with epsilon from ctl[3] and the
 * hash counter ctl[0] + 1 */
int ap_dqn_act_ctl(const float* q, int64_t ldq, const uint8_t* mask, int64_t ldm, int32_t E, int32_t A,
                   float epsilon_start, float epsilon_final, int64_t decay_iters, const int64_t* ctl, int32_t* actions,
                   void* stream);
/* Data-parallel learner step in one kernel: all-reduce (mean) of the
 * Q-gradient over NVLink peer memory + Adam (agent.py:229-250, t = ctl[3] + 1).
 * xbuf_peers / pad_peers are HOST arrays of `world` device pointers: every rank's
 * symmetric exchange buffer (2 * n floats) and flag row (world uint32, zeroed
 * once); counter is a local zeroed uint32.  Ranks average in rank order, so every
 * replica gets identical parameters.  Stream-capturable; replaces NCCL all-reduce
 * + ap_dqn_adam_ctl. */
int ap_dp_allreduce_adam(int32_t world, int32_t rank, const float* grad, float* const* xbuf_peers,
                         uint32_t* const* pad_peers, int64_t n, float* params, float* m, float* v, float lr,
                         float beta1, float beta2, float eps, const int64_t* ctl, uint32_t* counter, void* stream);
/* ap_dqn_adam_ctl that also writes the transposed weight copies: element i of
 * segment s (flat offset seg_off[s], [rows, cols] row-major) goes to
 * seg_dst[s][c * seg_ldd[s] + r] too (host descriptor arrays, <= 8 segments). */
int ap_dqn_adam_ctl_t(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1,
                      float beta2, float eps, const int64_t* ctl, int32_t nseg, const int64_t* seg_off,
                      const int32_t* seg_rows, const int32_t* seg_cols, float* const* seg_dst, const int64_t* seg_ldd,
                      void* stream);
/* Weight-gradient GEMM with Adam fused into its epilogue (throughput learner, first
 * layer): C[M, N] = A[M, K] B[N, K]^T is stored as the gradient and Adam updates
 * m, v and params (each at C's offset, row stride ldc) in place, t = ctl[TRAIN] +
 * (counter_advanced ? 0 : 1), same arithmetic as ap_dqn_adam_ctl_t; the updated
 * rows r < t_rows are also written transposed to t_dst[c * t_ld + r].
 * AP_ERR_UNSUPPORTED for shapes that need split-K (the caller runs the plain GEMM). */
int ap_gemm_tf32_adam(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int32_t M,
                      int32_t N, int32_t K, float* m, float* v, float* params, const int64_t* ctl,
                      int32_t counter_advanced, float lr, float beta1, float beta2, float eps, float* t_dst,
                      int64_t t_ld, int32_t t_rows, void* stream);

/* ap_dqn_adam_ctl_t when the learn-step counter ctl[AP_CTL_TRAIN] has already
 * been advanced for this step (counter_advanced = 1: t = ctl[TRAIN]; 0: t =
 * ctl[TRAIN] + 1) -- the pipelined learner runs the priority scatter, which
 * advances it, on a parallel branch that joins before Adam. */
int ap_dqn_adam_ctl_t_adv(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1,
                          float beta2, float eps, const int64_t* ctl, int32_t nseg, const int64_t* seg_off,
                          const int32_t* seg_rows, const int32_t* seg_cols, float* const* seg_dst,
                          const int64_t* seg_ldd, int32_t counter_advanced, void* stream);
/* ap_per_update_scaled that also counts the learn step: ctl[3] += 1. */
int ap_per_update_scaled_ctl(double* scaled, const int32_t* indices, const float* td, int32_t B, double alpha,
                             int64_t* ctl, void* stream);
/* Adam (agent.py:229-250) with bias corrections for t = ctl[3] + 1 */
int ap_dqn_adam_ctl(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1,
                    float beta2, float eps, const int64_t* ctl, void* stream);
/* ap_per_push at ring slot ctl[1] */
int ap_per_push_ctl(int32_t E, int32_t S, int32_t A, int64_t cap, const float* states, const float* next_states,
                    int64_t lds, const int32_t* actions, const float* rewards, const uint8_t* done,
                    const uint8_t* masks, float* r_states, float* r_next, int32_t* r_actions, float* r_rewards,
                    uint8_t* r_done, uint8_t* r_masks, double* r_prio, const double* max_prio, const int64_t* ctl,
                    void* stream);
/* ap_per_sample_fast over the first ctl[2] ring entries, uniforms from a counter
 * hash of (seed, ctl[3], row) (agent.py:207-223 semantics, throughput RNG) */
int ap_per_sample_ctl(const double* priorities, int64_t capacity, double beta, int32_t B, uint64_t seed,
                      double* cdf_scratch, int32_t* indices, float* weights, double* max_priority, const int64_t* ctl,
                      void* stream);
/* Vectorised PipeTrainEnv (envs.py:276-404), E envs on the device.  picks / positions
 * [E, P] (P = K - 1 candidate indices / their forward positions), n_applied [E].
 * ap_vec_pipe_apply appends actions[e] and flags the envs whose last pick it was. */
int ap_vec_pipe_apply(int32_t E, int32_t P, const int32_t* actions, const int32_t* cand_pos, int32_t* picks,
                      int32_t* positions, int32_t* n_applied, uint8_t* done, void* stream);
/* After ap_pipe_metrics + ap_pipe_length over every env's positions: terminal
 * rewards (reward_shape 0: 1/L, 1: 1/sqrt L; -1/sqrt L if infeasible; L >= 1e-12),
 * per-env incumbents (min L over feasible episodes, strict <, cli.py:315; global
 * episode id (ctl[0] * world + rank) * E + e), auto-reset (positions back to
 * dummy_pos [P]), and the next state inputs: applied_state [E, a_max] and the
 * action mask [E, C] (envs.py:284-293); next_mask = 0 for finished envs. */
int ap_vec_pipe_post(int32_t E, int32_t C, int32_t P, int32_t a_max, const double* length, const uint8_t* feasible,
                     const uint8_t* done, int32_t reward_shape, const int32_t* dummy_pos, float* rewards,
                     int32_t* picks, int32_t* positions, int32_t* n_applied, int32_t* applied_state, uint8_t* mask,
                     uint8_t* next_mask, double* best_len, int32_t* best_picks, int64_t* best_episode,
                     float* ep_return, float* finished_return, int32_t* episodes_done, const int64_t* ctl,
                     int32_t world, int32_t rank, void* stream);
/* Vectorised PipeInferEnv (envs.py:407-626): bnd / cut [E, P] picks (boundaries in
 * 1..G-1, device cuts in 1..D-1), nb / nc [E]; ap_vec_infer_apply routes action a
 * (a < G-1: boundary a+1, else cut a-(G-1)+1) and flags finished envs.
 * ap_vec_infer_post (after ap_infer_length over every row): terminal rewards
 * 1 / max(L, 1e-12), incumbents (min L, strict <), reset to the dummy tails, the
 * phased action mask [E, (G-1)+(D-1)] within the per-pick bands band_b [P, G] /
 * band_c [P, D] (1 = allowed), and the 2P pick slots at the end of each fp32 state row
 * (S wide, row stride ld_state). */
int ap_vec_infer_apply(int32_t E, int32_t P, int32_t G, const int32_t* actions, int32_t* bnd, int32_t* cut,
                       int32_t* nb, int32_t* nc, uint8_t* done, void* stream);
int ap_vec_infer_post(int32_t E, int32_t P, int32_t G, int32_t D, int32_t S, int64_t ld_state, const double* length,
                      const uint8_t* done, const int32_t* dummy_b, const int32_t* dummy_c, const uint8_t* band_b,
                      const uint8_t* band_c, float* rewards, int32_t* bnd, int32_t* cut, int32_t* nb, int32_t* nc,
                      uint8_t* mask, uint8_t* next_mask, float* state, double* best_len, int32_t* best_b,
                      int32_t* best_c, int64_t* best_episode, float* ep_return, float* finished_return,
                      int32_t* episodes_done, const int64_t* ctl, int32_t world, int32_t rank, void* stream);
/* mode 0: ctl[3] += 1 (one learn step); mode 1: ctl[0] += 1, ctl[1] = (ctl[1] + E) % cap,
 * ctl[2] = min(ctl[2] + E, cap) (one vector step) */
int ap_vec_ctl_advance(int64_t* ctl, int32_t mode, int64_t E, int64_t cap, void* stream);

/* E transitions into the device replay ring at slots (slot0 + e) % cap with
 * the running max priority (agent.py:197-205). */
int ap_per_push(int32_t E, int32_t S, int32_t A, int64_t slot0, int64_t cap, const float* states,
                const float* next_states, int64_t lds, const int32_t* actions, const float* rewards,
                const uint8_t* done, const uint8_t* masks, float* r_states, float* r_next, int32_t* r_actions,
                float* r_rewards, uint8_t* r_done, uint8_t* r_masks, double* r_prio, const double* max_prio,
                void* stream);

/* Throughput-mode PER sample (parallel scan; not numpy-ordered) over
 * priorities already raised to alpha; also refreshes the running max (in the
 * same scaled domain) that ap_per_push assigns.  cdf_scratch: n doubles. */
int ap_per_sample_fast(const double* scaled_priorities, int32_t n, double alpha, double beta, const float* uniforms,
                       int32_t B, double* cdf_scratch, int32_t* indices, float* weights, double* max_priority,
                       void* stream);
/* scaled[idx] = (|td| + 1e-6)**alpha, last duplicate wins (throughput mode). */
int ap_per_update_scaled(double* scaled, const int32_t* indices, const float* td, int32_t B, double alpha,
                         void* stream);

/* ---------------------------------------------------------------------------
 * Reference-semantics search loop on the device (parity mode, one env):
 * train_partition (cli.py:193-248) with agent.act / env.step / observe /
 * learn (agent.py:155-337, envs.py:103-175) as kernels, numpy's PCG64 stream
 * reproduced on the device, and a CUDA graph with WHILE / IF conditional nodes
 * looping over episodes without returning to the host.
 * ctl words 0..3 are the AP_CTL_* words of the vector driver.
 * ------------------------------------------------------------------------- */
enum {
  AP_PL_STEP = 0,       /* env steps of this launch (log index) */
  AP_PL_EPISODES = 4,   /* episodes finished in this launch */
  AP_PL_BUDGET = 5,     /* episodes to run in this launch */
  AP_PL_MAX_STEPS = 6,  /* log capacity (steps) */
  AP_PL_POS = 7,        /* candidate index up for decision (-1 none) */
  AP_PL_EP_STEPS = 8,   /* steps of the running episode */
  AP_PL_BEST_PART = 9,  /* incumbent partitions (-1 none) */
  AP_PL_BEST_EP = 10,   /* incumbent episode (run-relative) */
  AP_PL_SYNC = 11,      /* target sync due after this learn step */
  AP_PL_T_POS = 12,     /* decision position of the reset template */
  AP_PL_EP_BASE = 13,   /* run-relative index of this launch's first episode */
  AP_PL_TRAIN0 = 14,    /* train steps before the run (loss log base) */
  AP_PL_LOSS_BAD = 15,  /* first run-relative train step with a non-finite loss, or -1 */
  AP_PL_TAB_BASE = 16,  /* Adam step t of bias-correction table entry 0, minus 1 */
  AP_PL_ACTIVE = 17,    /* set by the act of each step: 0 once the budget is spent (the loop body's
                           later kernels then do nothing: several steps per WHILE iteration) */
  AP_PL_GEN = 18,       /* env steps ever taken by this loop state (advanced by env.step) */
  AP_PL_ACK = 19,       /* GEN + 1 once the step's early PER sample has read the ring and stream */
  AP_PL_FAULT = 20,     /* nonzero: a device-side wait gave up (the loop's results are void) */
  AP_PL_WORDS = 32
};
enum { AP_PLD_TOTAL = 0, AP_PLD_BEST_REWARD = 1, AP_PLD_WORDS = 2 };

typedef struct ap_parity_loop {
  int64_t* ctl;             /* [AP_PL_WORDS] */
  double* dctl;             /* [AP_PLD_WORDS]: episode return so far, incumbent return */
  uint64_t* rng;            /* numpy PCG64: state hi, lo, inc hi, lo, has_uint32, uinteger */
  int32_t n, ld;            /* candidate dims, seed / status row stride */
  int32_t num_actions;
  int8_t* seeds;            /* [ld] committed seeds of the episode */
  int8_t* seeds_try;        /* [ld] seeds + this step's decision (K1 input row) */
  int8_t* decided;          /* [ld] decided candidate statuses */
  const int8_t* status;     /* [ld] K1 candidate statuses of seeds_try */
  const uint8_t* outcome;   /* [1] K1 outcome */
  const int32_t* order;     /* [n] decision order (candidate indices) */
  const int8_t* t_seeds;    /* reset template (reset or finetune_reset) */
  const int8_t* t_decided;
  float* state;             /* [n + 1] current state row (the Q-network input) */
  float* r_states;          /* replay ring [cap, r_ld] */
  float* r_next;
  int64_t r_ld, cap;
  int32_t* r_actions;
  float* r_rewards;
  uint8_t* r_done;
  uint8_t* r_mask;          /* [cap, num_actions] */
  double* r_prio;
  double eps_start, eps_final;
  int64_t eps_decay;
  int8_t* best_row;         /* [ld] incumbent strategy */
  int32_t* log_action;      /* [max_steps] */
  double* log_reward;
  int32_t* log_pos;
  int8_t* log_decided;      /* [max_steps, ld] state rows before each step, or NULL */
  uint8_t* ep_conflict;     /* [budget] */
  int32_t* ep_len;
  double* ep_return;
  float* loss_log;          /* [loss_cap] summed batch loss per train step */
  int64_t loss_cap;
  int64_t learn_gate;       /* > 0: the learn-body kernels do nothing while the ring holds fewer
                               rows (a loop graph without the IF node); 0: ungated */
  double* r_scaled;         /* early_sample: [cap] priorities ** per_alpha, kept current by env.step
                               and the fused learn step (the early PER sample reads it) */
  double* pstat;            /* early_sample: [2] the ring's max priority and its ** per_alpha */
  double per_alpha;
  int64_t early_sample;     /* 1: each step's PER sample runs beside its act / env kernels
                               (ap_parity_sample early mode); the act then waits for its ack
                               before it advances the random stream */
} ap_parity_loop;

/* agent.act: eps-greedy with numpy's draws (random(), integers(A)) over Q of the
 * current state; writes the K1 input row seeds_try. */
int ap_parity_act(const ap_parity_loop* L, const float* q_dev, int32_t* action_dev, void* stream);
/* env.step after K1 + episode bookkeeping + agent.observe (ring push at the
 * current max priority) + reset to the template after a finished episode. */
int ap_parity_post(const ap_parity_loop* L, const int32_t* action_dev, void* stream);
/* agent.learn's B random() draws (the uniforms of rng.choice) and the PER sample of the ring
 * (agent.py:207-223), one kernel: indices [B], importance weights [B]; scratch holds 2 * cap + B
 * doubles; uniforms_out optional.  No-op while the loop's learn gate is closed.  1 <= B <= 1024.
 * Late mode (early == 0, after env.step): the pushed ring, the act's random stream, which it
 * advances.  Early mode (launched with the act of the step, L->early_sample): the ring and stream
 * as the step starts -- it replays the act's draws (random(), integers(A) when exploring),
 * counts the step's pending push (max priority at the current slot), acknowledges its read in
 * ctl[AP_PL_ACK] and leaves the final stream state in rng_next (6 words) for the learn step to
 * commit (ap_fused_learn.rng_from). */
int ap_parity_sample(const ap_parity_loop* L, int32_t B, double alpha, double beta, double* scratch,
                     int32_t* indices, float* weights, double* uniforms_out, uint64_t* rng_next, int32_t early,
                     void* stream);
/* loss log, train-step counter, target-sync flag. */
int ap_parity_learn_tail(const ap_parity_loop* L, const float* loss_dev, int32_t sync_every, void* stream);
/* scaled[i] = priorities[i] ** alpha for i < n (the PER sample's cache, CUDA pow as everywhere)
 * and, with pstat, pstat = {max priority (1.0 for n == 0), its ** alpha}. */
int ap_per_scaled(const double* priorities, int64_t n, double alpha, double* scaled, double* pstat, void* stream);
/* dst[k][:count[k]] = src[k][...] when ctl[AP_PL_SYNC] (n <= 8 segments). */
int ap_parity_target_sync(const int64_t* ctl, int32_t n, const float* const* src, float* const* dst,
                          const int64_t* count, void* stream);
/* ap_dqn_adam with the bias corrections of step t = ctl[AP_CTL_TRAIN] + t_offset + 1
 * read from a host-computed table: ctab[2 * k + {0, 1}] = fp32(1 - beta{1,2}^t)
 * for k = t - 1 - ctl[AP_PL_TAB_BASE] (the host's `1.0 - beta ** t`, agent.py:241-242). */
int ap_dqn_adam_tab(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1,
                    float beta2, float eps, const float* ctab, const int64_t* ctl, int64_t t_offset, void* stream);

/* Host-side run of the device's numpy PCG64 emulation (pcg64.cuh), for tests:
 * ops[i] = 0 draws random(), ops[i] = k >= 1 draws integers(k); state6 advances. */
int ap_pcg64_host_draws(uint64_t* state6, const int64_t* ops, int32_t n, double* out);

/* ---------------------------------------------------------------------------
 * Fused small-batch learner (csrc/fused_mlp.cu): one persistent cooperative
 * kernel per DQN learn step -- forwards of the online and target networks,
 * double-DQN TD + Huber (agent.py:258-299), the dueling-MLP backward
 * (agent.py:111-136), priorities (agent.py:226) and Adam (agent.py:229-250),
 * with grid barriers between dependent phases.  Network layout: the flat
 * parameter buffer of QNetwork (w_i [dims[i], dims[i+1]] and b_i at w_off[i] /
 * b_off[i], i <= L, the head at index L, dims[L+1] = 1 + A).
 * ------------------------------------------------------------------------- */
typedef struct ap_fused_learn {
  int32_t L;                /* hidden layers, 1..4 */
  int32_t dims[6];
  int64_t w_off[5], b_off[5];
  int32_t batch;            /* 1..256 */
  float* params;            /* online flat parameters (updated in place) */
  const float* target;      /* target flat parameters */
  const float* r_states;    /* replay ring [cap, r_ld] */
  const float* r_next;
  int64_t r_ld;
  const int32_t* r_actions;
  const float* r_rewards;
  const uint8_t* r_done;
  const uint8_t* r_mask;    /* [cap, A] */
  double* r_prio;           /* priorities[idx[b]] = |td| + 1e-6, the last duplicate wins */
  const int32_t* idx;       /* [batch] sampled ring rows */
  const float* weights;     /* [batch] importance weights */
  float gamma, huber_delta;
  float* grad;              /* [nparams] scratch gradient */
  float* m;
  float* v;
  int64_t nparams;
  float lr, beta1, beta2, eps;
  float correct1, correct2; /* bias corrections, unless ctab (ap_dqn_adam_tab semantics) */
  const float* ctab;
  const int64_t* ctl;
  int64_t t_offset;
  float* wt[5];             /* transposed weight copies to refresh, or NULL */
  int64_t wt_ld[5];
  float* td;                /* [batch] */
  float* loss;              /* [1] sum_b w_b huber(td_b) */
  float* workspace;         /* ap_mlp_fused_workspace(L, dims, batch, 0) floats */
  uint32_t* barrier;        /* [4] zero-initialised, private to the caller's stream */
  uint64_t* trace;          /* optional [16]: %globaltimer after each phase (profiling) */
  int64_t gate;             /* > 0 (with ctl): no-op while ctl[AP_CTL_SIZE] < gate */
  /* optional parity-loop tail (replaces ap_parity_learn_tail + ap_parity_target_sync):
   * with tail_ctl, after the update the kernel logs the loss at loss_log[t - ctl[AP_PL_TRAIN0]]
   * (t = ctl[AP_CTL_TRAIN]), records the first non-finite loss in ctl[AP_PL_LOSS_BAD],
   * advances ctl[AP_CTL_TRAIN], and when (t + 1) % sync_every == 0 copies
   * sync_src[k][:sync_count[k]] -> sync_dst[k] (the target sync, agent.py:142-144, 335-337) */
  int64_t* tail_ctl;
  float* loss_log;
  int64_t loss_cap;
  int32_t sync_every;
  int32_t sync_n;           /* <= 6 segments */
  const float* sync_src[6];
  float* sync_dst[6];
  int64_t sync_count[6];
  double* r_scaled;         /* optional [cap]: r_scaled[idx] = (|td| + 1e-6) ** per_alpha with each priority */
  double* pstat;            /* with r_scaled: [2] the ring's max priority after the update, its ** per_alpha */
  double per_alpha;
  int32_t lazy_wt0;         /* 1: leave the first layer's transposed copy stale (no fused kernel reads
                               it; the caller refreshes it, e.g. after a device-loop launch) */
  const uint64_t* rng_from; /* optional (tail mode): copied to rng_to (6 words) when the step learns */
  uint64_t* rng_to;
} ap_fused_learn;

int64_t ap_mlp_fused_workspace(int32_t L, const int32_t* dims, int32_t rows, int32_t forward_only);
int ap_dqn_learn_fused(const ap_fused_learn* args, void* stream);
/* Q [rows, A] of the online network for rows x [rows, ldx] (rows <= 256), same kernel
 * in forward mode: the act of the search loop. */
int ap_mlp_forward_fused(int32_t L, const int32_t* dims, const int64_t* w_off, const int64_t* b_off,
                         const float* params, const float* x, int64_t ldx, int32_t rows, float* q,
                         float* workspace, uint32_t* barrier, void* stream);

/* agent.act of the parity loop in one launch: Q of the loop's state row (the fused forward,
 * which for <= 4 rows and <= 7 actions splits every layer's K over the grid) and the
 * epsilon-greedy decision of ap_parity_act on it (params: the online network). */
int ap_parity_act_fused(const ap_parity_loop* L, int32_t hidden_layers, const int32_t* dims, const int64_t* w_off,
                        const int64_t* b_off, const float* params, float* q_dev, float* workspace,
                        uint32_t* barrier, int32_t* action_dev, void* stream);

typedef struct ap_loop* ap_loop_t;
/* Outer graph: WHILE(episodes < budget && steps < max_steps) { step_graph;
 * IF(ring size >= batch) { learn_graph } }.  The graphs (cudaGraph_t) are
 * cloned as child graphs. */
int ap_loop_graph_create(void* step_graph, void* learn_graph, const int64_t* ctl, int64_t batch, ap_loop_t* out);
int ap_loop_graph_launch(ap_loop_t loop, void* stream);
int ap_loop_graph_destroy(ap_loop_t loop);

const char* ap_last_error(void);
const char* ap_version(void);

#ifdef __cplusplus
}
#endif

#endif /* AUTOPLAN_B200_H */
