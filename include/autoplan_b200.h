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

const char* ap_last_error(void);
const char* ap_version(void);

#ifdef __cplusplus
}
#endif

#endif /* AUTOPLAN_B200_H */
