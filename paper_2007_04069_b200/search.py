"""Search drivers: the reference episode loops and plan payloads.

`train_partition` / `train_pipe` keep the loop structure, draw order and
best-plan rules of the reference drivers (`cli.py:193-329`): act ->
step -> observe -> learn per step, best OPP/ADP strategy by lexicographic
(partitions, reward) with first-wins ties, best pipeline by strictly
shorter feasible length.  Plan payloads and their self-validation follow
`cli.py:384-484`, so emitted plan JSON is byte-identical for the same
trajectory.  The hot work inside each step runs on the GPU (propagation,
cost model, Q-network); `VecOppSearch` is the batched device driver for
throughput.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from typing import Callable, Mapping, Sequence

import numpy as np

from .agent import AgentConfig, DqnAgent, Transition
from .envs import AdpEnv, PartitionSearchEnv, PipeInferEnv, PipeTrainEnv, adp_candidates
from .ir import DimIndex, decision_dims
from .pipecost import PipelinePlan, StageMetrics, device_groups, pipeline_length, stage_metrics
from .sharding import DimStatus, Outcome, propagate

TASK_DEFAULTS: dict[str, dict[str, float | int]] = {
    "opp": {"lr": 0.0005, "epsilon_decay_iters": 2000, "episodes": 2000},
    "adp": {"lr": 0.0005, "epsilon_decay_iters": 500, "episodes": 500},
    "pp-train": {"lr": 0.001, "epsilon_decay_iters": 10000, "episodes": 500},
    "pp-infer": {"lr": 0.001, "epsilon_decay_iters": 10000, "episodes": 50},
}


def agent_config_for(task: str, gamma=None, lr=None, batch_size=None, buffer=None, epsilon_decay=None) -> AgentConfig:
    """Task defaults over AgentConfig defaults (cli.py:116-128)."""
    d = TASK_DEFAULTS.get(task, {})
    return AgentConfig(
        gamma=gamma if gamma is not None else 0.6,
        lr=lr if lr is not None else float(d.get("lr", 0.001)),
        batch_size=batch_size if batch_size is not None else 64,
        buffer_capacity=buffer if buffer is not None else 2000,
        epsilon_decay_iters=epsilon_decay if epsilon_decay is not None else int(d.get("epsilon_decay_iters", 2000)),
    )


def state_digest(state: np.ndarray) -> str:
    """sha256[:12] of the fp64 state bytes (cli.py:168-169): the trajectory-parity key."""
    return hashlib.sha256(np.asarray(state, dtype=np.float64).tobytes()).hexdigest()[:12]


@dataclass
class PartitionOutcome:
    strategy: dict[DimIndex, DimStatus]
    partitions: int
    reward: float
    episode: int


@dataclass
class PipeOutcome:
    plan: PipelinePlan
    metrics: list[StageMetrics]
    pipeline_length: float
    reward: float
    episode: int
    feasible: bool


def train_partition(env: PartitionSearchEnv, agent: DqnAgent, episodes: int, curve=None, trace=None,
                    finetune_base: Mapping[DimIndex, DimStatus] | None = None, episode_offset: int = 0,
                    stop_when: Callable[[PartitionOutcome], bool] | None = None) -> PartitionOutcome | None:
    """OPP / ADP episodes; best conflict-free strategy (cli.py:193-248)."""
    best: PartitionOutcome | None = None
    for ep in range(episodes):
        if finetune_base is not None:
            state = env.finetune_reset(finetune_base)
            if env.done:
                break
        else:
            state = env.reset()
        total = 0.0
        losses: list[float] = []
        steps: list[dict] = []
        conflict = False
        while not env.done:
            mask = env.action_mask()
            action = agent.act(state, mask)
            result = env.step(action)
            agent.observe(Transition(state, action, result.reward, result.next_state, result.done, env.action_mask()))
            loss = agent.learn()
            if loss is not None:
                losses.append(loss)
            if trace is not None:
                steps.append({"state_digest": state_digest(state), "action": action, "reward": result.reward})
            total += result.reward
            conflict = bool(result.info.get("conflict", False))
            state = result.next_state
        if not conflict:
            outcome = PartitionOutcome(env.strategy(), env.partition_count, total, episode_offset + ep)
            if best is None or (outcome.partitions, outcome.reward) > (best.partitions, best.reward):
                best = outcome
        if curve is not None:
            curve.write(episode_offset + ep, sum(losses) / len(losses) if losses else None, total, agent.epsilon)
        if trace is not None:
            trace.write(episode_offset + ep, steps, "conflict" if conflict else "complete")
        if stop_when is not None and best is not None and stop_when(best):
            break
    return best


def train_pipe(envs: Sequence[PipeTrainEnv | PipeInferEnv], agent: DqnAgent, episodes: int, curve=None, trace=None,
               episode_cap_per_env: int | None = None) -> list[PipeOutcome | None]:
    """Round-robin pipeline episodes; best feasible plan per env (cli.py:261-329)."""
    best: list[PipeOutcome | None] = [None] * len(envs)
    visits = [0] * len(envs)
    ep = 0
    for _ in range(episodes):
        open_envs = [i for i in range(len(envs)) if episode_cap_per_env is None or visits[i] < episode_cap_per_env]
        if not open_envs:
            break
        idx = open_envs[ep % len(open_envs)]
        env = envs[idx]
        visits[idx] += 1
        state = env.reset()
        total = 0.0
        losses = []
        steps: list[dict] = []
        final_info: dict = {}
        while not env.done:
            mask = env.action_mask()
            action = agent.act(state, mask)
            result = env.step(action)
            agent.observe(Transition(state, action, result.reward, result.next_state, result.done, env.action_mask()))
            loss = agent.learn()
            if loss is not None:
                losses.append(loss)
            if trace is not None:
                steps.append({"state_digest": state_digest(state), "action": action, "reward": result.reward})
            total += result.reward
            final_info = result.info
            state = result.next_state
        feasible = bool(final_info.get("memory_feasible", True))
        outcome = PipeOutcome(final_info["plan"], list(final_info["metrics"]), final_info["pipeline_length"], total, ep,
                              feasible)
        incumbent = best[idx]
        if feasible and (incumbent is None or outcome.pipeline_length < incumbent.pipeline_length):
            best[idx] = outcome
        if curve is not None:
            curve.write(ep, sum(losses) / len(losses) if losses else None, total, agent.epsilon)
        if trace is not None:
            trace.write(ep, steps, "complete")
        ep += 1
    return best


# -- plan payloads (cli.py:384-406, 524-534, 584-597, 647-661) -----------------------


def strategy_payload(graph, strategy: Mapping[DimIndex, DimStatus]) -> dict[str, int]:
    out: dict[str, int] = {}
    for d, status in strategy.items():
        name = graph.instruction(d.instruction_id).name
        out.setdefault(name, -1)
        if status == DimStatus.PARTITIONED:
            out[name] = d.dim
    return out


def stage_payload(metrics: Sequence[StageMetrics], plan: PipelinePlan, topo) -> list[dict]:
    return [
        {"compute_ms": m.compute_ms, "activation_bytes": m.activation_bytes, "param_bytes": m.param_bytes,
         "devices": e - s}
        for m, (s, e) in zip(metrics, device_groups(plan.device_cuts, topo.num_devices))
    ]


def validate_payload(payload: dict, graph=None, topo=None, arrays=None, micro_batches=None,
                     micro_batch_size=None) -> tuple[bool, str]:
    """Re-derive a plan from first principles on the device and compare (cli.py:409-484)."""
    task = payload.get("task")
    if task in ("opp", "adp"):
        if graph is None:
            return False, "sharding validation needs the graph"
        names = (list(graph.trainable_variables) if task == "opp"
                 else [graph.instruction(i).name for i in adp_candidates(graph)])
        dims = decision_dims(graph, names)
        strategy = payload.get("strategy", {})
        if set(strategy) != set(names):
            return False, "strategy keys do not match the candidate tensors"
        seeds = {d: (DimStatus.PARTITIONED if strategy[graph.instruction(d.instruction_id).name] == d.dim
                     else DimStatus.REPLICATED) for d in dims}
        result = propagate(graph, seeds, dims)
        if result.outcome is not Outcome.COMPLETE:
            return False, f"strategy does not propagate cleanly: {result.outcome.name}"
        if sum(1 for v in strategy.values() if v >= 0) != payload.get("partition_count"):
            return False, "partition_count does not match the strategy"
        return True, "strategy propagates conflict-free"
    if task == "pp-train":
        if graph is None or topo is None:
            return False, "pipeline validation needs the graph and topology"
        by_name = {graph.instruction(i).name: i for i in graph.topological_order}
        try:
            pivots = tuple(by_name[n] for n in payload["pivots"])
        except KeyError as exc:
            return False, f"unknown pivot {exc}"
        plan = PipelinePlan(pivots, tuple(payload["device_cuts"]),
                            micro_batches if micro_batches is not None else payload.get("micro_batches", 1),
                            micro_batch_size if micro_batch_size is not None else payload.get("micro_batch_size", 16))
        length = pipeline_length(plan, stage_metrics(graph, pivots), topo)
        if abs(length - payload.get("pipeline_length_s", -1.0)) > 1e-9 * max(1.0, length):
            return False, f"recomputed pipeline length {length} disagrees"
        return True, "pipeline length matches the cost model"
    if task == "pp-infer":
        if arrays is None or topo is None:
            return False, "inference validation needs the profile and topology"
        env = PipeInferEnv(arrays, topo, num_stages=len(payload["boundaries"]) + 1,
                           micro_batches=micro_batches if micro_batches is not None else payload.get("micro_batches", 1),
                           micro_batch_size=micro_batch_size if micro_batch_size is not None
                           else payload.get("micro_batch_size", 16))
        length = pipeline_length(PipelinePlan(tuple(payload["boundaries"]), tuple(payload["device_cuts"]),
                                              env.micro_batches, env.micro_batch_size),
                                 env.decode_metrics(payload["boundaries"]), env.topo_norm)
        if abs(length - payload.get("pipeline_length_s", -1.0)) > 1e-9 * max(1.0, length):
            return False, f"recomputed pipeline length {length} disagrees"
        return True, "pipeline length matches the cost model"
    return False, f"unknown plan task {task!r}"


def write_json(path: str, payload: dict) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(payload, sort_keys=True, indent=2) + "\n")


class TraceWriter:
    """JSON-lines episode traces (cli.py:153-165)."""

    def __init__(self, path: str):
        self._fh = open(path, "w", encoding="utf-8")

    def write(self, episode: int, steps: list[dict], outcome: str) -> None:
        self._fh.write(json.dumps({"episode": episode, "steps": steps, "outcome": outcome}, sort_keys=True) + "\n")
        self._fh.flush()

    def close(self) -> None:
        self._fh.close()


class ListTrace:
    """In-memory trace sink with the TraceWriter interface."""

    def __init__(self):
        self.records: list[dict] = []

    def write(self, episode: int, steps: list[dict], outcome: str) -> None:
        self.records.append({"episode": episode, "steps": steps, "outcome": outcome})
