"""Round-2 fixtures: the BASELINE configs pinned to the reference (tests/golden/make_goldens_r2.py).

CPU (oracle + host logic):
* linkage groups / decision order of every linkage golden, including BERT-48 and T5-large,
  recomputed through the C oracle (linkage.py:43-83);
* the linkage cache file: our load_cache reads the reference's file and our save_cache writes
  it back byte for byte (linkage.py:94-128);
* the synthetic generators still produce the graphs the search goldens were run on (content hash,
  ir.py:412-414);
* validate_payload branches that return before any device work (cli.py:409-484).
GPU:
* free-running OPP / ADP searches with the finetune stage on MLP2, BERT-base and VGG-19
  (cli.py:193-248, :504-511; envs.py:110-130, :223-230): per-step digests, actions, rewards,
  best plans of both stages, the agent's RNG state afterwards;
* trace replay of the same runs (deterministic env functions only);
* validate_payload on every recorded payload.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from goldens import GOLDEN, linkage_names, load_linkage
from oracle import oracle
from paper_2007_04069_b200 import graphs
from paper_2007_04069_b200.ir import DimIndex
from paper_2007_04069_b200.linkage import LinkageGroup, load_cache, save_cache
from paper_2007_04069_b200.sharding import DimStatus

SEARCHES = sorted(p.stem[len("search_"):] for p in GOLDEN.glob("search_*.json")
                  if "graph_generator" in json.loads(p.read_text()))
VALIDATE = json.loads((GOLDEN / "validate.json").read_text())["cases"]


def _dims(f):
    pos = {int(i): p for p, i in enumerate(f.flat.ids)}
    return [DimIndex(k, i, d) for k, (i, d) in enumerate(f.cand)], pos


# -- CPU --------------------------------------------------------------------------


@pytest.mark.parametrize("name", linkage_names())
def test_oracle_linkage_matches_reference(name):
    """2|D| single-seed triggers through the C oracle -> groups, infeasible flags, decision order."""
    f = load_linkage(name)
    n = len(f.cand)
    trig = np.full((2 * n, n), -1, np.int8)
    trig[2 * np.arange(n), np.arange(n)] = 1  # row 2k: dim k PARTITIONED
    trig[2 * np.arange(n) + 1, np.arange(n)] = 0  # row 2k+1: dim k REPLICATED
    state, outcome, _ = oracle.propagate_batch(f.flat, f.cand_slots, trig, f.cand_slots)
    cand = state[:, f.cand_slots]
    infeasible = outcome == 2
    np.testing.assert_array_equal(infeasible.astype(np.uint8), f["infeasible"])
    implied = np.where((trig == -1) & ~infeasible[:, None], cand, -1).astype(np.int8)
    np.testing.assert_array_equal(implied, f["implied"])
    size = (implied != -1).sum(1).reshape(n, 2).max(1)
    order = sorted(range(n), key=lambda k: (-size[k], k))
    np.testing.assert_array_equal(order, f["order"])


@pytest.mark.parametrize("name", ["mlp2", "vgg19"])
def test_linkage_cache_reads_and_writes_reference_file(name, tmp_path):
    ref = GOLDEN / f"linkage_cache_{name}.json"
    g = graphs.generate(name)
    groups = load_cache(str(ref), g)
    assert groups is not None and len(groups) > 0
    for (d, st), grp in groups.items():
        assert isinstance(grp, LinkageGroup) and grp.trigger == (d, st)
    out = tmp_path / "cache.json"
    save_cache(str(out), g, groups)
    assert out.read_bytes() == ref.read_bytes()
    # a cache built for another graph is ignored (linkage.py:117-119); unreadable files too
    assert load_cache(str(ref), graphs.generate("bert_base")) is None
    (tmp_path / "bad.json").write_text("{not json")
    assert load_cache(str(tmp_path / "bad.json"), g) is None
    assert load_cache(str(tmp_path / "missing.json"), g) is None


@pytest.mark.parametrize("name", SEARCHES)
def test_search_golden_graph_is_the_generator_graph(name):
    rec = json.loads((GOLDEN / f"search_{name}.json").read_text())
    assert graphs.generate(rec["graph_generator"]).content_hash() == rec["graph_hash"]


def _payload_context(case):
    from paper_2007_04069_b200.topology import PRESETS, DeviceTopology

    ctx = case["context"]
    kw = {}
    if "graph" in ctx:
        kw["graph"] = graphs.generate(ctx["graph"])
    if "topo" in ctx:
        kw["topo"] = PRESETS[ctx["topo"]] if isinstance(ctx["topo"], str) else DeviceTopology(*ctx["topo"])
    if "arrays" in ctx:
        # the reference's build_environment_arrays(zoo.bert48_profile()), as recorded in the infer golden
        arr = np.load(GOLDEN / "infer_bert48_profile_configc.npz")["arrays"]

        class Arrays:
            c, a, w = arr[:128], arr[128:256], arr[256:]

        kw["arrays"] = Arrays
    for k in ("micro_batches", "micro_batch_size"):
        if k in ctx:
            kw[k] = ctx[k]
    return kw


HOST_ONLY = ("no_graph", "no_topo", "no_arrays", "unknown_task", "missing_key", "unknown_pivot")


@pytest.mark.parametrize("k", [k for k, c in enumerate(VALIDATE) if c["kind"] in HOST_ONLY])
def test_validate_payload_host_branches(k):
    from paper_2007_04069_b200.search import validate_payload

    case = VALIDATE[k]
    assert validate_payload(case["payload"], **_payload_context(case)) == (case["ok"], case["message"])


# -- GPU --------------------------------------------------------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(VALIDATE)))
def test_validate_payload_matches_reference(cuda, k):
    from paper_2007_04069_b200.search import validate_payload

    case = VALIDATE[k]
    assert validate_payload(case["payload"], **_payload_context(case)) == (case["ok"], case["message"])


def _run_search(rec):
    from paper_2007_04069_b200.agent import AgentConfig, DqnAgent
    from paper_2007_04069_b200.envs import AdpEnv, OppEnv
    from paper_2007_04069_b200.search import ListTrace, strategy_payload, train_partition

    g = graphs.generate(rec["graph_generator"])
    env = OppEnv(g) if rec["task"] == "opp" else AdpEnv(g)
    assert [d.flat_index for d in env.order] == rec["order"]
    agent = DqnAgent(AgentConfig(lr=rec["lr"], epsilon_decay_iters=rec["epsilon_decay"]), env.state_dim,
                     env.num_actions, rec["seed"])
    trace = ListTrace()
    best = stage1 = train_partition(env, agent, rec["episodes"], None, trace)
    stage2 = None
    if best is not None and rec["finetune_episodes"]:
        stage2 = train_partition(env, agent, rec["finetune_episodes"], None, trace, finetune_base=best.strategy,
                                 episode_offset=rec["episodes"])
        if stage2 is not None and (stage2.partitions, stage2.reward) > (best.partitions, best.reward):
            best = stage2

    def plan(o):
        return None if o is None else {"strategy": strategy_payload(g, o.strategy), "partitions": o.partitions,
                                       "reward": o.reward, "episode": o.episode}

    return trace.records, plan(stage1), plan(stage2), plan(best), agent


def _steps(records):
    return [(r["episode"], s["state_digest"], s["action"], s["reward"], r["outcome"])
            for r in records for s in r["steps"]]


@pytest.mark.gpu
@pytest.mark.parametrize("name", SEARCHES)
def test_search_free_running_with_finetune(cuda, name):
    """Identical trajectories and best plans of both stages (SURVEY §7 hard part 2, layer iii)."""
    rec = json.loads((GOLDEN / f"search_{name}.json").read_text())
    records, s1, s2, best, agent = _run_search(rec)
    assert _steps(records) == _steps(rec["trace"])
    assert s1 == rec["best_stage1"]
    assert s2 == rec["best_stage2"]
    assert best == rec["best"]
    assert agent.train_steps == rec["train_steps"]
    assert agent.rng.bit_generator.state == rec["rng_state"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", SEARCHES)
def test_search_trace_replay(cuda, name):
    """Replaying the reference's actions gives its digests and rewards bit for bit (layer ii),
    including finetune_reset starts from the recorded stage-1 plan."""
    from paper_2007_04069_b200.envs import AdpEnv, OppEnv
    from paper_2007_04069_b200.search import state_digest

    rec = json.loads((GOLDEN / f"search_{name}.json").read_text())
    g = graphs.generate(rec["graph_generator"])
    env = OppEnv(g) if rec["task"] == "opp" else AdpEnv(g)
    base = None
    if rec["best_stage1"] is not None:
        strat = rec["best_stage1"]["strategy"]
        base = {d: (DimStatus.PARTITIONED if strat[g.instruction(d.instruction_id).name] == d.dim
                    else DimStatus.REPLICATED) for d in env.dims}
    got = []
    for r in rec["trace"]:
        state = env.finetune_reset(base) if r["episode"] >= rec["episodes"] else env.reset()
        for s in r["steps"]:
            res = env.step(s["action"])
            got.append((r["episode"], state_digest(state), s["action"], res.reward))
            state = res.next_state
        assert env.done
    assert got == [(e, d, a, rw) for e, d, a, rw, _ in _steps(rec["trace"])]
