"""The drop-in boundary, exercised with the REFERENCE's own objects (baseline/_ref).

The reference planner (`autoplan`, installed unmodified into baseline/_ref, which travels
to the GPU box) builds its own HloGraph / DimIndex / DimStatus / DeviceTopology objects;
they go straight into this package's entry points, and into the reference-side ctypes
binding of integration/autoplan_b200_binding.py (the FFI a maintainer would add to the
reference, no import of this package), and the answers are the reference's.

CPU: ir.flatten + ap_graph_create over reference graphs give the same compiled tables as
over our own parse of the same JSON; the binding's compile_graph agrees.
GPU: propagate / PropagationEngine.run, OppEnv, AdpEnv and PipeTrainEnv driven by
reference objects == the reference's results; the binding == reference PropagationEngine.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
if REF.exists() and str(REF) not in sys.path:
    sys.path.append(str(REF))
autoplan = pytest.importorskip("autoplan", reason="reference not installed in baseline/_ref")
from autoplan import zoo  # noqa: E402
from autoplan.ir import decision_dims as ref_decision_dims  # noqa: E402
from autoplan.sharding import DimStatus as RefStatus  # noqa: E402
from autoplan.sharding import PropagationEngine as RefEngine  # noqa: E402

sys.path.insert(0, str(ROOT / "integration"))

from paper_2007_04069_b200 import _native, graphs  # noqa: E402
from paper_2007_04069_b200.ir import flatten, graph_from_dict  # noqa: E402


def ref_graphs():
    from autoplan.ir import graph_from_dict as ref_from_dict

    return {
        "attention_block": zoo.attention_block(),
        "t5_block": zoo.t5_block(),
        "vgg_classifier": zoo.vgg_classifier(),
        "uniform_chain": zoo.uniform_chain(length=12),
        "bert_base": ref_from_dict(graphs.generate("bert_base").to_dict()),
    }


@pytest.mark.parametrize("name", sorted(ref_graphs()))
def test_reference_graph_compiles_like_ours(name):
    rg = ref_graphs()[name]
    ours = graph_from_dict(rg.to_dict())
    a = _native.DeviceGraph(flatten(rg)).export()
    b = _native.DeviceGraph(ours.flat()).export()
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    import autoplan_b200_binding as binding

    h, instrs, offs = binding.compile_graph(rg)
    assert int(offs[-1]) == len(a["class_of_slot"])
    binding.lib().ap_graph_destroy(h)


def _rand_seeds(rng, dims, k):
    pick = rng.permutation(len(dims))[:k]
    return {dims[j]: (RefStatus.PARTITIONED if rng.random() < 0.5 else RefStatus.REPLICATED) for j in pick}


def _same(a, b):
    assert a.outcome.name == b.outcome.name
    assert a.conflict_site == b.conflict_site
    assert [(d.flat_index, int(s)) for d, s in a.newly_decided] == [(d.flat_index, int(s)) for d, s in b.newly_decided]
    assert {i: tuple(s.statuses) for i, s in a.assignments.items()} == \
           {i: tuple(s.statuses) for i, s in b.assignments.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(ref_graphs()))
def test_propagate_takes_reference_objects(cuda, name):
    from paper_2007_04069_b200.sharding import PropagationEngine, propagate

    rg = ref_graphs()[name]
    names = rg.trainable_variables or [i.name for i in rg.instructions if i.opcode == "parameter"]
    dims = ref_decision_dims(rg, names)
    ref, ours = RefEngine(rg, dims), PropagationEngine(rg, dims)
    rng = np.random.default_rng(3)
    for _ in range(40):
        seeds = _rand_seeds(rng, dims, int(rng.integers(1, len(dims) + 1)))
        _same(ours.run(seeds), ref.run(seeds))
    seeds = _rand_seeds(rng, dims, 2)
    _same(propagate(rg, seeds), autoplan.propagate(rg, seeds))  # candidates from the seeded tensors


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["attention_block", "t5_block", "vgg_classifier", "uniform_chain"])
def test_reference_side_binding_matches_reference(cuda, name):
    import autoplan_b200_binding as binding

    rg = ref_graphs()[name]
    names = rg.trainable_variables or [i.name for i in rg.instructions if i.opcode == "parameter"]
    dims = ref_decision_dims(rg, names)
    ours, ref = binding.B200PropagationEngine(rg, dims), RefEngine(rg, dims)
    rng = np.random.default_rng(11)
    for _ in range(48):
        seeds = _rand_seeds(rng, dims, int(rng.integers(1, len(dims) + 1)))
        _same(ours.run(seeds), ref.run(seeds))
    ours.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name,task", [("attention_block", "opp"), ("t5_block", "opp"), ("vgg_classifier", "adp")])
def test_partition_envs_take_reference_graphs(cuda, name, task):
    from autoplan.envs import AdpEnv as RefAdp
    from autoplan.envs import OppEnv as RefOpp

    from paper_2007_04069_b200.envs import AdpEnv, OppEnv

    rg = ref_graphs()[name]
    ours = OppEnv(rg) if task == "opp" else AdpEnv(rg)
    ref = RefOpp(rg) if task == "opp" else RefAdp(rg)
    rng = np.random.default_rng(5)
    for _ in range(12):
        np.testing.assert_array_equal(ours.reset(), ref.reset())
        while not ref.done:
            a = int(rng.integers(2))
            r1, r2 = ours.step(a), ref.step(a)
            np.testing.assert_array_equal(r1.next_state, r2.next_state)
            assert (r1.reward, r1.done) == (r2.reward, r2.done)
            np.testing.assert_array_equal(ours.action_mask(), ref.action_mask())
        assert ours.done


@pytest.mark.gpu
def test_pipe_train_env_takes_reference_graph_and_topology(cuda):
    from autoplan.envs import PipeTrainEnv as RefPipe
    from autoplan.topology import PRESETS as REF_PRESETS

    from paper_2007_04069_b200.envs import PipeTrainEnv

    rg = zoo.uniform_chain()
    topo = REF_PRESETS["configa"]
    for K in (2, 3):
        ours, ref = PipeTrainEnv(rg, topo, K, radius=3), RefPipe(rg, topo, K, radius=3)
        rng = np.random.default_rng(K)
        for _ in range(3):
            np.testing.assert_array_equal(ours.reset(), ref.reset())
            while not ref.done:
                allowed = np.flatnonzero(ref.action_mask())
                np.testing.assert_array_equal(np.flatnonzero(ours.action_mask()), allowed)
                a = int(allowed[rng.integers(len(allowed))])
                r1, r2 = ours.step(a), ref.step(a)
                np.testing.assert_array_equal(r1.next_state, r2.next_state)
                assert (r1.reward, r1.done) == (r2.reward, r2.done)
