"""Pin the pipeline-cost oracle (oracle/pipecost_oracle.py) on the reference goldens."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import pipecost_oracle as po
from paper_2007_04069_b200.ir import forward_subgraph, graph_from_dict

GOLDEN = Path(__file__).resolve().parent / "golden"
PIPES = sorted(p.stem[len("pipe_"):] for p in GOLDEN.glob("pipe_*.npz"))
INFERS = sorted(p.stem[len("infer_"):] for p in GOLDEN.glob("infer_*.npz"))


def load(kind, name):
    z = np.load(GOLDEN / f"{kind}_{name}.npz", allow_pickle=False)
    return {k: z[k] for k in z.files}


def graph_of(d):
    return graph_from_dict(json.loads(bytes(d["graph_json"]).decode()))


@pytest.mark.parametrize("name", PIPES)
def test_oracle_stage_metrics_and_length(name):
    d = load("pipe", name)
    g = graph_of(d)
    order = forward_subgraph(g)
    ns, gps, intra, inter = d["topo"]
    topo = po.topo_dict(ns, gps, intra, inter)
    mem = float(d["mem"][0])
    for r in range(len(d["metric_K"])):
        K, M = int(d["metric_K"][r]), int(d["metric_M"][r])
        piv = [order[p] for p in d["metric_piv"][r][: K - 1]]
        m = po.stage_metrics(g, piv)
        vals = d["metric_vals"][r][:K]
        assert [x[:3] for x in m] == [tuple(v[:3]) for v in vals]
        assert [x[3] for x in m] == [int(v[3]) for v in vals]
        counts = po.proportional_counts([x[0] for x in m], topo["d"])
        cuts = [int(x) for x in np.cumsum(counts)[:-1]]  # Python ints, as proportional_device_cuts builds them
        assert cuts == list(d["metric_cuts"][r][: K - 1])
        assert po.pipeline_length(m, cuts, M, topo) == d["metric_len"][r]
        if mem >= 0:
            assert po.memory_feasible(m, cuts, M, topo, mem) == bool(d["metric_feas"][r])


@pytest.mark.parametrize("dist,seed", [("uniform", 11), ("normal", 12), ("binomial", 13)])
def test_dataproc_matches_reference_arrays(dist, seed):
    from paper_2007_04069_b200.dataproc import generate_environment

    d = load("infer", f"gen_{dist}_configa")
    arr = generate_environment(dist, 1280, seed)
    np.testing.assert_array_equal(np.concatenate([arr.c, arr.a, arr.w]), d["arrays"])


@pytest.mark.parametrize("name", INFERS)
def test_oracle_infer_lengths(name):
    d = load("infer", name)
    G = 128
    arr = d["arrays"]
    c, a, w = arr[:G], arr[G:2 * G], arr[2 * G:]
    ns, gps, intra, inter = d["topo"]
    topo_n = po.topo_dict(ns, gps, 1.0, inter / intra)
    K, M, _ = (int(x) for x in d["meta"])
    for b, cu, ln in zip(d["pts_b"], d["pts_c"], d["lens"]):
        assert po.decode_length(c, a, w, list(b), list(cu), M, topo_n) == ln
    best = max(po.decode_length(c, a, w, list(d["best_b"]), list(d["best_c"]), M, topo_n), 1e-12)
    assert best == d["best_len"][0]


def test_pcg64_state_words_restate_numpy_stream():
    """dataproc.pcg64_states packs default_rng(seed)'s PCG64 state; stepping it with the XSL-RR
    output (the device generator's algorithm, csrc/dataplane.cu) reproduces numpy's uniform draws,
    also after a jump-ahead (PCG advance)."""
    import numpy as np

    from paper_2007_04069_b200.dataproc import pcg64_states

    M = 0x2360ED051FC65DA44385DF649FCCF645
    mask = (1 << 128) - 1

    def advance(state, inc, delta):
        cm, cp, am, ap = M, inc, 1, 0
        while delta:
            if delta & 1:
                am, ap = (am * cm) & mask, (ap * cm + cp) & mask
            cp, cm = ((cm + 1) * cp) & mask, (cm * cm) & mask
            delta >>= 1
        return (am * state + ap) & mask

    def draw(state, inc):
        state = (state * M + inc) & mask
        x = ((state >> 64) ^ state) & ((1 << 64) - 1)
        rot = state >> 122
        r = ((x >> rot) | (x << ((64 - rot) % 64))) & ((1 << 64) - 1)
        return state, (r >> 11) * (1.0 / 9007199254740992.0)

    for seed in (0, 7, 20201007):
        w = [int(v) for v in pcg64_states([seed])[0]]
        state, inc = (w[0] << 64) | w[1], (w[2] << 64) | w[3]
        ref = np.random.default_rng(seed).uniform(0.0, 1.0, 40)
        s = state
        for k in range(40):
            s, x = draw(s, inc)
            assert x == ref[k]
        s = advance(state, inc, 33)
        assert draw(s, inc)[1] == ref[33]
