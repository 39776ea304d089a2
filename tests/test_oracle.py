"""Pin the CPU oracle against the reference's own outputs (tests/golden/).

The oracle (oracle/ap_oracle.c) restates the reference sweep algorithm; it
must reproduce every golden row exactly: outcome, every slot status
(including the schedule-dependent CONFLICT snapshot) and the conflict site.
"""

import math
import random

import numpy as np
import pytest

from goldens import load_prop, prop_names
from oracle import oracle


@pytest.mark.parametrize("name", prop_names())
def test_oracle_matches_reference(name):
    f = load_prop(name)
    state, outcome, site = oracle.propagate_batch(f.flat, f.cand_slots, f["seeds"], f.cand_slots)
    ids = f.flat.ids
    site_id = np.where(site >= 0, ids[np.maximum(site, 0)], -1)
    np.testing.assert_array_equal(outcome, f["outcome"])
    np.testing.assert_array_equal(state, f["slots"])
    np.testing.assert_array_equal(site_id, f["site"])


def test_oracle_newly_mask():
    """newly = candidates decided by propagation and not seeded (sharding.py:240-245)."""
    for name in ("linkage_chain", "two_layer", "t5_block", "bert_base"):
        f = load_prop(name)
        state, outcome, _ = oracle.propagate_batch(f.flat, f.cand_slots, f["seeds"], f.cand_slots)
        cand = state[:, f.cand_slots]
        newly = (cand != -1) & (f["seeds"] == -1) & (outcome[:, None] != 2)
        np.testing.assert_array_equal(newly.astype(np.int8), f["newly"])


def test_cpython_sum_restatement():
    rng = random.Random(7)
    for _ in range(20000):
        xs = [rng.choice([rng.random(), rng.random() * 1e12, 1e-9, 0.1, 1e16, -1e16, rng.uniform(-1, 1)])
              for _ in range(rng.randint(0, 9))]
        a, b = sum(xs), oracle.cpython_sum(xs)
        assert a == b and math.copysign(1, a) == math.copysign(1, b)
