"""numpy's normal / binomial samplers restated for the device (csrc/np_samplers.cuh) and the
synthetic PP-infer environments they feed (reference dataproc.py:123-145).

CPU: the samplers, run on the host through ap_np_samples_host, reproduce numpy 2.3's
Generator.standard_normal (ziggurat, tables read from numpy's own libnpyrandom.a by
csrc/gen_np_ziggurat.py) and Generator.binomial(100, 0.5) (BTPE) draw for draw, and leave
the bit generator in numpy's state.
GPU: generate_environments_device("normal" | "binomial", n, seeds) equals the host
generate_environment bit for bit (short / long / non-multiple-of-G lengths) and the
reference's own arrays in tests/golden/infer_gen_*_configa.npz.
"""

import numpy as np
import pytest

from goldens import GOLDEN
from paper_2007_04069_b200 import _native
from paper_2007_04069_b200.devloop import _rng_words


@pytest.mark.parametrize("seed", [0, 1, 12, 13, 99991])
@pytest.mark.parametrize("kind", [0, 1])
def test_host_samplers_match_numpy(seed, kind):
    lib = _native.load_library()
    rng = np.random.default_rng(seed)
    rng.random()
    rng.integers(5)  # a buffered 32-bit half must not disturb the 64-bit draws
    words = _rng_words(rng.bit_generator.state).view(np.uint64).copy()
    N = 200000
    out = np.zeros(N)
    _native.check(lib.ap_np_samples_host(_native.ptr(words), kind, N, 100, 0.5, _native.ptr(out)))
    ref = rng.standard_normal(N) if kind == 0 else rng.binomial(100, 0.5, N).astype(np.float64)
    np.testing.assert_array_equal(out, ref)
    st = rng.bit_generator.state
    assert int(words[0]) << 64 | int(words[1]) == st["state"]["state"]


def test_host_binomial_other_parameters():
    """BTPE away from the reference's (100, 0.5): p > 0.5 mirrors, larger n reaches Step52."""
    lib = _native.load_library()
    for n, p in ((100, 0.7), (1000, 0.3), (5000, 0.5), (61, 0.5)):
        rng = np.random.default_rng(n)
        words = _rng_words(rng.bit_generator.state).view(np.uint64).copy()
        out = np.zeros(20000)
        _native.check(lib.ap_np_samples_host(_native.ptr(words), 1, out.size, n, p, _native.ptr(out)))
        np.testing.assert_array_equal(out, rng.binomial(n, p, out.size).astype(np.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("dist", ["normal", "binomial"])
@pytest.mark.parametrize("n", [1, 100, 128, 129, 1280])
def test_device_sampled_envs_match_host(cuda, dist, n):
    from paper_2007_04069_b200.dataproc import generate_environment, generate_environments_device

    seeds = list(range(40)) + [12, 13, 2 ** 31 + 5]
    out = generate_environments_device(dist, n, seeds).cpu().numpy()
    for k, s in enumerate(seeds):
        ref = generate_environment(dist, n, s)
        np.testing.assert_array_equal(out[k], np.stack([ref.c, ref.a, ref.w]), err_msg=f"{dist} n={n} seed={s}")


@pytest.mark.gpu
@pytest.mark.parametrize("dist,seed", [("normal", 12), ("binomial", 13), ("uniform", 11)])
def test_device_envs_match_reference_golden(cuda, dist, seed):
    from paper_2007_04069_b200.dataproc import generate_environments_device

    ref = np.load(GOLDEN / f"infer_gen_{dist}_configa.npz")["arrays"]
    out = generate_environments_device(dist, 1280, [seed]).cpu().numpy()[0].reshape(-1)
    np.testing.assert_array_equal(out, ref)
