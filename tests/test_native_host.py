"""Host-side checks of the C-ABI engine (no GPU needed).

* the in-tree library loads and exports every function include/*.h declares;
* the host rule compile (ap_graph_create -> ap_graph_export) yields link
  classes / forced classes / implication lists whose closure reproduces the
  reference on every golden row.  The closure is restated here in numpy
  (test code); on the GPU the same tables drive csrc/propagate.cu.
"""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from goldens import load_prop, prop_names
from paper_2007_04069_b200 import _native
from paper_2007_04069_b200.sharding import _forced_slot_list, graph_engine

HEADERS = sorted((Path(__file__).resolve().parents[1] / "include").glob("*.h"))


def declared_functions() -> set[str]:
    names = set()
    for h in HEADERS:
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"^\s*(?:int|int64_t|const char\*|void)\s+(ap_\w+)\s*\(", text, flags=re.M))
    return names


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    declared = declared_functions()
    assert len(declared) >= 9
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.SIGNATURES), "ctypes signature table out of sync with the header"
    assert lib.ap_version().decode().startswith("autoplan_b200")


def test_error_path_reports_message():
    lib = _native.load_library()
    handle = ctypes.c_void_p()
    rc = lib.ap_graph_create(None, ctypes.byref(handle))
    assert rc == _native.AP_ERR_INVALID
    assert b"descriptor" in lib.ap_last_error()


def closure_rows(tables, dec_class, dec_forced, first_same, seeds):
    """numpy restatement of the class closure."""
    C = len(tables["class_forced"])
    out_conf = np.zeros(len(seeds), bool)
    out_status = []
    for b, row in enumerate(seeds):
        P = np.zeros(C, bool)
        R = tables["class_forced"].astype(bool).copy()
        conf = False
        for j, v in enumerate(row):
            if v == 1:
                P[dec_class[j]] = True
            elif v == 0:
                R[dec_class[j]] = True
            elif v == 2 and (dec_forced[j] or (row[first_same[j]:j] == 1).any()):
                conf = True
        for c in np.flatnonzero(P):
            R[tables["imp_target"][tables["imp_offset"][c]:tables["imp_offset"][c + 1]]] = True
        out_conf[b] = conf or bool((P & R).any())
        out_status.append(np.where(P, 1, np.where(R, 0, -1)).astype(np.int8)[tables["class_of_slot"]])
    return out_conf, np.array(out_status)


@pytest.mark.parametrize("name", [n for n in prop_names() if not n.startswith("random_")] + ["random_000", "random_117"])
def test_compiled_tables_closure_matches_reference(name):
    f = load_prop(name)
    dev = _native.DeviceGraph(f.flat)
    tables = dev.export()
    forced = np.zeros(dev.num_slots, bool)
    forced[_forced_slot_list(graph_engine(f.graph))] = True
    owner = np.repeat(np.arange(f.flat.num_instructions), np.diff(f.flat.slot_offset))
    first_same = np.zeros(len(f.cand_slots), np.int64)
    for j in range(1, len(f.cand_slots)):
        same = owner[f.cand_slots[j]] == owner[f.cand_slots[j - 1]]
        first_same[j] = first_same[j - 1] if same else j
    conf, status = closure_rows(tables, tables["class_of_slot"][f.cand_slots], forced[f.cand_slots], first_same,
                                f["seeds"])
    np.testing.assert_array_equal(conf, f["outcome"] == 2)
    ok = ~conf
    np.testing.assert_array_equal(status[ok], f["slots"][ok])


def test_class_counts_bert48():
    """The closure's size on the headline graph (DESIGN.md records these)."""
    f = load_prop("bert48")
    dev = _native.DeviceGraph(f.flat)
    assert dev.num_slots == 5633
    assert 0 < dev.num_classes < 1024


def test_unpack_slots2_inverts_the_documented_packing():
    """unpack_slots2 decodes the ap_pack_slots2 layout (code = status + 1, slot j in bits 2*(j%4) of
    byte j/4), restated here with numpy, for ragged |S| and padded packed rows."""
    import numpy as np

    from paper_2007_04069_b200.sharding import unpack_slots2

    rng = np.random.default_rng(3)
    for n in (1, 4, 15, 16, 17, 5633):
        st = rng.integers(-1, 2, size=(9, n)).astype(np.int8)
        stride = max(4, (n + 15) // 16 * 4)
        codes = np.zeros((9, stride * 4), dtype=np.uint8)
        codes[:, :n] = (st + 1).astype(np.uint8)
        c = codes.reshape(9, stride, 4)
        packed = c[..., 0] | (c[..., 1] << 2) | (c[..., 2] << 4) | (c[..., 3] << 6)
        assert np.array_equal(unpack_slots2(packed, n), st)
