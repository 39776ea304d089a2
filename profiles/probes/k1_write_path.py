"""K1 write-path probe: per-lane streaming stores vs TMA bulk row stores (AP_K1_BULK=1), and the
slot output in HBM allocated as compressible memory (cuMemCreate with
CU_MEM_ALLOCATION_COMP_GENERIC) vs cudaMalloc.  BERT-48, the bench's headline batch.

    python profiles/probes/k1_write_path.py [--batch 4194304] [--launches 20]
"""

import argparse
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2007_04069_b200 import graphs  # noqa: E402
from paper_2007_04069_b200.ir import decision_dims  # noqa: E402
from paper_2007_04069_b200.sharding import PropagationEngine  # noqa: E402
from paper_2007_04069_b200.workloads import prefix_seed_batch  # noqa: E402


class DevBuf:
    """A raw device allocation with the tensor attributes launch() reads."""

    def __init__(self, ptr, rows, stride):
        self.ptr, self.shape, self._stride = ptr, (rows, stride), stride

    def data_ptr(self):
        return self.ptr

    def stride(self, dim=0):
        return self._stride if dim == 0 else 1


def compressible(nbytes):
    import cuda.bindings.driver as drv

    def ok(r):
        err = r[0] if isinstance(r, tuple) else r
        if err != drv.CUresult.CUDA_SUCCESS:
            raise RuntimeError(str(err))
        return r[1] if isinstance(r, tuple) and len(r) > 1 else None

    ok(drv.cuInit(0))
    dev = ok(drv.cuDeviceGet(torch.cuda.current_device()))
    sup = ok(drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, dev))
    prop = drv.CUmemAllocationProp()
    prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = torch.cuda.current_device()
    prop.allocFlags.compressionType = drv.CUmemAllocationCompType.CU_MEM_ALLOCATION_COMP_GENERIC
    gran = ok(drv.cuMemGetAllocationGranularity(prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
    size = (nbytes + gran - 1) // gran * gran
    h = ok(drv.cuMemCreate(size, prop, 0))
    got = ok(drv.cuMemGetAllocationPropertiesFromHandle(h))
    ptr = ok(drv.cuMemAddressReserve(size, 0, 0, 0))
    ok(drv.cuMemMap(ptr, size, 0, h, 0))
    acc = drv.CUmemAccessDesc()
    acc.location = prop.location
    acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    ok(drv.cuMemSetAccess(ptr, size, [acc], 1))
    return int(ptr), bool(sup), int(got.allocFlags.compressionType)


def time_k1(eng, seeds, slots, launches, label):
    B = seeds.shape[0]
    oc = torch.empty(B, dtype=torch.uint8, device="cuda")
    cnt = torch.empty((B, 4), dtype=torch.int32, device="cuda")
    for _ in range(3):
        eng.launch(seeds, oc, cnt, slots)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(launches):
        eng.launch(seeds, oc, cnt, slots)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / launches
    n, S = len(eng.candidates), eng._eng.num_slots
    gbs = B * (n + S + 17) / ms / 1e6
    print(f"{label:48s} {ms:7.3f} ms  {B / ms / 1e3:8.1f} M plans/s  {gbs:7.1f} GB/s algorithmic", flush=True)
    return oc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1 << 22)
    ap.add_argument("--launches", type=int, default=20)
    a = ap.parse_args()
    g = graphs.generate("bert48")
    dims = decision_dims(g, g.trainable_variables)
    order = np.load(ROOT / "tests" / "golden" / "linkage_bert48.npz")["order"]
    eng = PropagationEngine(g, dims)
    B = a.batch
    seeds = prefix_seed_batch(order, 0, B, device="cuda", chunk=1 << 18)
    plain = torch.empty((B, eng.slots_stride), dtype=torch.int8, device="cuda")
    ref_oc = time_k1(eng, seeds, plain, a.launches, "cudaMalloc slots, per-lane st.global.cs")
    os.environ["AP_K1_BULK"] = "1"
    time_k1(eng, seeds, plain, a.launches, "cudaMalloc slots, TMA bulk row stores")
    os.environ["AP_K1_BULK"] = "0"
    ref_rows = plain[:4096].clone()
    del plain
    torch.cuda.empty_cache()
    ptr, sup, ctype = compressible(B * eng.slots_stride)
    print(f"generic compression supported={sup} allocation compressionType={ctype}")
    buf = DevBuf(ptr, B, eng.slots_stride)
    time_k1(eng, seeds, buf, a.launches, "compressible slots, per-lane st.global.cs")
    os.environ["AP_K1_BULK"] = "1"
    time_k1(eng, seeds, buf, a.launches, "compressible slots, TMA bulk row stores")
    os.environ["AP_K1_BULK"] = "0"
    view = torch.empty((4096, eng.slots_stride), dtype=torch.int8, device="cuda")
    import cuda.bindings.driver as drv

    drv.cuMemcpyDtoD(view.data_ptr(), ptr, view.numel())
    torch.cuda.synchronize()
    print("compressible rows equal plain rows:", bool(torch.equal(view, ref_rows)))


if __name__ == "__main__":
    main()
