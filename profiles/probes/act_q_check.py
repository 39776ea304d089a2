"""The loop's fused act on a full and a reduced grid against the host forward (same barrier buffer)."""
import sys, ctypes
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2007_04069_b200 import _native
from paper_2007_04069_b200.agent import QNetwork
from paper_2007_04069_b200.devloop import _rng_words
net = QNetwork(9, 2, (32, 32), np.random.default_rng(0))
x = torch.randn((1, 9), dtype=torch.float32, device="cuda")
q0 = net.forward_fused(x).clone()
ws, bar = net._fused_scratch(256, True)
Lh, dims, w_off, b_off = net.fused_layout()[:4]
lib = _native.require_device()
for early in (0, 1, 0, 1):
    t = {"ctl": torch.zeros(_native.PL["WORDS"], dtype=torch.int64, device="cuda"), "rng": torch.zeros(6, dtype=torch.int64, device="cuda")}
    t["ctl"][_native.PL["BUDGET"]] = 1; t["ctl"][_native.PL["MAX_STEPS"]] = 1; t["ctl"][_native.PL["TRAIN"]] = 10**6; t["ctl"][_native.PL["ACK"]] = 1
    g = np.random.default_rng(5); t["rng"].copy_(torch.from_numpy(_rng_words(g.bit_generator.state)))
    seeds = torch.full((16,), -1, dtype=torch.int8, device="cuda"); st = seeds.clone()
    log = torch.zeros(4, dtype=torch.int32, device="cuda")
    d = _native.ParityLoopDesc()
    d.ctl, d.rng, d.state, d.num_actions, d.ld = t["ctl"].data_ptr(), t["rng"].data_ptr(), x.data_ptr(), 2, 16
    d.seeds, d.seeds_try, d.decided = seeds.data_ptr(), st.data_ptr(), seeds.data_ptr()
    d.log_action, d.log_pos = log.data_ptr(), log.data_ptr()
    d.eps_start, d.eps_final, d.eps_decay = 1.0, 0.05, 100
    d.early_sample = early
    q = torch.zeros((1, 2), dtype=torch.float32, device="cuda"); a = torch.zeros(1, dtype=torch.int32, device="cuda")
    _native.check(lib.ap_parity_act_fused(ctypes.byref(d), Lh, dims, w_off, b_off, _native.ptr(net.flat), _native.ptr(q), _native.ptr(ws), _native.ptr(bar), _native.ptr(a), None))
    torch.cuda.synchronize()
    print(early, q.tolist(), q0.tolist(), net.forward_fused(x).tolist(), net.forward_device(x).tolist(), flush=True)
