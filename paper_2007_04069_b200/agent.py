"""Dueling double DQN with prioritized replay, device-resident.

Same public surface as reference `autoplan.agent` (`pkg/src/autoplan/agent.py:21-392`):
`AgentConfig`, `epsilon_at`, `QNetwork`, `masked_argmax`, `act`,
`Transition`, `PrioritizedReplayBuffer`, `AdamOptimizer`, `huber`,
`train_step`, `DqnAgent` (act / observe / learn / save / load), and the
same `.npz` checkpoint layout.

Where it runs:
* Q-network forward / backward contractions: tcgen05 tensor-core GEMMs
  (3xTF32, fp32-accurate) with bias + ReLU fused into the GEMM epilogue;
* dueling combine, TD / Huber / head gradients, ReLU backward, bias
  gradients, Adam, PER sampling and priority updates: fused kernels
  (`csrc/dqn.cu`);
* replay ring, both networks, Adam moments and priorities live in HBM;
  the target sync is a device copy.
Random draws come from the same `numpy.random.Generator` stream as the
reference (network init, epsilon-greedy, the uniforms behind `rng.choice`),
so with identical inputs the agent takes the same decisions; Q-values agree
with the fp64 reference within fp32 tolerance.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass
from typing import Sequence

import numpy as np

from . import _native
from .tc import gemm


def fork_to(side) -> None:
    """`side` waits for all work issued so far on the current stream (a graph fork under capture)."""
    import torch

    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream())
    side.wait_event(ev)


def join_from(side) -> None:
    """The current stream waits for `side` (a graph join under capture)."""
    import torch

    ev = torch.cuda.Event()
    ev.record(side)
    torch.cuda.current_stream().wait_event(ev)


def stream_or_current(side):
    import contextlib

    import torch

    return torch.cuda.stream(side) if side is not None else contextlib.nullcontext()


class CheckpointError(Exception):
    """A checkpoint file does not match the expected layout."""


class DivergenceError(Exception):
    """Training produced a non-finite loss."""


@dataclass(frozen=True)
class AgentConfig:
    gamma: float = 0.6
    lr: float = 0.001
    batch_size: int = 64
    buffer_capacity: int = 2000
    per_alpha: float = 0.2
    per_beta: float = 0.6
    target_sync_every: int = 100
    epsilon_start: float = 1.0
    epsilon_final: float = 0.1
    epsilon_decay_iters: int = 2000
    hidden: tuple[int, ...] = (256, 256)
    huber_delta: float = 1.0
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8


def epsilon_at(iteration: int, config: AgentConfig) -> float:
    """Linear decay from epsilon_start to epsilon_final (agent.py:50-55)."""
    if config.epsilon_decay_iters <= 0:
        return config.epsilon_final
    frac = min(1.0, max(0.0, iteration / config.epsilon_decay_iters))
    return config.epsilon_start + (config.epsilon_final - config.epsilon_start) * frac


def _stream():
    return _native.stream_handle()


class QNetwork:
    """Dueling MLP on the device: ReLU trunk, value head, advantage head.

    Parameters live in one flat fp32 buffer (views: w_i [fan_in, width],
    b_i, then the fused head wh = [wv | wa] [width, 1 + A] and bh).
    """

    def __init__(self, state_dim: int, num_actions: int, hidden: Sequence[int] = (256, 256),
                 rng: np.random.Generator | None = None, _init: bool = True):
        if state_dim < 1 or num_actions < 1:
            raise ValueError("state_dim and num_actions must be positive")
        if not hidden:
            raise ValueError("the trunk needs at least one hidden layer")
        import torch

        self.state_dim = state_dim
        self.num_actions = num_actions
        self.hidden = tuple(hidden)
        self.precision = 3  # 3xTF32 (fp32-accurate); the throughput trainer may set 1 (TF32)
        shapes = []
        fan_in = state_dim
        for i, width in enumerate(self.hidden):
            shapes += [(f"w{i}", (fan_in, width)), (f"b{i}", (width,))]
            fan_in = width
        shapes += [("wh", (fan_in, 1 + num_actions)), ("bh", (1 + num_actions,))]
        self._shapes = shapes
        total = sum(int(np.prod(s)) for _, s in shapes)
        self.flat = torch.zeros(total, dtype=torch.float32, device="cuda")
        self.grad = torch.zeros(total, dtype=torch.float32, device="cuda")
        self.views: dict[str, "torch.Tensor"] = {}
        self.grads: dict[str, "torch.Tensor"] = {}
        off = 0
        for name, shape in shapes:
            n = int(np.prod(shape))
            self.views[name] = self.flat[off: off + n].view(shape)
            self.grads[name] = self.grad[off: off + n].view(shape)
            off += n
        # [out, in] copies of every weight: the forward GEMMs then read both
        # operands K-major (the pipelined tcgen05 kernel); refreshed whenever
        # the parameters change
        # (rows padded to a 16-byte stride: the TMA-fed GEMM needs it for any fan-in)
        self.wt = {name: torch.empty((s[1], (s[0] + 3) // 4 * 4), dtype=torch.float32, device="cuda")[:, : s[0]]
                   for name, s in shapes if len(s) == 2}
        if _init:
            rng = rng or np.random.default_rng(0)
            params = {}
            fan_in = state_dim
            for i, width in enumerate(self.hidden):
                params[f"w{i}"] = self._init(rng, fan_in, width)
                params[f"b{i}"] = self._init(rng, fan_in, width, bias=True)
                fan_in = width
            params["wv"] = self._init(rng, fan_in, 1)
            params["bv"] = self._init(rng, fan_in, 1, bias=True)
            params["wa"] = self._init(rng, fan_in, num_actions)
            params["ba"] = self._init(rng, fan_in, num_actions, bias=True)
            self.load_params(params)

    @staticmethod
    def _init(rng, fan_in: int, width: int, bias: bool = False) -> np.ndarray:
        """Same draws as the reference initializer (agent.py:87-91)."""
        bound = 1.0 / np.sqrt(fan_in)
        return rng.uniform(-bound, bound, size=(width,) if bias else (fan_in, width)).astype(np.float64)

    # -- reference-layout parameter access -------------------------------------------

    @property
    def params(self) -> dict[str, np.ndarray]:
        """Host fp64 copies in the reference layout (w*, b*, wv, bv, wa, ba)."""
        out = {}
        for i in range(len(self.hidden)):
            out[f"w{i}"] = self.views[f"w{i}"].double().cpu().numpy()
            out[f"b{i}"] = self.views[f"b{i}"].double().cpu().numpy()
        wh = self.views["wh"].double().cpu().numpy()
        bh = self.views["bh"].double().cpu().numpy()
        out["wv"], out["wa"] = wh[:, :1].copy(), wh[:, 1:].copy()
        out["bv"], out["ba"] = bh[:1].copy(), bh[1:].copy()
        return out

    def load_params(self, params: dict[str, np.ndarray]) -> None:
        import torch

        for i in range(len(self.hidden)):
            self.views[f"w{i}"].copy_(torch.from_numpy(np.asarray(params[f"w{i}"])))
            self.views[f"b{i}"].copy_(torch.from_numpy(np.asarray(params[f"b{i}"])))
        wh = np.concatenate([np.asarray(params["wv"]), np.asarray(params["wa"])], axis=1)
        bh = np.concatenate([np.asarray(params["bv"]), np.asarray(params["ba"])])
        self.views["wh"].copy_(torch.from_numpy(wh))
        self.views["bh"].copy_(torch.from_numpy(bh))
        self.refresh_transposed()

    def adam_segments(self, skip_w0: bool = False):
        """Host descriptors for ap_dqn_adam_ctl_t: (n, flat offsets, rows, cols, transposed
        destinations, their row strides) of every weight matrix (cached; tensors never move).
        skip_w0: the layers after the first [in + 1, out] block (w0 and b0), offsets relative
        to that block's end -- the first layer's update is fused into its gradient GEMM."""
        import ctypes

        key = "_aseg_skip" if skip_w0 else "_aseg"
        if getattr(self, key, None) is None:
            names = list(self.wt)
            start = self.w0_block() if skip_w0 else 0
            if skip_w0:
                names = names[1:]
            n = len(names)
            base = self.flat.storage_offset() + start
            src = [self.views[k] for k in names]
            dst = [self.wt[k] for k in names]
            setattr(self, key, (
                n,
                (ctypes.c_int64 * n)(*[t.storage_offset() - base for t in src]),
                (ctypes.c_int32 * n)(*[t.shape[0] for t in src]),
                (ctypes.c_int32 * n)(*[t.shape[1] for t in src]),
                (ctypes.c_void_p * n)(*[t.data_ptr() for t in dst]),
                (ctypes.c_int64 * n)(*[t.stride(0) for t in dst]),
            ))
        return getattr(self, key)

    def w0_block(self) -> int:
        """Length of the leading [in + 1, out] block of the flat buffers (w0 then b0)."""
        w0 = self.views["w0"]
        assert w0.storage_offset() == self.flat.storage_offset(), "w0 leads the flat parameter buffer"
        return (w0.shape[0] + 1) * w0.shape[1]

    def refresh_transposed(self) -> None:
        """All transposed weight copies in one launch (ap_transpose_batch)."""
        import ctypes

        if getattr(self, "_tdesc", None) is None:  # descriptors: the tensors never move
            names = list(self.wt)
            n = len(names)
            src = [self.views[k] for k in names]
            dst = [self.wt[k] for k in names]
            self._tdesc = (
                n,
                (ctypes.c_void_p * n)(*[t.data_ptr() for t in src]),
                (ctypes.c_int64 * n)(*[t.stride(0) for t in src]),
                (ctypes.c_void_p * n)(*[t.data_ptr() for t in dst]),
                (ctypes.c_int64 * n)(*[t.stride(0) for t in dst]),
                (ctypes.c_int32 * n)(*[t.shape[0] for t in src]),
                (ctypes.c_int32 * n)(*[t.shape[1] for t in src]),
            )
        n, src, lds, dst, ldd, rows, cols = self._tdesc
        lib = _native.require_device()
        _native.check(lib.ap_transpose_batch(n, src, lds, dst, ldd, rows, cols, _stream()))

    # -- compute ----------------------------------------------------------------------

    def forward_device(self, x, cache: bool = False):
        """Q [B, A] for device states x [B, state_dim] fp32 (and the activations when cache)."""
        import torch

        acts = [x]
        h = x
        for i in range(len(self.hidden)):
            h = gemm(h, self.wt[f"w{i}"], trans_b=True, bias=self.views[f"b{i}"], relu=True, precision=self.precision)
            acts.append(h)
        b = x.shape[0]
        q = torch.empty((b, self.num_actions), dtype=torch.float32, device="cuda")
        lib = _native.require_device()
        wt = self.wt["wh"]
        if 1 + self.num_actions <= 8:  # narrow head: dot products + dueling in one warp-per-row kernel
            _native.check(lib.ap_dqn_head_forward(_native.ptr(h), h.stride(0), _native.ptr(wt), wt.stride(0),
                                                  _native.ptr(self.views["bh"]), b, h.shape[1],
                                                  1 + self.num_actions, _native.ptr(q), q.stride(0), _stream()))
        else:
            z = gemm(h, wt, trans_b=True, bias=self.views["bh"], precision=self.precision)
            _native.check(lib.ap_dqn_dueling(_native.ptr(z), z.stride(0), _native.ptr(q), q.stride(0), b,
                                             self.num_actions, _stream()))
        return (q, acts) if cache else q

    # -- fused small-batch path (csrc/fused_mlp.cu) -----------------------------------

    def fused_layout(self):
        """ctypes descriptors of the flat layout for the fused kernels (cached: tensors never move)."""
        import ctypes

        if getattr(self, "_flay", None) is None:
            L = len(self.hidden)
            names_w = [f"w{i}" for i in range(L)] + ["wh"]
            names_b = [f"b{i}" for i in range(L)] + ["bh"]
            base = self.flat.storage_offset()
            pad = [0] * (5 - (L + 1))
            dims = (ctypes.c_int32 * 6)(*([self.state_dim, *self.hidden, 1 + self.num_actions] + [0] * (4 - L)))
            w_off = (ctypes.c_int64 * 5)(*([self.views[k].storage_offset() - base for k in names_w] + pad))
            b_off = (ctypes.c_int64 * 5)(*([self.views[k].storage_offset() - base for k in names_b] + pad))
            wt = (ctypes.c_void_p * 5)(*([self.wt[k].data_ptr() for k in names_w] + [None] * len(pad)))
            wt_ld = (ctypes.c_int64 * 5)(*([self.wt[k].stride(0) for k in names_w] + pad))
            self._flay = (L, dims, w_off, b_off, wt, wt_ld)
        return self._flay

    def _fused_scratch(self, rows: int, forward_only: bool):
        """Per-network workspace + grid barrier of the fused kernels (grow-only; one stream at a time)."""
        import torch

        L, dims = self.fused_layout()[:2]
        need = int(_native.require_device().ap_mlp_fused_workspace(L, dims, rows, int(forward_only)))
        key = "_fws_f" if forward_only else "_fws_l"
        ws = self.__dict__.get(key)
        if ws is None or ws[0].numel() < need:
            ws = (torch.empty(need, dtype=torch.float32, device="cuda"), torch.zeros(4, dtype=torch.int32, device="cuda"))
            self.__dict__[key] = ws
        return ws

    def forward_fused(self, x, out=None):
        """Q [rows, A] for device states x [rows, state_dim] (rows <= 256): one persistent
        kernel (ap_mlp_forward_fused), fp32 CUDA-core tiles, grid barriers between layers."""
        import torch

        L, dims, w_off, b_off = self.fused_layout()[:4]
        rows = x.shape[0]
        q = out if out is not None else torch.empty((rows, self.num_actions), dtype=torch.float32, device="cuda")
        ws, bar = self._fused_scratch(256, True)
        _native.check(_native.require_device().ap_mlp_forward_fused(
            L, dims, w_off, b_off, _native.ptr(self.flat), _native.ptr(x), x.stride(0), rows, _native.ptr(q),
            _native.ptr(ws), _native.ptr(bar), _stream()))
        return q

    def forward(self, states) -> np.ndarray:
        import torch

        x = torch.as_tensor(np.atleast_2d(np.asarray(states, dtype=np.float64)), dtype=torch.float32).cuda()
        if x.shape[1] != self.state_dim:
            raise ValueError(f"expected state dim {self.state_dim}, got {x.shape[1]}")
        return self.forward_device(x).double().cpu().numpy()

    def backward_device(self, acts, dz, dz_t=None, side=None, dueling_td: bool = False, fused_w0_adam=None) -> bool:
        """Gradients into self.grad from dLoss/dz (z = [V, A] head outputs).

        `dz_t` (optional) is dz^T already materialised (ap_dqn_td_ring writes it).

        Weight gradients are K-major GEMMs contracting over the batch, dW = h^T dz
        (A = h^T [in, B], B-operand = dz^T [out, B]).  Each layer's activations are
        transposed into a ones-augmented [in + 1, B] buffer (all layers in one
        launch), and since b_i follows w_i in the flat buffer the GEMM writes the
        [in + 1, out] block [dW_i; db_i] at once: the bias gradient is the ones-row
        product, the column sum of dh (agent.py:118, 134).

        `dueling_td`: dz is the TD kernels' dueling gradient (one advantage entry
        differs from -g/A per row), so a wide head back-propagates in closed form
        (ap_dqn_head_backward_dueling).

        `fused_w0_adam` (dict: m, v, ctl, counter_advanced, lr, beta1, beta2, eps and an
        optional `wait` event): the first layer's weight-gradient GEMM also applies Adam to
        w0 / b0 and writes w0's transposed copy (ap_gemm_tf32_adam).  Returns True when it
        did; the caller's Adam then skips that block (adam_segments(skip_w0=True)).

        `side` (a CUDA stream): the weight-gradient GEMMs run there, a parallel
        branch beside the data-gradient chain (one graph branch under capture);
        joined back before returning.  Tensors read across streams stay
        referenced until the join, so the caching allocator cannot recycle them."""
        import ctypes

        import torch

        lib = _native.require_device()
        P = _native.ptr
        L = len(self.hidden)
        b = dz.shape[0]
        aug = self._augmented(b)
        n = L + 1
        keep = []
        fused = False
        if dz_t is None:
            dz_t = dz.t().contiguous()
        if side is not None:
            fork_to(side)
        with stream_or_current(side):
            # the ones-augmented activation transposes only feed the weight-gradient
            # GEMMs, so with a side stream they leave the data-gradient chain entirely
            _native.check(lib.ap_transpose_batch(
                n, (ctypes.c_void_p * n)(*[a.data_ptr() for a in acts]),
                (ctypes.c_int64 * n)(*[a.stride(0) for a in acts]), (ctypes.c_void_p * n)(*[t.data_ptr() for t in aug]),
                (ctypes.c_int64 * n)(*[t.stride(0) for t in aug]), (ctypes.c_int32 * n)(*[b] * n),
                (ctypes.c_int32 * n)(*[a.shape[1] for a in acts]), _stream()))
            gemm(aug[L], dz_t, trans_b=True, out=self._grad_block("wh"), precision=self.precision)
        # head -> last hidden layer: K = 1 + A is too narrow for the tensor cores;
        # one kernel does dz @ wh^T, the ReLU mask and the transposed copy
        h = acts[-1]
        wh = self.views["wh"]
        H = wh.shape[0]
        dh = torch.empty((b, H), dtype=torch.float32, device="cuda")
        dh_t = torch.empty((H, b), dtype=torch.float32, device="cuda")
        if dueling_td and dz.shape[1] > 32:
            rs = self.__dict__.get("_rowsum")
            if rs is None or rs.numel() < H:
                rs = self._rowsum = torch.empty(H, dtype=torch.float32, device="cuda")
            _native.check(lib.ap_dqn_head_backward_dueling(P(dz), dz.stride(0), P(wh), wh.stride(0), P(h), h.stride(0),
                                                           b, H, dz.shape[1], P(rs), P(dh), dh.stride(0), P(dh_t),
                                                           dh_t.stride(0), _stream()))
        else:
            _native.check(lib.ap_dqn_head_backward(P(dz), dz.stride(0), P(wh), wh.stride(0), P(h), h.stride(0), b, H,
                                                   dz.shape[1], P(dh), dh.stride(0), P(dh_t), dh_t.stride(0),
                                                   _stream()))
        for i in range(L - 1, -1, -1):
            if side is not None:
                fork_to(side)  # the branch waits for this layer's dh_t
                keep.append(dh_t)
            with stream_or_current(side):
                done = False
                if i == 0 and fused_w0_adam is not None:
                    fa = fused_w0_adam
                    if fa.get("wait") is not None:
                        torch.cuda.current_stream().wait_event(fa["wait"])
                    n0 = self.w0_block()
                    out = self._grad_block("w0")
                    wt0 = self.wt["w0"]
                    rc = lib.ap_gemm_tf32_adam(P(aug[0]), aug[0].stride(0), P(dh_t), dh_t.stride(0), P(out),
                                               out.stride(0), out.shape[0], out.shape[1], b, P(fa["m"]), P(fa["v"]),
                                               P(self.flat), P(fa["ctl"]), int(fa["counter_advanced"]),
                                               float(fa["lr"]), float(fa["beta1"]), float(fa["beta2"]),
                                               float(fa["eps"]), P(wt0), wt0.stride(0), out.shape[0] - 1, _stream())
                    if rc != _native.AP_ERR_UNSUPPORTED:
                        _native.check(rc)
                        done = fused = True
                    assert n0 == out.numel()
                if not done:
                    gemm(aug[i], dh_t, trans_b=True, out=self._grad_block(f"w{i}"), precision=self.precision)
            if i > 0:  # gradient into layer i-1's output: dh @ W_i^T, ReLU mask, K-major copy
                dh = gemm(dh, self.views[f"w{i}"], trans_b=True, precision=self.precision)
                hin = acts[i]
                dh_t = torch.empty((dh.shape[1], b), dtype=torch.float32, device="cuda")
                _native.check(lib.ap_dqn_relu_backward_t(P(dh), dh.stride(0), P(hin), hin.stride(0), b, dh.shape[1],
                                                         P(dh_t), dh_t.stride(0), _stream()))
        if side is not None:
            join_from(side)
        del keep
        return fused

    def _augmented(self, b: int):
        """Per-batch-size [in + 1, b] buffers (last row ones) for each layer's input."""
        import torch

        cache = self.__dict__.setdefault("_aug_cache", {})
        if b not in cache:
            ins = [self.state_dim, *self.hidden]
            bufs = []
            for w in ins:
                t = torch.empty((w + 1, b), dtype=torch.float32, device="cuda")
                t[w].fill_(1.0)
                bufs.append(t)
            cache[b] = bufs
        return cache[b]

    def _grad_block(self, wname: str):
        """The contiguous [in + 1, out] gradient block of weight `wname` and its bias."""
        g = self.grads[wname]
        return self.grad[g.storage_offset() - self.grad.storage_offset():][: (g.shape[0] + 1) * g.shape[1]].view(
            g.shape[0] + 1, g.shape[1])

    def forward_cached(self, states):
        import torch

        x = torch.as_tensor(np.atleast_2d(np.asarray(states, dtype=np.float64)), dtype=torch.float32).cuda()
        q, acts = self.forward_device(x, cache=True)
        return q.double().cpu().numpy(), {"acts": acts}

    def backward(self, cache: dict, dq: np.ndarray) -> dict[str, np.ndarray]:
        """Reference-layout gradients for dLoss/dQ (agent.py:111-136)."""
        import torch

        dq = np.asarray(dq, dtype=np.float64)
        dz = np.concatenate([dq.sum(axis=1, keepdims=True), dq - dq.sum(axis=1, keepdims=True) / self.num_actions],
                            axis=1)
        self.backward_device(cache["acts"], torch.from_numpy(dz).float().cuda().contiguous())
        out = {}
        for i in range(len(self.hidden)):
            out[f"w{i}"] = self.grads[f"w{i}"].double().cpu().numpy()
            out[f"b{i}"] = self.grads[f"b{i}"].double().cpu().numpy()
        gh = self.grads["wh"].double().cpu().numpy()
        gb = self.grads["bh"].double().cpu().numpy()
        out["wv"], out["wa"], out["bv"], out["ba"] = gh[:, :1], gh[:, 1:], gb[:1], gb[1:]
        return out

    def copy_from(self, other: "QNetwork") -> None:
        self.flat.copy_(other.flat)
        self.refresh_transposed()

    def clone(self) -> "QNetwork":
        twin = QNetwork(self.state_dim, self.num_actions, self.hidden, _init=False)
        twin.precision = self.precision
        twin.copy_from(self)
        return twin


def sync_target(net: QNetwork, target_net: QNetwork) -> None:
    """Hard device copy of the online parameters (agent.py:142-144)."""
    target_net.copy_from(net)


def masked_argmax(q: np.ndarray, mask: np.ndarray) -> int:
    """Highest allowed Q, ties to the lowest index (agent.py:147-152)."""
    if not mask.any():
        raise ValueError("no action is allowed")
    return int(np.argmax(np.where(mask, q, -np.inf)))


def act(net: QNetwork, state: np.ndarray, mask: np.ndarray, epsilon: float, rng: np.random.Generator) -> int:
    """Epsilon-greedy over the allowed set (agent.py:155-170), same draw order as the reference."""
    import torch

    mask = np.asarray(mask, dtype=bool)
    if not mask.any():
        raise ValueError("no action is allowed")
    if rng.random() < epsilon:
        allowed = np.flatnonzero(mask)
        return int(allowed[rng.integers(len(allowed))])
    x = torch.as_tensor(np.asarray(state, dtype=np.float64), dtype=torch.float32).cuda().view(1, -1)
    q = net.forward_fused(x) if getattr(net, "fused_act", False) else net.forward_device(x)
    m = torch.from_numpy(mask.astype(np.uint8)).cuda().view(1, -1)
    out = torch.empty(1, dtype=torch.int32, device="cuda")
    lib = _native.require_device()
    _native.check(lib.ap_dqn_act(_native.ptr(q), q.stride(0), _native.ptr(m), m.stride(0), 1, net.num_actions, 0.0, 0,
                                 _native.ptr(out), _stream()))
    return int(out.item())


@dataclass(frozen=True)
class Transition:
    state: np.ndarray
    action: int
    reward: float
    next_state: np.ndarray
    done: bool
    next_mask: np.ndarray


class PrioritizedReplayBuffer:
    """Device ring buffer with proportional prioritized sampling (agent.py:183-226)."""

    def __init__(self, capacity: int = 2000, state_dim: int | None = None, num_actions: int | None = None):
        if capacity < 1:
            raise ValueError("capacity must be positive")
        self.capacity = capacity
        self.state_dim = state_dim
        self.num_actions = num_actions
        self._size = 0
        self._next = 0
        self._store = None

    def _alloc(self, state_dim: int, num_actions: int) -> None:
        import torch

        c = self.capacity
        dev = "cuda"
        self.state_dim, self.num_actions = state_dim, num_actions
        self._store = {
            "states": torch.zeros((c, state_dim), dtype=torch.float32, device=dev),
            "next_states": torch.zeros((c, state_dim), dtype=torch.float32, device=dev),
            "actions": torch.zeros(c, dtype=torch.int32, device=dev),
            "rewards": torch.zeros(c, dtype=torch.float32, device=dev),
            "done": torch.zeros(c, dtype=torch.uint8, device=dev),
            "next_mask": torch.zeros((c, num_actions), dtype=torch.uint8, device=dev),
            "priorities": torch.zeros(c, dtype=torch.float64, device=dev),
            "scratch": torch.zeros(2 * c + 1024, dtype=torch.float64, device=dev),
        }

    def __len__(self) -> int:
        return self._size

    @property
    def store(self):
        return self._store

    def push(self, t: Transition) -> None:
        """Insert with the current maximum priority (agent.py:197-205)."""
        import torch

        if self._store is None:
            self._alloc(len(t.state), len(t.next_mask))
        s = self._store
        k = self._next
        s["states"][k].copy_(torch.as_tensor(np.asarray(t.state, np.float64), dtype=torch.float32))
        s["next_states"][k].copy_(torch.as_tensor(np.asarray(t.next_state, np.float64), dtype=torch.float32))
        s["actions"][k] = int(t.action)
        s["rewards"][k] = float(t.reward)
        s["done"][k] = int(bool(t.done))
        s["next_mask"][k].copy_(torch.as_tensor(np.asarray(t.next_mask, dtype=np.uint8)))
        self.push_priority(k)
        self._size = min(self._size + 1, self.capacity)
        self._next = (k + 1) % self.capacity

    def push_priority(self, slot: int) -> None:
        pr = self._store["priorities"]
        if self._size:
            pr[slot] = pr[: self._size].max()  # device-side, no sync
        else:
            pr[slot] = 1.0

    def sample_device(self, batch_size: int, alpha: float, beta: float, uniforms):
        """Indices [B] int32 and IS weights [B] fp32 on the device for the given uniforms."""
        import torch

        n = self._size
        if n < batch_size:
            raise ValueError("not enough transitions to sample a batch")
        s = self._store
        u = torch.as_tensor(uniforms, dtype=torch.float64).cuda()
        idx = torch.empty(batch_size, dtype=torch.int32, device="cuda")
        w = torch.empty(batch_size, dtype=torch.float32, device="cuda")
        if s["scratch"].numel() < 2 * n + batch_size:
            s["scratch"] = torch.zeros(2 * n + batch_size, dtype=torch.float64, device="cuda")
        lib = _native.require_device()
        _native.check(lib.ap_per_sample(_native.ptr(s["priorities"]), n, float(alpha), float(beta), _native.ptr(u),
                                        batch_size, _native.ptr(s["scratch"]), _native.ptr(idx), _native.ptr(w),
                                        _stream()))
        return idx, w

    def sample(self, batch_size: int, alpha: float, beta: float, rng: np.random.Generator):
        """(indices, None, weights) on the host; draws rng.random(B) exactly like rng.choice would."""
        u = rng.random(batch_size)
        idx, w = self.sample_device(batch_size, alpha, beta, u)
        return idx.cpu().numpy().astype(np.int64), None, w.double().cpu().numpy()

    def update_priorities_device(self, indices, td) -> None:
        lib = _native.require_device()
        _native.check(lib.ap_per_update(_native.ptr(self._store["priorities"]), _native.ptr(indices), _native.ptr(td),
                                        int(indices.numel()), _stream()))

    @property
    def priorities(self) -> np.ndarray:
        return self._store["priorities"][: self._size].cpu().numpy()


class AdamOptimizer:
    """Adam with bias correction over the network's flat buffer (agent.py:229-250)."""

    def __init__(self, net: QNetwork, config: AgentConfig):
        import torch

        self.net = net
        self.lr = config.lr
        self.beta1 = config.adam_beta1
        self.beta2 = config.adam_beta2
        self.eps = config.adam_eps
        self.t = 0
        self.m = torch.zeros_like(net.flat)
        self.v = torch.zeros_like(net.flat)

    def step(self) -> None:
        self.t += 1
        c1 = 1.0 - self.beta1 ** self.t
        c2 = 1.0 - self.beta2 ** self.t
        lib = _native.require_device()
        _native.check(lib.ap_dqn_adam(_native.ptr(self.net.flat), _native.ptr(self.net.grad), _native.ptr(self.m),
                                      _native.ptr(self.v), self.net.flat.numel(), self.lr, self.beta1, self.beta2,
                                      self.eps, c1, c2, _stream()))
        self.net.refresh_transposed()


def huber(x: np.ndarray, delta: float) -> np.ndarray:
    ax = np.abs(x)
    return np.where(ax <= delta, 0.5 * x ** 2, delta * (ax - 0.5 * delta))


class _Batch:
    """Preallocated device minibatch buffers for one (B, state_dim, A)."""

    def __init__(self, b: int, s: int, a: int):
        import torch

        self.states = torch.empty((b, s), dtype=torch.float32, device="cuda")
        self.next_states = torch.empty((b, s), dtype=torch.float32, device="cuda")
        self.dz = torch.empty((b, 1 + a), dtype=torch.float32, device="cuda")
        self.td = torch.empty(b, dtype=torch.float32, device="cuda")
        self.loss_rows = torch.empty(b, dtype=torch.float32, device="cuda")
        self.loss = torch.empty(1, dtype=torch.float32, device="cuda")


def train_step_device(net: QNetwork, target_net: QNetwork, buffer: PrioritizedReplayBuffer, config: AgentConfig,
                      optimizer: AdamOptimizer, uniforms, batch: _Batch | None = None):
    """One double-DQN update, all on the device; returns the loss as a device scalar (agent.py:258-299)."""
    b = config.batch_size
    batch = batch or _Batch(b, net.state_dim, net.num_actions)
    idx, weights = buffer.sample_device(b, config.per_alpha, config.per_beta, uniforms)
    return update_on_indices(net, target_net, buffer, config, idx, weights, batch, optimizer.step)


def update_on_indices(net: QNetwork, target_net: QNetwork, buffer: PrioritizedReplayBuffer, config: AgentConfig,
                      idx, weights, batch: _Batch, adam_step) -> "torch.Tensor":
    """The update of train_step (agent.py:277-299) for sampled ring indices / IS weights on the
    device: gathers, double-DQN targets, Huber TD, backward, `adam_step()`, priorities, loss.
    Shared by the host-driven agent and the device search loop (devloop.py), which captures it."""
    lib = _native.require_device()
    b = config.batch_size
    s = buffer.store
    for src, dst in ((s["states"], batch.states), (s["next_states"], batch.next_states)):
        _native.check(lib.ap_gather_rows(_native.ptr(src), src.stride(0), _native.ptr(idx), b, src.shape[1],
                                         _native.ptr(dst), dst.stride(0), _stream()))
    il = idx.long()
    actions = s["actions"][il]
    rewards = s["rewards"][il]
    done = s["done"][il]
    masks = s["next_mask"][il].contiguous()
    online_next = net.forward_device(batch.next_states)
    target_next = target_net.forward_device(batch.next_states)
    q_all, acts = net.forward_device(batch.states, cache=True)
    _native.check(lib.ap_dqn_td(_native.ptr(q_all), _native.ptr(online_next), _native.ptr(target_next),
                                q_all.stride(0), _native.ptr(actions), _native.ptr(rewards), _native.ptr(done),
                                _native.ptr(masks), masks.stride(0), _native.ptr(weights), b, net.num_actions,
                                float(config.gamma), float(config.huber_delta), _native.ptr(batch.dz),
                                batch.dz.stride(0), _native.ptr(batch.td), _native.ptr(batch.loss_rows), _stream()))
    net.backward_device(acts, batch.dz)
    adam_step()
    buffer.update_priorities_device(idx, batch.td)
    _native.check(lib.ap_dqn_colsum(_native.ptr(batch.loss_rows), 1, b, 1, _native.ptr(batch.loss), _stream()))
    return batch.loss


class FusedLearnState:
    """Device buffers of the fused learn step (td, loss, workspace, barrier) and its ctypes descriptor."""

    def __init__(self, net: "QNetwork", target: "QNetwork", buffer: "PrioritizedReplayBuffer", config: AgentConfig,
                 optimizer: "AdamOptimizer"):
        import torch

        B = config.batch_size
        self.td = torch.zeros(B, dtype=torch.float32, device="cuda")
        self.loss = torch.zeros(1, dtype=torch.float32, device="cuda")
        self.ws, self.bar = net._fused_scratch(B, False)
        L, dims, w_off, b_off, wt, wt_ld = net.fused_layout()
        s = buffer.store
        P = _native.ptr
        self.desc = _native.FusedLearnDesc(
            L=L, dims=dims, w_off=w_off, b_off=b_off, batch=B, params=P(net.flat), target=P(target.flat),
            r_states=P(s["states"]), r_next=P(s["next_states"]), r_ld=s["states"].stride(0),
            r_actions=P(s["actions"]), r_rewards=P(s["rewards"]), r_done=P(s["done"]), r_mask=P(s["next_mask"]),
            r_prio=P(s["priorities"]), gamma=float(config.gamma), huber_delta=float(config.huber_delta),
            grad=P(net.grad), m=P(optimizer.m), v=P(optimizer.v), nparams=net.flat.numel(), lr=optimizer.lr,
            beta1=optimizer.beta1, beta2=optimizer.beta2, eps=optimizer.eps, wt=wt, wt_ld=wt_ld, td=P(self.td),
            loss=P(self.loss), workspace=P(self.ws), barrier=P(self.bar))

    def run(self, idx, weights, correct1=1.0, correct2=1.0, ctab=None, ctl=None, t_offset=0, gate=0, tail=None,
            scaled=None, pstat=None, alpha=0.0, lazy_wt0=False):
        """One learn step.  `tail` (parity loop): (loss_log, loss_cap, sync_every, [(src, dst, count)]
        [, (rng_from, rng_to)]) -- the kernel also logs the loss, advances ctl's train counter,
        syncs the target and commits the early PER sample's random-stream state."""
        import ctypes

        d = self.desc
        d.idx, d.weights = idx.data_ptr(), weights.data_ptr()
        d.correct1, d.correct2 = correct1, correct2
        d.ctab = None if ctab is None else ctab.data_ptr()
        d.ctl = None if ctl is None else ctl.data_ptr()
        d.t_offset = int(t_offset)
        d.gate = int(gate)
        # optional priorities ** alpha cache kept current with each new priority (the device loop's PER sample)
        d.r_scaled, d.per_alpha = (None, 0.0) if scaled is None else (scaled.data_ptr(), float(alpha))
        d.pstat = None if pstat is None else pstat.data_ptr()
        d.lazy_wt0 = int(lazy_wt0)
        if tail is None:
            d.tail_ctl = None
        else:
            loss_log, loss_cap, sync_every, segs = tail[:4]
            rng = tail[4] if len(tail) > 4 else None
            d.rng_from, d.rng_to = (None, None) if rng is None else (rng[0].data_ptr(), rng[1].data_ptr())
            if len(segs) > 6:
                raise ValueError("at most 6 target-sync segments")
            d.tail_ctl = d.ctl
            d.loss_log, d.loss_cap, d.sync_every, d.sync_n = loss_log.data_ptr(), int(loss_cap), int(sync_every), len(segs)
            for k, (src, dst, cnt) in enumerate(segs):
                d.sync_src[k], d.sync_dst[k], d.sync_count[k] = src, dst, cnt
        _native.check(_native.require_device().ap_dqn_learn_fused(ctypes.byref(d), _stream()))
        return self.loss


def train_step(net, target_net, buffer, config, optimizer, rng) -> float:
    """Reference signature: draws the sampling uniforms from `rng`, returns the loss."""
    loss = train_step_device(net, target_net, buffer, config, optimizer, rng.random(config.batch_size))
    return float(loss.item()) / config.batch_size


class DqnAgent:
    """Network, target, replay buffer and Adam together (agent.py:302-392)."""

    def __init__(self, config: AgentConfig, state_dim: int, num_actions: int, seed: int = 0):
        self.config = config
        self.rng = np.random.default_rng(seed)
        self.net = QNetwork(state_dim, num_actions, config.hidden, self.rng)
        self.target = self.net.clone()
        self.buffer = PrioritizedReplayBuffer(config.buffer_capacity, state_dim, num_actions)
        self.optimizer = AdamOptimizer(self.net, config)
        self.train_steps = 0
        self._batch = None
        # "fused": one persistent fp32 kernel per learn step and act forward (csrc/fused_mlp.cu),
        # "gemm": the tcgen05 3xTF32 GEMM sequence (the throughput trainer's kernels)
        self.learner = "fused"
        self.net.fused_act = True
        self._fused = None

    @property
    def epsilon(self) -> float:
        return epsilon_at(self.train_steps, self.config)

    def act(self, state: np.ndarray, mask: np.ndarray, greedy: bool = False) -> int:
        return act(self.net, state, mask, 0.0 if greedy else self.epsilon, self.rng)

    def observe(self, transition: Transition) -> None:
        self.buffer.push(transition)

    def learn(self) -> float | None:
        if len(self.buffer) < self.config.batch_size:
            return None
        if self.learner == "fused":
            cfg = self.config
            if self._fused is None:
                self._fused = FusedLearnState(self.net, self.target, self.buffer, cfg, self.optimizer)
            idx, w = self.buffer.sample_device(cfg.batch_size, cfg.per_alpha, cfg.per_beta,
                                               self.rng.random(cfg.batch_size))
            opt = self.optimizer
            opt.t += 1
            loss_t = self._fused.run(idx, w, 1.0 - opt.beta1 ** opt.t, 1.0 - opt.beta2 ** opt.t)
        else:
            if self._batch is None:
                self._batch = _Batch(self.config.batch_size, self.net.state_dim, self.net.num_actions)
            loss_t = train_step_device(self.net, self.target, self.buffer, self.config, self.optimizer,
                                       self.rng.random(self.config.batch_size), self._batch)
        loss = float(loss_t.item()) / self.config.batch_size
        if not np.isfinite(loss):
            raise DivergenceError(f"training loss diverged to {loss}")
        self.train_steps += 1
        if self.train_steps % self.config.target_sync_every == 0:
            sync_target(self.net, self.target)
        return loss

    # -- checkpoints (reference .npz layout, agent.py:341-392) ----------------------

    def save(self, path: str) -> None:
        arrays = {f"net.{k}": v for k, v in self.net.params.items()}
        arrays.update({f"target.{k}": v for k, v in self.target.params.items()})
        for slot, buf in (("m", self.optimizer.m), ("v", self.optimizer.v)):
            tmp = QNetwork(self.net.state_dim, self.net.num_actions, self.net.hidden, _init=False)
            tmp.flat.copy_(buf)
            arrays.update({f"adam.{slot}.{k}": v for k, v in tmp.params.items()})
        header = {
            "version": 1,
            "config": asdict(self.config),
            "state_dim": self.net.state_dim,
            "num_actions": self.net.num_actions,
            "train_steps": self.train_steps,
            "adam_t": self.optimizer.t,
            "rng_state": self.rng.bit_generator.state,
        }
        with open(path, "wb") as fh:
            np.savez(fh, header=np.frombuffer(json.dumps(header).encode(), dtype=np.uint8), **arrays)

    @classmethod
    def load(cls, path: str) -> "DqnAgent":
        try:
            with np.load(path) as blob:
                header = json.loads(bytes(blob["header"]).decode())
                arrays = {k: blob[k] for k in blob.files if k != "header"}
        except (OSError, KeyError, ValueError, json.JSONDecodeError) as exc:
            raise CheckpointError(f"cannot read checkpoint {path}: {exc}") from exc
        if header.get("version") != 1:
            raise CheckpointError(f"unsupported checkpoint version {header.get('version')}")
        raw = dict(header["config"])
        raw["hidden"] = tuple(raw["hidden"])
        config = AgentConfig(**raw)
        agent = cls(config, header["state_dim"], header["num_actions"])
        expected = agent.net.params
        for scope, net in (("net", agent.net), ("target", agent.target)):
            params = {}
            for key, ref in expected.items():
                stored = arrays.get(f"{scope}.{key}")
                if stored is None or stored.shape != ref.shape:
                    raise CheckpointError(f"checkpoint parameter {scope}.{key} is missing or has the wrong shape")
                params[key] = stored.astype(np.float64)
            net.load_params(params)
        for slot, buf in (("m", agent.optimizer.m), ("v", agent.optimizer.v)):
            params = {}
            for key, ref in expected.items():
                stored = arrays.get(f"adam.{slot}.{key}")
                if stored is None or stored.shape != ref.shape:
                    raise CheckpointError(f"checkpoint slot adam.{slot}.{key} is missing or malformed")
                params[key] = stored.astype(np.float64)
            tmp = QNetwork(header["state_dim"], header["num_actions"], config.hidden, _init=False)
            tmp.load_params(params)
            buf.copy_(tmp.flat)
        agent.train_steps = int(header["train_steps"])
        agent.optimizer.t = int(header["adam_t"])
        agent.rng = np.random.default_rng()
        agent.rng.bit_generator.state = header["rng_state"]
        return agent
