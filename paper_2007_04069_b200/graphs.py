"""Deterministic synthetic HLO graphs of the BASELINE models.

The reference ships no generators for its benchmark models (its zoo holds
only toy blocks, reference `zoo.py:105-266`), so these build them in the
reference's own 15-opcode vocabulary (`ir.py:33-68`) and JSON schema, so
the reference planner loads the identical graph.  Vocabulary constraints
shape the lowering (SURVEY §7 hard part 5):

* dot is rank-2 only, so attention is single-head and convolutions are
  im2col-style (broadcast a patch axis, reshape, dot);
* broadcast / reduce dims pair greedily by extent, so every generator keeps
  the extents that meet in one op distinct (sequence, hidden, ffn, ...);
* `compute_cost_ms` is 2*m*k*n/1e9 for dot and output bytes/1e9 otherwise
  (SURVEY §8(d)); element size 4 bytes.

All graphs are forward-only (`is_forward` true) unless `backward=True`,
which appends a gradient-shaped backward chain per dot for the
forward+backward variant.
"""

from __future__ import annotations

import math
from typing import Callable

from .ir import HloGraph, Instruction, TensorShape

ELEMENT_BYTES = 4


class GraphWriter:
    """Sequential-id builder that attaches the deterministic cost model."""

    def __init__(self) -> None:
        self.rows: list[Instruction] = []
        self.trainable: list[str] = []

    def _cost(self, opcode: str, shape: tuple[int, ...], operands: tuple[int, ...]) -> float | None:
        if opcode in ("parameter", "constant", "tuple"):
            return None
        if opcode == "dot":
            (m, k) = self.rows[operands[0]].shape.dims
            n = shape[1]
            return 2.0 * m * k * n / 1e9
        return math.prod(shape) * ELEMENT_BYTES / 1e9

    def op(self, name: str, opcode: str, shape, operands=(), forward: bool = True) -> int:
        shape = tuple(int(d) for d in shape)
        operands = tuple(operands)
        iid = len(self.rows)
        self.rows.append(
            Instruction(
                id=iid,
                name=name,
                opcode=opcode,
                operand_ids=operands,
                shape=TensorShape(shape, ELEMENT_BYTES),
                is_forward=forward,
                compute_cost_ms=self._cost(opcode, shape, operands),
            )
        )
        return iid

    def param(self, name: str, shape, trainable: bool = True) -> int:
        if trainable:
            self.trainable.append(name)
        return self.op(name, "parameter", shape)

    def shape(self, iid: int) -> tuple[int, ...]:
        return self.rows[iid].shape.dims

    def graph(self) -> HloGraph:
        return HloGraph(self.rows, self.trainable)

    # -- composite blocks -----------------------------------------------------

    def bias_add(self, tag: str, x: int, bias: int) -> int:
        b = self.op(f"{tag}_b", "broadcast", self.shape(x), [bias])
        return self.op(f"{tag}_add", "add", self.shape(x), [x, b])

    def layer_norm(self, tag: str, x: int, hidden: int, with_bias: bool = True) -> int:
        """Mean-subtracted layer norm (as the reference zoo's, zoo.py:73-86)."""
        s = self.shape(x)[0]
        scale = self.param(f"{tag}_scale", (hidden,))
        mean = self.op(f"{tag}_mean", "reduce", (s,), [x])
        mean_b = self.op(f"{tag}_mean_b", "broadcast", (s, hidden), [mean])
        centered = self.op(f"{tag}_centered", "subtract", (s, hidden), [x, mean_b])
        sq = self.op(f"{tag}_sq", "multiply", (s, hidden), [centered, centered])
        var = self.op(f"{tag}_var", "reduce", (s,), [sq])
        var_b = self.op(f"{tag}_var_b", "broadcast", (s, hidden), [var])
        normed = self.op(f"{tag}_normed", "divide", (s, hidden), [centered, var_b])
        scale_b = self.op(f"{tag}_scale_b", "broadcast", (s, hidden), [scale])
        out = self.op(f"{tag}_scaled", "multiply", (s, hidden), [normed, scale_b])
        if with_bias:
            bias = self.param(f"{tag}_bias", (hidden,))
            out = self.bias_add(f"{tag}_bias", out, bias)
        return out

    def rms_norm(self, tag: str, x: int, hidden: int) -> int:
        """T5 layer norm: scale only, no mean subtraction."""
        s = self.shape(x)[0]
        scale = self.param(f"{tag}_scale", (hidden,))
        sq = self.op(f"{tag}_sq", "multiply", (s, hidden), [x, x])
        ms = self.op(f"{tag}_ms", "reduce", (s,), [sq])
        ms_b = self.op(f"{tag}_ms_b", "broadcast", (s, hidden), [ms])
        normed = self.op(f"{tag}_normed", "divide", (s, hidden), [x, ms_b])
        scale_b = self.op(f"{tag}_scale_b", "broadcast", (s, hidden), [scale])
        return self.op(f"{tag}_out", "multiply", (s, hidden), [normed, scale_b])

    def linear(self, tag: str, x: int, out_features: int, bias: bool) -> int:
        rows, k = self.shape(x)
        w = self.param(f"{tag}_w", (k, out_features))
        y = self.op(f"{tag}_mm", "dot", (rows, out_features), [x, w])
        if bias:
            b = self.param(f"{tag}_bias", (out_features,))
            y = self.bias_add(f"{tag}_bias", y, b)
        return y

    def attention(self, tag: str, q_src: int, kv_src: int, hidden: int, bias: bool, mask: int | None = None) -> int:
        """Single-head scaled-dot attention; q rows from q_src, keys/values from kv_src."""
        sq = self.shape(q_src)[0]
        sk = self.shape(kv_src)[0]
        q = self.linear(f"{tag}_q", q_src, hidden, bias)
        k = self.linear(f"{tag}_k", kv_src, hidden, bias)
        v = self.linear(f"{tag}_v", kv_src, hidden, bias)
        kt = self.op(f"{tag}_kt", "transpose", (hidden, sk), [k])
        scores = self.op(f"{tag}_scores", "dot", (sq, sk), [q, kt])
        if mask is not None:
            scores = self.op(f"{tag}_masked", "add", (sq, sk), [scores, mask])
        e = self.op(f"{tag}_exp", "exp", (sq, sk), [scores])
        den = self.op(f"{tag}_sum", "reduce", (sq,), [e])
        den_b = self.op(f"{tag}_sum_b", "broadcast", (sq, sk), [den])
        probs = self.op(f"{tag}_probs", "divide", (sq, sk), [e, den_b])
        ctx = self.op(f"{tag}_ctx", "dot", (sq, hidden), [probs, v])
        return self.linear(f"{tag}_o", ctx, hidden, bias)

    def squared_loss(self, tag: str, pred: int, labels: int) -> int:
        shape = self.shape(pred)
        diff = self.op(f"{tag}_diff", "subtract", shape, [pred, labels])
        sq = self.op(f"{tag}_sq", "multiply", shape, [diff, diff])
        return self.op(f"{tag}_loss", "reduce", (), [sq])


# -- models -------------------------------------------------------------------------


def mlp2() -> HloGraph:
    """2-layer MLP: the reference's `two_layer_graph` (tests/helpers.py:68-76), x[4,8] w1[8,6] w2[6,5]."""
    w = GraphWriter()
    x = w.param("x", (4, 8), trainable=False)
    w1 = w.param("w1", (8, 6))
    w2 = w.param("w2", (6, 5))
    h = w.op("h", "dot", (4, 6), [x, w1])
    w.op("y", "dot", (4, 5), [h, w2])
    g = w.rows
    # the reference fixture carries no costs; keep it byte-identical
    w.rows = [Instruction(i.id, i.name, i.opcode, i.operand_ids, i.shape) for i in g]
    return w.graph()


def bert(layers: int, hidden: int, ffn: int, seq: int = 128, labels: int = 2) -> HloGraph:
    """BERT encoder stack (post-LN, single-head attention, tanh for GELU) + a token-classifier loss."""
    if len({hidden, ffn, seq, labels}) != 4:
        raise ValueError("hidden, ffn, seq and labels must be pairwise distinct")
    w = GraphWriter()
    x = w.param("embeddings", (seq, hidden), trainable=False)
    y = w.param("labels", (seq, labels), trainable=False)
    h = x
    for layer in range(layers):
        t = f"l{layer:02d}"
        a = w.attention(f"{t}_attn", h, h, hidden, bias=True)
        h = w.op(f"{t}_res1", "add", (seq, hidden), [h, a])
        h = w.layer_norm(f"{t}_ln1", h, hidden)
        f = w.linear(f"{t}_ffn1", h, ffn, bias=True)
        f = w.op(f"{t}_act", "tanh", (seq, ffn), [f])
        f = w.linear(f"{t}_ffn2", f, hidden, bias=True)
        h = w.op(f"{t}_res2", "add", (seq, hidden), [h, f])
        h = w.layer_norm(f"{t}_ln2", h, hidden)
    logits = w.linear("cls", h, labels, bias=True)
    loss = w.squared_loss("head", logits, y)
    w.op("root", "tuple", (), [loss])
    return w.graph()


def bert_base() -> HloGraph:
    return bert(12, 768, 3072)


def bert48() -> HloGraph:
    """BERT-48 (large): 48 layers, H=1024, F=4096 (paper PAPER.md:433)."""
    return bert(48, 1024, 4096)


_VGG19 = [64, 64, "M", 128, 128, "M", 256, 256, 256, 256, "M", 512, 512, 512, 512, "M", 512, 512, 512, 512, "M"]


def vgg19(batch: int = 32, image: int = 224, classes: int = 1000) -> HloGraph:
    """VGG-19: 16 im2col 3x3 convs, 5 sum-pools, 3 FC layers, squared loss.

    Activations are [batch*h*w, channels].  A conv broadcasts a 9-wide patch
    axis, folds it into the contracting dim and multiplies by the
    [9*C_in, C_out] filter.  Pooling splits the row dim into (rows/4, 4) and
    reduces the window axis.
    """
    w = GraphWriter()
    side = image
    chans = 3
    x = w.param("images", (batch * side * side, chans), trainable=False)
    y = w.param("labels", (batch, classes), trainable=False)
    h = x
    conv = 0
    pool = 0
    for item in _VGG19:
        rows = batch * side * side
        if item == "M":
            pool += 1
            split = w.op(f"pool{pool}_split", "reshape", (rows // 4, 4, chans), [h])
            h = w.op(f"pool{pool}", "reduce", (rows // 4, chans), [split])
            side //= 2
            continue
        conv += 1
        t = f"conv{conv:02d}"
        patches = w.op(f"{t}_patches", "broadcast", (rows, 9, chans), [h])
        cols = w.op(f"{t}_im2col", "reshape", (rows, 9 * chans), [patches])
        h = w.linear(t, cols, int(item), bias=True)
        h = w.op(f"{t}_act", "tanh", (rows, int(item)), [h])
        chans = int(item)
    flat = w.op("flatten", "reshape", (batch, side * side * chans), [h])
    h = flat
    for k, width in enumerate((4096, 4096, classes)):
        h = w.linear(f"fc{k + 1}", h, width, bias=True)
        if k < 2:
            h = w.op(f"fc{k + 1}_act", "tanh", (batch, width), [h])
    loss = w.squared_loss("head", h, y)
    w.op("root", "tuple", (), [loss])
    return w.graph()


def t5(layers: int = 24, hidden: int = 1024, ffn: int = 4096, enc_seq: int = 512, dec_seq: int = 128,
       vocab: int = 32128) -> HloGraph:
    """T5 encoder-decoder: RMS norms, no biases, causal self-attention mask, cross-attention."""
    if len({hidden, ffn, enc_seq, dec_seq, vocab}) != 5:
        raise ValueError("extents must be pairwise distinct")
    w = GraphWriter()
    src = w.param("encoder_embeddings", (enc_seq, hidden), trainable=False)
    tgt = w.param("decoder_embeddings", (dec_seq, hidden), trainable=False)
    mask = w.op("causal_mask", "constant", (dec_seq, dec_seq))
    y = w.param("labels", (dec_seq, vocab), trainable=False)
    h = src
    for layer in range(layers):
        t = f"enc{layer:02d}"
        n = w.rms_norm(f"{t}_ln1", h, hidden)
        a = w.attention(f"{t}_self", n, n, hidden, bias=False)
        h = w.op(f"{t}_res1", "add", (enc_seq, hidden), [h, a])
        n = w.rms_norm(f"{t}_ln2", h, hidden)
        f = w.linear(f"{t}_wi", n, ffn, bias=False)
        f = w.op(f"{t}_act", "tanh", (enc_seq, ffn), [f])
        f = w.linear(f"{t}_wo", f, hidden, bias=False)
        h = w.op(f"{t}_res2", "add", (enc_seq, hidden), [h, f])
    memory = w.rms_norm("enc_final", h, hidden)
    h = tgt
    for layer in range(layers):
        t = f"dec{layer:02d}"
        n = w.rms_norm(f"{t}_ln1", h, hidden)
        a = w.attention(f"{t}_self", n, n, hidden, bias=False, mask=mask)
        h = w.op(f"{t}_res1", "add", (dec_seq, hidden), [h, a])
        n = w.rms_norm(f"{t}_ln2", h, hidden)
        c = w.attention(f"{t}_cross", n, memory, hidden, bias=False)
        h = w.op(f"{t}_res2", "add", (dec_seq, hidden), [h, c])
        n = w.rms_norm(f"{t}_ln3", h, hidden)
        f = w.linear(f"{t}_wi", n, ffn, bias=False)
        f = w.op(f"{t}_act", "tanh", (dec_seq, ffn), [f])
        f = w.linear(f"{t}_wo", f, hidden, bias=False)
        h = w.op(f"{t}_res3", "add", (dec_seq, hidden), [h, f])
    h = w.rms_norm("dec_final", h, hidden)
    logits = w.linear("lm_head", h, vocab, bias=False)
    loss = w.squared_loss("head", logits, y)
    w.op("root", "tuple", (), [loss])
    return w.graph()


def t5_large() -> HloGraph:
    return t5()


GENERATORS: dict[str, Callable[[], HloGraph]] = {
    "mlp2": mlp2,
    "bert_base": bert_base,
    "bert48": bert48,
    "vgg19": vgg19,
    "t5_large": t5_large,
}


def generate(name: str) -> HloGraph:
    try:
        return GENERATORS[name]()
    except KeyError:
        raise KeyError(f"unknown synthetic graph {name!r}; choose from {sorted(GENERATORS)}") from None
