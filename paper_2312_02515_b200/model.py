"""Multi-LoRA fine-tuning of a whole decoder on the fused batch (configs C1, C4).

Every job shares ONE frozen base model; each job owns a LoRA adapter on every
linear of every layer.  The jobs' token sequences are fused into one row
batch (job order, then sequence order — the reference FusedBatch order,
/root/reference/proj/src/lora.cpp:143-156) and one training step runs

    embed -> L x [ RMSNorm -> q,k,v -> attention (RoPE) -> o -> +res
                   -> RMSNorm -> gate,up -> SwiGLU -> down -> +res ]
          -> RMSNorm -> LM head -> padding-masked CE (per-job mean)

forward and backward with every linear as the BatchFusion multi-LoRA linear
(mlora_down_group / mlora_base_fwd / mlora_base_dx / mlora_grad_group, each
HBM-bound op grouped over the projections that share a wave), then one AdamW
with per-job learning rates over every adapter of every layer.  Only the
adapters train: embeddings, norms, W0 and the LM head are frozen, as in LoRA.

The reference has no model: the linears are pinned to its
fused_forward by the layer-level parity tests; the model around them
(attention, norms, SwiGLU, CE) is "parity unpinned" and checked against a
PyTorch fp32 autograd restatement (tests/test_gpu_decoder.py).

Architectures: "llama" (separate q, k, v, o, gate, up, down; grouped-query
attention when kv_heads < heads) and "chatglm2" (fused qkv with multi-query
attention: kv_heads = 2, dense, fused h_to_4h = [gate; up], 4h_to_h).  RoPE is
rotate-half over the full head dim for both (ChatGLM2's half-dim interleaved
rotary is a positional-encoding detail outside the hot path).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _native as N
from . import errors
from . import fused as F
from . import model_ops as M
from .layer import AdapterJobsMixin


@dataclass(frozen=True)
class DecoderConfig:
    name: str
    hidden: int
    ffn: int
    heads: int
    kv_heads: int
    vocab: int
    layers: int
    arch: str = "llama"
    rope_base: float = 10000.0
    eps: float = 1e-6

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def projections(self) -> list[tuple[str, int, int]]:
        """(name, d_out, k_in) of every LoRA'd linear of one layer, in forward order."""
        h, f, kv = self.hidden, self.ffn, self.kv_heads * self.head_dim
        if self.arch == "llama":
            return [("q", h, h), ("k", kv, h), ("v", kv, h), ("o", h, h), ("gate", f, h), ("up", f, h),
                    ("down", h, f)]
        if self.arch == "chatglm2":
            return [("qkv", h + 2 * kv, h), ("dense", h, h), ("h_to_4h", 2 * f, h), ("4h_to_h", h, f)]
        raise errors.UsageError(f"unknown arch {self.arch!r}")

    def with_layers(self, n: int) -> "DecoderConfig":
        return DecoderConfig(self.name, self.hidden, self.ffn, self.heads, self.kv_heads, self.vocab, n, self.arch,
                             self.rope_base, self.eps)


# C1: 2 layers, h = 256, ffn = 688, 4 heads, V = 1024.
TINY_LLAMA = DecoderConfig("tiny-llama", 256, 688, 4, 4, 1024, 2)
LLAMA_7B = DecoderConfig("llama-7b", 4096, 11008, 32, 32, 32000, 32)
LLAMA_13B = DecoderConfig("llama-13b", 5120, 13824, 40, 40, 32000, 40)
# C4: ChatGLM2-6B (multi-query attention with 2 groups, V = 65024).
CHATGLM2_6B = DecoderConfig("chatglm2-6b", 4096, 13696, 32, 2, 65024, 28, "chatglm2")
TINY_CHATGLM2 = DecoderConfig("tiny-chatglm2", 256, 688, 4, 2, 1024, 2, "chatglm2")

CONFIGS = {c.name: c for c in (TINY_LLAMA, LLAMA_7B, LLAMA_13B, CHATGLM2_6B, TINY_CHATGLM2)}


# ---------------------------------------------------------------- fused token batch
@dataclass
class TokenBatch:
    """One fused batch of token sequences (host side).

    seg: J+1 job row offsets; seq_offsets / seq_lens: the attention layout;
    tokens / labels (next token within the sequence) / mask (1 = a position
    whose label counts) are row-aligned int lists.  `padded` reproduces the
    reference's fuse() layout (every sequence zero-padded to the global
    max_len, lora.cpp:114-158); otherwise sequences are packed back to back."""
    seg: list[int]
    seq_offsets: list[int]
    seq_lens: list[int]
    tokens: list[int]
    labels: list[int]
    mask: list[int]
    padded: bool = False
    real_tokens: int = 0

    @property
    def rows(self) -> int:
        return self.seg[-1]


def pack_tokens(job_sequences, padded: bool = False) -> TokenBatch:
    """job_sequences[j] = list of token-id sequences of job j (possibly empty)."""
    seqs = [(j, s) for j, ss in enumerate(job_sequences) for s in ss]
    if not seqs:
        raise errors.UsageError("empty fused batch")
    if any(len(s) == 0 for _, s in seqs):
        raise errors.UsageError("empty sequence")  # as fuse(), lora.cpp:131
    max_len = max(len(s) for _, s in seqs)
    seg, off, lens, tok, lab, msk = [0], [0], [], [], [], []
    for j, ss in enumerate(job_sequences):
        for s in ss:
            n = len(s)
            slot = max_len if padded else n
            tok += list(s) + [0] * (slot - n)
            lab += list(s[1:]) + [0] * (slot - n + 1)
            msk += [1] * (n - 1) + [0] * (slot - n + 1)
            lens.append(n)
            off.append(off[-1] + slot)
        seg.append(off[-1])
    return TokenBatch(seg, off, lens, tok, lab, msk, padded, sum(lens))


# ---------------------------------------------------------------- the model
@dataclass
class _Proj:
    name: str
    d: int
    k: int
    W0: torch.Tensor
    A: F.AdamState
    B: F.AdamState
    dA: torch.Tensor
    dB: torch.Tensor
    Y: torch.Tensor
    H: torch.Tensor


@dataclass
class _Layer:
    norm1: torch.Tensor
    norm2: torch.Tensor
    proj: dict = field(default_factory=dict)
    x1: torch.Tensor | None = None      # residual stream after attention
    h1: torch.Tensor | None = None      # RMSNorm(x_in)
    h2: torch.Tensor | None = None      # RMSNorm(x1)
    rstd1: torch.Tensor | None = None
    rstd2: torch.Tensor | None = None
    attn: torch.Tensor | None = None    # attention output
    qr: torch.Tensor | None = None      # RoPE(q), RoPE(k): rotated once, read by every attention tile
    kr: torch.Tensor | None = None
    lse: torch.Tensor | None = None
    act: torch.Tensor | None = None     # SwiGLU output


class MultiLoraDecoder(AdapterJobsMixin):
    """J LoRA jobs fine-tuning one frozen decoder on fused batches, on one GPU."""

    def __init__(self, ctx: F.Context, cfg: DecoderConfig, ranks, scales, lrs, capacity: int, seed: int = 0,
                 lora_init: str = "random", weight_decay: float = 0.0, frozen: "MultiLoraDecoder | None" = None):
        """frozen: share another decoder's frozen base (embedding, norms, W0, LM
        head) instead of initialising one — e.g. to resume jobs on the same base."""
        if capacity < 1:
            raise errors.UsageError("capacity must be >= 1 row")
        self.ctx, self.cfg = ctx, cfg
        self.ranks, self.scales, self.lrs = list(ranks), list(scales), list(lrs)
        self.J = len(self.ranks)
        self.capacity = capacity
        self.weight_decay = weight_decay
        self.step_count = [0] * self.J
        dev = ctx.device
        self.plan = F.Plan(ctx, [0] * self.J + [capacity], self.ranks, self.scales)
        R = self.plan.rank_padded
        g = torch.Generator(device=dev).manual_seed(seed)  # seeded init, generated in HBM

        def U(*shape, scale=1.0):
            return (torch.rand(*shape, generator=g, device=dev) * 2 - 1) * scale

        h, V, rows = cfg.hidden, cfg.vocab, capacity
        bf = torch.bfloat16
        if frozen is not None and frozen.cfg != cfg:
            raise errors.ShapeError("frozen base has a different config")
        if frozen is None:
            self.embed_w = U(V, h).to(bf)
            self.head_w = U(V, h, scale=h ** -0.5).to(bf)
            self.final_norm = (1 + U(h, scale=0.1)).to(bf)
        else:
            self.embed_w, self.head_w, self.final_norm = frozen.embed_w, frozen.head_w, frozen.final_norm
        self.layers: list[_Layer] = []
        for li in range(cfg.layers):
            if frozen is None:
                L = _Layer((1 + U(h, scale=0.1)).to(bf), (1 + U(h, scale=0.1)).to(bf))
            else:
                L = _Layer(frozen.layers[li].norm1, frozen.layers[li].norm2)
            for name, d, k in cfg.projections():
                W0 = U(d, k, scale=k ** -0.5).to(bf) if frozen is None else frozen.layers[li].proj[name].W0
                As = [U(r, k, scale=k ** -0.5) for r in self.ranks]
                if lora_init == "zero_b":
                    Bs = [torch.zeros(d, r, device=dev) for r in self.ranks]
                else:
                    Bs = [U(d, r, scale=r ** -0.5) for r in self.ranks]
                A32, B32, A16, B16 = F.pack_adapters(ctx, self.plan, d, k, As, Bs)
                L.proj[name] = _Proj(name, d, k, W0, F.AdamState.of(A32, A16, 0), F.AdamState.of(B32, B16, 1),
                                     torch.zeros(R, k, device=dev), torch.zeros(d, R, device=dev),
                                     torch.empty(rows, d, dtype=bf, device=dev),
                                     torch.empty(rows, R, dtype=bf, device=dev))
            L.x1 = torch.empty(rows, h, dtype=bf, device=dev)
            L.h1 = torch.empty(rows, h, dtype=bf, device=dev)
            L.h2 = torch.empty(rows, h, dtype=bf, device=dev)
            L.rstd1 = torch.empty(rows, dtype=torch.float32, device=dev)
            L.rstd2 = torch.empty(rows, dtype=torch.float32, device=dev)
            L.attn = torch.empty(rows, h, dtype=bf, device=dev)
            L.qr = torch.empty(rows, h, dtype=bf, device=dev)
            L.kr = torch.empty(rows, cfg.kv_heads * cfg.head_dim, dtype=bf, device=dev)
            L.lse = torch.empty(cfg.heads, rows, dtype=torch.float32, device=dev)
            L.act = torch.empty(rows, cfg.ffn, dtype=bf, device=dev)
            self.layers.append(L)
        # residual stream entering each layer, and after the last one
        self.xs = [torch.empty(rows, h, dtype=bf, device=dev) for _ in range(cfg.layers + 1)]
        self.hf = torch.empty(rows, h, dtype=bf, device=dev)
        self.rstdf = torch.empty(rows, dtype=torch.float32, device=dev)
        self.logits = torch.empty(rows, V, dtype=bf, device=dev)
        self.dlogits = torch.empty(rows, V, dtype=bf, device=dev)
        self.loss = torch.zeros(self.J, dtype=torch.float32, device=dev)
        # backward scratch, shared by all layers (consumed in stream order)
        self._g = {name: torch.empty(rows, R, dtype=bf, device=dev) for name, _, _ in cfg.projections()}
        self._dy = {name: torch.empty(rows, d, dtype=bf, device=dev) for name, d, _ in cfg.projections()}
        self._dx = {name: torch.empty(rows, k, dtype=bf, device=dev) for name, _, k in cfg.projections()}
        self._dres = [torch.empty(rows, h, dtype=bf, device=dev) for _ in range(3)]
        self._dsum = torch.empty(cfg.heads, rows, dtype=torch.float32, device=dev)
        self._row_loss = torch.empty(rows, dtype=torch.float32, device=dev)
        self._inv = torch.empty(self.J, dtype=torch.float32, device=dev)
        self.batch: TokenBatch | None = None

    def frozen_tensors(self) -> dict:
        """Every frozen base tensor by name (what a multi-GPU run replicates once
        from rank 0: parallel.broadcast_base_weights)."""
        out = {"embed": self.embed_w, "head": self.head_w, "final_norm": self.final_norm}
        for li, L in enumerate(self.layers):
            out[f"{li}.norm1"], out[f"{li}.norm2"] = L.norm1, L.norm2
            for name, p in L.proj.items():
                out[f"{li}.{name}.W0"] = p.W0
        return out

    def named_projections(self):
        """(key, projection) of every LoRA'd linear: keys 'layer.name' (checkpoints, quarantine)."""
        return [(f"{li}.{name}", p) for li, L in enumerate(self.layers) for name, p in L.proj.items()]

    # ------------------------------------------------------------ batch
    def set_batch(self, batch: TokenBatch) -> None:
        """Install one fused batch: job segments (plan), attention layout, tokens."""
        if len(batch.seg) != self.J + 1:
            raise errors.UsageError(f"batch has {len(batch.seg) - 1} jobs, model has {self.J}")
        rows = batch.rows
        if rows < 1 or rows > self.capacity:
            raise errors.UsageError(f"batch rows {rows} outside [1, capacity {self.capacity}]")
        if any(t < 0 or t >= self.cfg.vocab for t in batch.tokens + batch.labels):
            raise errors.UsageError("token id outside the vocabulary")
        dev = self.ctx.device
        self.plan.update(batch.seg)
        self.layout = M.AttnLayout(batch.seq_offsets, batch.seq_lens, device=dev)
        self.tokens = torch.tensor(batch.tokens, dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
        self.labels = torch.tensor(batch.labels, dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
        self.mask = torch.tensor(batch.mask, dtype=torch.uint8).pin_memory().to(dev, non_blocking=True)
        self.seg_dev = torch.tensor(batch.seg, dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
        self.batch = batch
        self.rows = rows

    # ------------------------------------------------------------ helpers
    def _down(self, probs, backward: bool, s) -> None:
        """Grouped rank-r down-projection for [(proj, input)] (H forward, G backward)."""
        n = len(probs)
        L = N.lib()
        if backward:
            width = [p.d for p, _ in probs]
            adapt = [p.B.p_bf16 for p, _ in probs]
            out = [self._g[p.name][: self.rows] for p, _ in probs]
        else:
            width = [p.k for p, _ in probs]
            adapt = [p.A.p_bf16 for p, _ in probs]
            out = [p.H[: self.rows] for p, _ in probs]
        N.check(L.mlora_down_group(self.ctx.handle, self.plan.handle, n, 1 if backward else 0,
                                   (N.i32 * n)(*width), (N.vp * n)(*[x.data_ptr() for _, x in probs]),
                                   (N.vp * n)(*[a.data_ptr() for a in adapt]),
                                   (N.vp * n)(*[o.data_ptr() for o in out]), s), self.ctx.handle)

    def _fwd_gemm(self, p: _Proj, x: torch.Tensor, s) -> torch.Tensor:
        Y = p.Y[: self.rows]
        N.check(N.lib().mlora_base_fwd(self.ctx.handle, self.plan.handle, p.d, p.k, x.data_ptr(), p.W0.data_ptr(),
                                       p.H.data_ptr(), p.B.p_bf16.data_ptr(), Y.data_ptr(), None, s),
                self.ctx.handle)
        return Y

    def _dx_gemm(self, p: _Proj, dY: torch.Tensor, s) -> torch.Tensor:
        dX = self._dx[p.name][: self.rows]
        N.check(N.lib().mlora_base_dx(self.ctx.handle, self.plan.handle, p.d, p.k, dY.data_ptr(), p.W0.data_ptr(),
                                      self._g[p.name].data_ptr(), p.A.p_bf16.data_ptr(), dX.data_ptr(), s),
                self.ctx.handle)
        return dX

    def _grads(self, items, s) -> None:
        """dA, dB of [(proj, X, dY)] in one grouped launch pair."""
        n = len(items)
        N.check(N.lib().mlora_grad_group(
            self.ctx.handle, self.plan.handle, n, (N.i32 * n)(*[p.d for p, _, _ in items]),
            (N.i32 * n)(*[p.k for p, _, _ in items]), (N.vp * n)(*[x.data_ptr() for _, x, _ in items]),
            (N.vp * n)(*[dy.data_ptr() for _, _, dy in items]), (N.vp * n)(*[p.H.data_ptr() for p, _, _ in items]),
            (N.vp * n)(*[self._g[p.name].data_ptr() for p, _, _ in items]),
            (N.vp * n)(*[p.dA.data_ptr() for p, _, _ in items]), (N.vp * n)(*[p.dB.data_ptr() for p, _, _ in items]),
            s), self.ctx.handle)

    def _guard(self, tensors, s) -> None:
        """Job isolation under divergence (as the layer step's guard):
        for every job whose CE is not finite, zero its rows of the tensors the
        grouped dA / dB reductions read.  Those reductions run over several jobs'
        rows inside one 64-column rank block and rely on structural zeros
        (H, G block-diagonal); 0 * inf = NaN would otherwise leak a diverged job
        into its neighbours' gradients.  All-finite: one launch reading J floats."""
        uniq = {}
        for t in tensors:
            uniq.setdefault(t.data_ptr(), t.shape[1])
        n = len(uniq)
        N.check(N.lib().mlora_zero_nonfinite_rows(self.ctx.handle, self.plan.handle, self.loss.data_ptr(),
                                                  (N.vp * n)(*uniq.keys()), (N.i32 * n)(*uniq.values()), n, s),
                self.ctx.handle)

    def _qkv_views(self, L: _Layer, grad: bool = False):
        cfg, r = self.cfg, self.rows
        kv = cfg.kv_heads * cfg.head_dim
        if cfg.arch == "llama":
            src = self._dy if grad else {n: p.Y for n, p in L.proj.items()}
            return src["q"][:r], src["k"][:r], src["v"][:r]
        Y = (self._dy["qkv"] if grad else L.proj["qkv"].Y)[:r]
        h = cfg.hidden
        return Y[:, :h], Y[:, h:h + kv], Y[:, h + kv:h + 2 * kv]

    def _ffn_views(self, L: _Layer, grad: bool = False):
        r, f = self.rows, self.cfg.ffn
        if self.cfg.arch == "llama":
            src = self._dy if grad else {n: p.Y for n, p in L.proj.items()}
            return src["gate"][:r], src["up"][:r]
        Y = (self._dy["h_to_4h"] if grad else L.proj["h_to_4h"].Y)[:r]
        return Y[:, :f], Y[:, f:]

    # ------------------------------------------------------------ forward
    def forward(self, stream=None) -> torch.Tensor:
        """Forward over the installed batch; returns the per-job mean CE (device
        fp32 [J]) and leaves d(sum_j loss_j)/dlogits in self.dlogits."""
        if self.batch is None:
            raise errors.StateError("set_batch() first")
        cfg, r = self.cfg, self.rows
        s = F._stream_handle(stream)
        sm = stream
        names = [n for n, _, _ in cfg.projections()]
        attn_p, out_p, up_p, down_p = (names[:3], names[3], names[4:6], names[6]) if cfg.arch == "llama" else \
            (names[:1], names[1], names[2:3], names[3])
        M.embed(self.tokens[:r], self.embed_w, out=self.xs[0][:r], stream=sm)
        L0 = self.layers[0]
        M.add_rmsnorm(self.xs[0][:r], None, L0.norm1, cfg.eps, y=L0.h1[:r], rstd=L0.rstd1[:r], stream=sm)
        for li, L in enumerate(self.layers):
            P = L.proj
            self._down([(P[n], L.h1[:r]) for n in attn_p], False, s)
            for n in attn_p:
                self._fwd_gemm(P[n], L.h1[:r], s)
            q, k, v = self._qkv_views(L)
            self._attn_fwd(L, q, k, v, sm)
            self._down([(P[out_p], L.attn[:r])], False, s)
            Yo = self._fwd_gemm(P[out_p], L.attn[:r], s)
            M.add_rmsnorm(self.xs[li][:r], Yo, L.norm2, cfg.eps, x_out=L.x1[:r], y=L.h2[:r], rstd=L.rstd2[:r],
                          stream=sm)
            self._down([(P[n], L.h2[:r]) for n in up_p], False, s)
            for n in up_p:
                self._fwd_gemm(P[n], L.h2[:r], s)
            gate, up = self._ffn_views(L)
            M.swiglu_fwd(gate, up, out=L.act[:r], stream=sm)
            self._down([(P[down_p], L.act[:r])], False, s)
            Yd = self._fwd_gemm(P[down_p], L.act[:r], s)
            last = li == len(self.layers) - 1
            nxt_w = self.final_norm if last else self.layers[li + 1].norm1
            nxt_y = self.hf if last else self.layers[li + 1].h1
            nxt_r = self.rstdf if last else self.layers[li + 1].rstd1
            M.add_rmsnorm(L.x1[:r], Yd, nxt_w, cfg.eps, x_out=self.xs[li + 1][:r], y=nxt_y[:r], rstd=nxt_r[:r],
                          stream=sm)
        # frozen LM head (no LoRA term) + padding-masked per-job CE
        N.check(N.lib().mlora_base_fwd(self.ctx.handle, self.plan.handle, cfg.vocab, cfg.hidden,
                                       self.hf[:r].data_ptr(), self.head_w.data_ptr(), None, None,
                                       self.logits[:r].data_ptr(), None, s), self.ctx.handle)
        N.check(N.lib().mlora_masked_ce(self.J, self.seg_dev.data_ptr(), r, cfg.vocab, self.logits[:r].data_ptr(),
                                        self.labels[:r].data_ptr(), self.mask[:r].data_ptr(),
                                        self._row_loss[:r].data_ptr(), self.loss.data_ptr(), self._inv.data_ptr(),
                                        self.dlogits[:r].data_ptr(), s))
        return self.loss

    def _attn_fwd(self, L: _Layer, q, k, v, stream) -> None:
        cfg, r = self.cfg, self.rows
        lse = L.lse.view(-1)[: cfg.heads * r].view(cfg.heads, r)
        qr, kr = L.qr[:r], L.kr[:r]
        M.attn_rope(self.layout, q, cfg.heads, cfg.head_dim, cfg.rope_base, out=qr, stream=stream)
        M.attn_rope(self.layout, k, cfg.kv_heads, cfg.head_dim, cfg.rope_base, out=kr, stream=stream)
        M.attn_fwd(self.layout, qr, kr, v, cfg.heads, cfg.kv_heads, cfg.head_dim, cfg.rope_base, out=L.attn[:r],
                   lse=lse, prerotated=True, stream=stream)

    # ------------------------------------------------------------ backward
    def backward(self, stream=None) -> None:
        """Adapter gradients of sum_j loss_j (each job's mean CE) into every proj's dA / dB."""
        cfg, r = self.cfg, self.rows
        s = F._stream_handle(stream)
        sm = stream
        names = [n for n, _, _ in cfg.projections()]
        llama = cfg.arch == "llama"
        attn_p, out_p, up_p, down_p = (names[:3], names[3], names[4:6], names[6]) if llama else \
            (names[:1], names[1], names[2:3], names[3])
        dh = self._dx["o" if llama else "dense"]  # scratch [rows, h] for the LM-head dX
        N.check(N.lib().mlora_base_dx(self.ctx.handle, self.plan.handle, cfg.vocab, cfg.hidden,
                                      self.dlogits[:r].data_ptr(), self.head_w.data_ptr(), None, None,
                                      dh[:r].data_ptr(), s), self.ctx.handle)
        d_out = M.rmsnorm_bwd_sum([dh[:r]], None, self.xs[-1][:r], self.final_norm, self.rstdf[:r],
                                  out=self._dres[0][:r], stream=sm)
        free = [self._dres[1], self._dres[2]]
        for li in reversed(range(len(self.layers))):
            L = self.layers[li]
            P = L.proj
            # ---- MLP: x_out = x1 + down(act), act = swiglu(gate(h2), up(h2))
            self._down([(P[down_p], d_out)], True, s)
            d_act = self._dx_gemm(P[down_p], d_out, s)
            gate, up = self._ffn_views(L)
            dgate, dup = self._ffn_views(L, grad=True)
            M.swiglu_bwd(gate, up, d_act, dgate, dup, stream=sm)
            dys_up = [self._dy[n][:r] for n in up_p]
            self._down([(P[n], dy) for n, dy in zip(up_p, dys_up)], True, s)
            dx_up = [self._dx_gemm(P[n], dy, s) for n, dy in zip(up_p, dys_up)]
            d_x1 = M.rmsnorm_bwd_sum(dx_up, d_out, L.x1[:r], L.norm2, L.rstd2[:r], out=free[0][:r], stream=sm)
            # ---- attention: x1 = x_in + o(attn(q, k, v))
            self._down([(P[out_p], d_x1)], True, s)
            d_attn = self._dx_gemm(P[out_p], d_x1, s)
            _, _, v = self._qkv_views(L)
            dq, dk, dv = self._qkv_views(L, grad=True)
            lse = L.lse.view(-1)[: cfg.heads * r].view(cfg.heads, r)
            dsum = self._dsum.view(-1)[: cfg.heads * r].view(cfg.heads, r)
            M.attn_bwd(self.layout, L.qr[:r], L.kr[:r], v, L.attn[:r], d_attn, lse, dq, dk, dv, cfg.heads,
                       cfg.kv_heads, cfg.head_dim, cfg.rope_base, dsum=dsum, prerotated=True, stream=sm)
            dys_attn = [self._dy[n][:r] for n in attn_p]
            self._down([(P[n], dy) for n, dy in zip(attn_p, dys_attn)], True, s)
            d_in = None
            if li > 0:  # the embedding is frozen: layer 0 needs no input gradient
                dx_attn = [self._dx_gemm(P[n], dy, s) for n, dy in zip(attn_p, dys_attn)]
                d_in = M.rmsnorm_bwd_sum(dx_attn, d_x1, self.xs[li][:r], L.norm1, L.rstd1[:r], out=free[1][:r],
                                         stream=sm)
            # ---- adapter gradients of the whole layer: one grouped dA + one grouped dB launch
            items = [(P[n], L.h1[:r], dy) for n, dy in zip(attn_p, dys_attn)]
            items.append((P[out_p], L.attn[:r], d_x1))
            items += [(P[n], L.h2[:r], dy) for n, dy in zip(up_p, dys_up)]
            items.append((P[down_p], L.act[:r], d_out))
            self._guard([x for _, x, _ in items] + [dy for _, _, dy in items], s)
            self._grads(items, s)
            if d_in is not None:
                # the next (lower) layer's output gradient; the buffer d_out held is
                # free again once this layer's grad launches (stream-ordered) read it
                d_out = d_in
                free = [b for b in self._dres if b.data_ptr() != d_in.data_ptr()]

    # ------------------------------------------------------------ optimizer
    def adapter_tensors(self):
        """(AdamState, grad) of every adapter tensor, layer by layer."""
        out = []
        for L in self.layers:
            for p in L.proj.values():
                out += [(p.A, p.dA), (p.B, p.dB)]
        return out

    def optimizer_step(self, active=None, stream=None) -> None:
        """One AdamW over every adapter (per-job lr; jobs with no rows in the
        batch, marked inactive, or whose loss this step is not finite are left
        untouched)."""
        if active is None:
            seg = self.batch.seg
            active = [seg[j + 1] > seg[j] for j in range(self.J)]
        self.step_count = [c + (1 if a else 0) for c, a in zip(self.step_count, active)]
        steps = [c if a else 0 for c, a in zip(self.step_count, active)]
        st = self.adapter_tensors()
        # skip-on-overflow: a job whose CE is not finite this step keeps its adapter
        # (no host sync), so its NaN gradient cannot reach the fused tiles it shares
        F.adam_step(self.ctx, self.plan, [a for a, _ in st], [g for _, g in st], self.lrs, steps,
                    weight_decay=self.weight_decay, stream=stream, loss_gate=self.loss)

    def step(self, batch: TokenBatch | None = None, stream=None) -> torch.Tensor:
        """One fine-tuning step of every job in the batch: forward, per-job CE,
        backward, AdamW.  Returns the per-job losses (device, before the update)."""
        if batch is not None:
            self.set_batch(batch)
        loss = self.forward(stream)
        self.backward(stream)
        self.optimizer_step(stream=stream)
        return loss

    # ------------------------------------------------------------ accounting
    def flops_per_step(self) -> int:
        """Algorithmic FLOPs of one step over the batch's rows: every LoRA'd
        linear 4dk + 6r(d+k) per row of its job, the frozen
        LM head 4hV per row (forward + dX), causal attention 2 * 2 * len^2 * h
        forward-equivalent x 3.5 (fwd + recompute-based bwd) per sequence."""
        cfg, b = self.cfg, self.batch
        tot = 0
        for j in range(self.J):
            n = b.seg[j + 1] - b.seg[j]
            for _, d, k in cfg.projections():
                tot += cfg.layers * n * (4 * d * k + 6 * self.ranks[j] * (d + k))
        tot += b.rows * 4 * cfg.hidden * cfg.vocab
        tot += int(sum(3.5 * 2 * n * n * cfg.hidden for n in b.seq_lens)) * cfg.layers
        return tot
