"""Synthetic pruned-parameter sets of the BASELINE.json configs.

The reference has no GPT model; SURVEY.md Appendix B defines the GPT-style
parameter sets (tensor list, [in, out] row-major weights as init_params,
train.hpp:105-123; 2-D weights prunable, 1-D LN/bias tensors non-prunable as
train.hpp:116-119).  Values come from the counter-based generator of the C ABI
(samo_synth_uniform_*), so any element can be regenerated on the host by the
test oracle.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Tensor:
    name: str
    shape: tuple[int, ...]

    @property
    def numel(self) -> int:
        n = 1
        for e in self.shape:
            n *= e
        return n

    @property
    def prunable(self) -> bool:
        return len(self.shape) == 2

    @property
    def init_bound(self) -> float:
        # uniform_symmetric(1/sqrt(in_features)) for weights (train.hpp:112-115);
        # 1-D tensors get a small symmetric range (their values do not matter
        # for the mask: non-prunable tensors keep every index).
        return (1.0 / float(self.shape[0]) ** 0.5) if self.prunable else 0.02


def gpt_tensors(n_layer: int, d: int, vocab: int = 50257, ctx: int = 2048) -> list[Tensor]:
    """GPT-2/3 style tensor list."""
    ts = [Tensor("wte", (vocab, d)), Tensor("wpe", (ctx, d))]
    for b in range(n_layer):
        p = f"h{b}."
        ts += [Tensor(p + "ln_1.weight", (d,)), Tensor(p + "ln_1.bias", (d,)),
               Tensor(p + "attn.qkv.weight", (d, 3 * d)), Tensor(p + "attn.qkv.bias", (3 * d,)),
               Tensor(p + "attn.proj.weight", (d, d)), Tensor(p + "attn.proj.bias", (d,)),
               Tensor(p + "ln_2.weight", (d,)), Tensor(p + "ln_2.bias", (d,)),
               Tensor(p + "mlp.fc.weight", (d, 4 * d)), Tensor(p + "mlp.fc.bias", (4 * d,)),
               Tensor(p + "mlp.proj.weight", (4 * d, d)), Tensor(p + "mlp.proj.bias", (d,))]
    ts += [Tensor("ln_f.weight", (d,)), Tensor("ln_f.bias", (d,))]
    return ts


@dataclass(frozen=True)
class Workload:
    name: str
    tensors: tuple[Tensor, ...]
    sparsity: float
    description: str

    @property
    def phi(self) -> int:
        return sum(t.numel for t in self.tensors)


def gpt_1_3b(p: float = 0.9) -> Workload:
    return Workload(f"gpt-1.3b-p{p}", tuple(gpt_tensors(24, 2048)), p,
                    "GPT-3 XL style set: L=24, d=2048, vocab 50257, ctx 2048 (292 tensors)")


def gpt_2_7b(p: float = 0.9) -> Workload:
    return Workload(f"gpt-2.7b-p{p}", tuple(gpt_tensors(32, 2560)), p,
                    "GPT-3 2.7B style set: L=32, d=2560, vocab 50257, ctx 2048 (388 tensors)")


def fc(n: int, p: float = 0.9) -> Workload:
    """Paper Fig. 1 FC layer [n, n] (BASELINE configs 1-2)."""
    return Workload(f"fc{n}-p{p}", (Tensor("fc0.weight", (n, n)),), p,
                    f"single {n}x{n} FC layer")


WORKLOADS = {
    "gpt-2.7b": gpt_2_7b,
    "gpt-1.3b": gpt_1_3b,
    "fc4096": lambda p=0.9: fc(4096, p),
}


def get(name: str, p: float | None = None) -> Workload:
    if name.startswith("fc") and name[2:].isdigit():
        return fc(int(name[2:]), 0.9 if p is None else p)
    fn = WORKLOADS[name]
    return fn() if p is None else fn(p)
