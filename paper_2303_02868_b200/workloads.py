"""Synthetic page-table workloads of BASELINE.json.

The reference generates tensors with ``hiermem.footprint.tensor_inventory``
(hiermem/footprint.py:184-219, rows from :105-122).  That module is input
plumbing, not part of the update path, but the GPU box has no reference
checkout, so the param16 part of it is restated here: per layer, in
emission order, the param-bearing rows qkv (3·d²), attn-out (d²),
layer_norm (d), ffn-in (d·d_ffn), ffn-out (d·d_ffn), layer_norm (d) — each
param16 element count being params_bytes/4 of its Table-1 row.  GPT configs
append the embeddings (wte, wpe), which the reference excludes
(footprint.py:8).  tests/test_workloads.py pins these lists against the
reference's own inventory.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError

KINDS = ("param16", "grad16", "optim32", "activation16")


@dataclass(frozen=True)
class TensorSpec:
    """Same fields and validation as hiermem/footprint.py:89-102."""

    name: str
    kind: str
    bytes: int
    layer_index: int

    def __post_init__(self):
        if self.bytes <= 0:
            raise ConfigError(f"tensor {self.name!r} has non-positive size {self.bytes}")
        if self.kind not in KINDS:
            raise ConfigError(f"tensor {self.name!r} has unknown kind {self.kind!r}")


@dataclass(frozen=True)
class GPTShape:
    seq_len: int
    d_model: int
    d_ffn: int
    num_layers: int
    vocab: int = 50257


def gpt_param16(shape: GPTShape, embeddings: bool = True) -> list[TensorSpec]:
    """param16 specs of a GPT model in tensor_inventory emission order."""
    d, f = shape.d_model, shape.d_ffn
    rows = (("attn.linear_qkv", 3 * d * d), ("attn.linear_out", d * d),
            ("post_attn.layer_norm", d), ("ffn.linear_in", d * f),
            ("ffn.linear_out", d * f), ("post_ffn.layer_norm", d))
    specs = []
    for layer in range(shape.num_layers):
        for name, elems in rows:
            specs.append(TensorSpec(f"L{layer}.{name}.param16", "param16", 2 * elems, layer))
    if embeddings:
        last = shape.num_layers - 1
        specs.append(TensorSpec("wte.param16", "param16", 2 * shape.vocab * d, last))
        specs.append(TensorSpec("wpe.param16", "param16", 2 * shape.seq_len * d, last))
    return specs


def moe_param16(layers: int = 16, d_model: int = 1024, d_ffn: int = 4096,
                experts: int = 9, router_experts: int = 64) -> list[TensorSpec]:
    """C4: T5-MoE expert-sharded page pools (builder-defined):
    per layer a router, per-expert W_in/W_out plus their biases, and two
    LayerNorms — many sub-page tensors next to page-multiple ones."""
    specs = []
    for layer in range(layers):
        specs.append(TensorSpec(f"L{layer}.router.param16", "param16",
                                2 * d_model * router_experts, layer))
        for e in range(experts):
            specs.append(TensorSpec(f"L{layer}.e{e}.w_in.param16", "param16", 2 * d_model * d_ffn, layer))
            specs.append(TensorSpec(f"L{layer}.e{e}.b_in.param16", "param16", 2 * d_ffn, layer))
            specs.append(TensorSpec(f"L{layer}.e{e}.w_out.param16", "param16", 2 * d_ffn * d_model, layer))
            specs.append(TensorSpec(f"L{layer}.e{e}.b_out.param16", "param16", 2 * d_model, layer))
        for ln in ("ln1", "ln2"):
            specs.append(TensorSpec(f"L{layer}.{ln}.param16", "param16", 2 * 2 * d_model, layer))
    return specs


MIB = 2 ** 20

# name -> (specs factory, default page bytes, description)
CONFIGS = {
    "c1": (lambda: gpt_param16(GPTShape(1024, 768, 3072, 12)), 4 * MIB,
           "GPT-2 small 124M param set, 4 MiB pages"),
    "c2": (lambda: gpt_param16(GPTShape(2048, 2048, 8192, 24)), 4 * MIB,
           "GPT-3 1.3B param set, 4 MiB pages"),
    "c3": (lambda: gpt_param16(GPTShape(2048, 5120, 20480, 40)), 4 * MIB,
           "GPT-3 13B param set, 4 MiB pages, pinned-host state"),
    "c4": (lambda: moe_param16(), 256 * 1024,
           "T5-MoE expert-sharded pools, 256 KiB pages"),
    "c5": (lambda: gpt_param16(GPTShape(2048, 12288, 49152, 1), embeddings=False), 4 * MIB,
           "GPT-3 175B single-layer slice (page size swept 1-64 MiB)"),
}


def config_specs(name: str) -> list[TensorSpec]:
    if name not in CONFIGS:
        raise ConfigError(f"unknown workload {name!r}; known: {sorted(CONFIGS)}")
    return CONFIGS[name][0]()


def config_page_bytes(name: str) -> int:
    return CONFIGS[name][1]


def total_elems(specs) -> int:
    return sum(s.bytes // 2 for s in specs)
