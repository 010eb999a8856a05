"""State-dict layouts of the benchmark architectures, without instantiating them.

The benchmark configs (BASELINE.json) hash random-init fp32 weights of GPT-2,
GPT2-XL, BERT-large and VGG19; bert-base and ResNet152 complete the paper's model table. Only the ordered list of (name, shape) matters to
the hashing path, so the layouts are derived here from the architecture
hyper-parameters; they reproduce the ``state_dict()`` entry order and sizes of
``transformers`` 5.5 / ``torchvision`` 0.26 (149 / 581 / 391 /
38 entries, byte totals checked in tests/test_shapes.py).

``lm_head.weight`` of the GPT-2 LM-head models is tied to ``wte.weight``: the
same storage appears twice in the state dict and is hashed twice.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Tuple

Layout = List[Tuple[str, Tuple[int, ...], Optional[str]]]   # (name, shape, name of the entry it aliases)


def gpt2_lm_head(n_embd: int = 768, n_layer: int = 12, vocab: int = 50257, n_pos: int = 1024) -> Layout:
    d = n_embd
    out: Layout = [("transformer.wte.weight", (vocab, d), None), ("transformer.wpe.weight", (n_pos, d), None)]
    for i in range(n_layer):
        p = f"transformer.h.{i}."
        out += [
            (p + "ln_1.weight", (d,), None), (p + "ln_1.bias", (d,), None),
            (p + "attn.c_attn.weight", (d, 3 * d), None), (p + "attn.c_attn.bias", (3 * d,), None),
            (p + "attn.c_proj.weight", (d, d), None), (p + "attn.c_proj.bias", (d,), None),
            (p + "ln_2.weight", (d,), None), (p + "ln_2.bias", (d,), None),
            (p + "mlp.c_fc.weight", (d, 4 * d), None), (p + "mlp.c_fc.bias", (4 * d,), None),
            (p + "mlp.c_proj.weight", (4 * d, d), None), (p + "mlp.c_proj.bias", (d,), None),
        ]
    out += [("transformer.ln_f.weight", (d,), None), ("transformer.ln_f.bias", (d,), None),
            ("lm_head.weight", (vocab, d), "transformer.wte.weight")]
    return out


def gpt2_model(n_embd: int = 768, n_layer: int = 12, vocab: int = 50257, n_pos: int = 1024) -> Layout:
    """``GPT2Model`` (no LM head): the LM-head layout without ``lm_head.weight`` and without the ``transformer.``
    prefix -- 148 / 580 entries, the "124M" / "1.5B" parameter counts."""
    return [(name[len("transformer."):], shape, alias) for name, shape, alias in gpt2_lm_head(n_embd, n_layer, vocab, n_pos)
            if name != "lm_head.weight"]


def bert_model(hidden: int = 1024, layers: int = 24, intermediate: int = 4096, vocab: int = 30522,
               max_pos: int = 512, type_vocab: int = 2) -> Layout:
    h = hidden
    out: Layout = [
        ("embeddings.word_embeddings.weight", (vocab, h), None),
        ("embeddings.position_embeddings.weight", (max_pos, h), None),
        ("embeddings.token_type_embeddings.weight", (type_vocab, h), None),
        ("embeddings.LayerNorm.weight", (h,), None), ("embeddings.LayerNorm.bias", (h,), None),
    ]
    for i in range(layers):
        p = f"encoder.layer.{i}."
        for proj in ("query", "key", "value"):
            out += [(p + f"attention.self.{proj}.weight", (h, h), None), (p + f"attention.self.{proj}.bias", (h,), None)]
        out += [
            (p + "attention.output.dense.weight", (h, h), None), (p + "attention.output.dense.bias", (h,), None),
            (p + "attention.output.LayerNorm.weight", (h,), None), (p + "attention.output.LayerNorm.bias", (h,), None),
            (p + "intermediate.dense.weight", (intermediate, h), None), (p + "intermediate.dense.bias", (intermediate,), None),
            (p + "output.dense.weight", (h, intermediate), None), (p + "output.dense.bias", (h,), None),
            (p + "output.LayerNorm.weight", (h,), None), (p + "output.LayerNorm.bias", (h,), None),
        ]
    out += [("pooler.dense.weight", (h, h), None), ("pooler.dense.bias", (h,), None)]
    return out


def vgg19() -> Layout:
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, 256, "M", 512, 512, 512, 512, "M", 512, 512, 512, 512, "M"]
    out: Layout = []
    idx, cin = 0, 3
    for v in cfg:
        if v == "M":
            idx += 1
            continue
        out += [(f"features.{idx}.weight", (v, cin, 3, 3), None), (f"features.{idx}.bias", (v,), None)]
        cin = v
        idx += 2          # conv + ReLU
    for j, (fin, fout) in zip((0, 3, 6), ((512 * 7 * 7, 4096), (4096, 4096), (4096, 1000))):
        out += [(f"classifier.{j}.weight", (fout, fin), None), (f"classifier.{j}.bias", (fout,), None)]
    return out


def resnet_bottleneck(blocks=(3, 8, 36, 3), num_classes: int = 1000) -> Layout:
    """torchvision ``resnet152`` (blocks 3-8-36-3): 932 state-dict entries, 241,378,168 bytes.

    Every BatchNorm contributes weight, bias, running_mean, running_var and the int64 scalar
    ``num_batches_tracked`` (8 bytes -- listed here as two fp32 words, same byte count): the
    many-tiny-tensors end of the paper's model table.
    """
    out: Layout = []

    def bn(prefix: str, c: int) -> None:
        out.extend([(prefix + ".weight", (c,), None), (prefix + ".bias", (c,), None),
                    (prefix + ".running_mean", (c,), None), (prefix + ".running_var", (c,), None),
                    (prefix + ".num_batches_tracked", (2,), None)])

    out.append(("conv1.weight", (64, 3, 7, 7), None))
    bn("bn1", 64)
    cin = 64
    for stage, (n_blocks, width) in enumerate(zip(blocks, (64, 128, 256, 512)), start=1):
        for b in range(n_blocks):
            p = f"layer{stage}.{b}."
            out.append((p + "conv1.weight", (width, cin, 1, 1), None)); bn(p + "bn1", width)
            out.append((p + "conv2.weight", (width, width, 3, 3), None)); bn(p + "bn2", width)
            out.append((p + "conv3.weight", (4 * width, width, 1, 1), None)); bn(p + "bn3", 4 * width)
            if b == 0:
                out.append((p + "downsample.0.weight", (4 * width, cin, 1, 1), None)); bn(p + "downsample.1", 4 * width)
            cin = 4 * width
    out += [("fc.weight", (num_classes, cin), None), ("fc.bias", (num_classes,), None)]
    return out


ARCHITECTURES = {
    "gpt2": lambda: gpt2_lm_head(768, 12),
    "gpt2-xl": lambda: gpt2_lm_head(1600, 48),
    "gpt2-model": lambda: gpt2_model(768, 12),
    "gpt2-xl-model": lambda: gpt2_model(1600, 48),
    "bert-large": lambda: bert_model(1024, 24, 4096),
    "vgg19": vgg19,
    "bert-base": lambda: bert_model(768, 12, 3072),
    "resnet152": resnet_bottleneck,
}


def numel(shape) -> int:
    n = 1
    for s in shape:
        n *= s
    return n


def layout_stats(layout: Layout, block_size: int = 8192, itemsize: int = 4) -> Dict[str, int]:
    sizes = [numel(shape) * itemsize for _, shape, _ in layout]
    return {
        "entries": len(layout),
        "bytes": sum(sizes),
        "leaves": sum(-(-s // block_size) for s in sizes),
        "ragged": sum(1 for s in sizes if s % block_size),
    }


def synthetic_state_dict(arch: str, device, seed: int = 0, scale: float = 1.0):
    """Random-init fp32 tensors of the named architecture, each its own allocation.

    ``scale`` < 1 shrinks every dimension-0 extent (tests); the benchmark uses 1.
    Returns a list of (name, tensor) in state-dict order; tied entries share storage.
    """
    import torch

    layout = ARCHITECTURES[arch]()
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    made: Dict[str, "torch.Tensor"] = {}
    out = []
    for name, shape, alias in layout:
        if alias is not None:
            out.append((name, made[alias]))
            continue
        if scale != 1.0:
            shape = (max(1, int(shape[0] * scale)),) + tuple(shape[1:])
        t = torch.empty(shape, dtype=torch.float32, device=device)
        t.normal_(0.0, 0.02, generator=gen)
        made[name] = t
        out.append((name, t))
    return out
