"""Parameter-shape tables of the paper's four models (workload definitions only).

This module holds NO arithmetic of the method: it lists parameter shapes so
that synthetic gradients can be generated "shaped like the paper's models"
(BASELINE.json configs; "ResNet-50, ResNet-152, BERT-Base and
BERT-Large"). Both the oracle tests and the CUDA path consume these lists.

Shapes follow torchvision's Bottleneck ResNet (v1.5, stride on the 3x3) and
HF ``BertForPreTraining`` (decoder weight tied to the word embeddings, so it
is counted once). SURVEY.md Appendix A derives them and Appendix B shows the
totals reproduce Table I: 25.6 / 60.2 / 110.1 / 336.2 M.

Order: ``forward_params`` returns named shapes in FORWARD (registration)
order. Gradients become ready in REVERSE order during back-propagation
("the registered hook function will be called when each gradient is
ready"), so ``ready_order`` reverses the list; the C ABI takes tensors in
ready order.
"""
from __future__ import annotations

from typing import List, Tuple

Shape = Tuple[int, ...]
Named = Tuple[str, Shape]

_RESNET_BLOCKS = {"resnet50": (3, 4, 6, 3), "resnet152": (3, 8, 36, 3)}


def _resnet(blocks) -> List[Named]:
    out: List[Named] = [("conv1.weight", (64, 3, 7, 7)),
                        ("bn1.weight", (64,)), ("bn1.bias", (64,))]
    cin = 64
    for s, nb in enumerate(blocks):
        w = 64 * 2 ** s
        cout = 4 * w
        for b in range(nb):
            p = f"layer{s + 1}.{b}."
            out += [(p + "conv1.weight", (w, cin, 1, 1)),
                    (p + "bn1.weight", (w,)), (p + "bn1.bias", (w,)),
                    (p + "conv2.weight", (w, w, 3, 3)),
                    (p + "bn2.weight", (w,)), (p + "bn2.bias", (w,)),
                    (p + "conv3.weight", (cout, w, 1, 1)),
                    (p + "bn3.weight", (cout,)), (p + "bn3.bias", (cout,))]
            if b == 0:
                out += [(p + "downsample.0.weight", (cout, cin, 1, 1)),
                        (p + "downsample.1.weight", (cout,)),
                        (p + "downsample.1.bias", (cout,))]
            cin = cout
    out += [("fc.weight", (1000, 2048)), ("fc.bias", (1000,))]
    return out


def _bert(H: int, I: int, L: int, vocab: int = 30522, pos: int = 512,
          types: int = 2) -> List[Named]:
    e = "bert.embeddings."
    out: List[Named] = [(e + "word_embeddings.weight", (vocab, H)),
                        (e + "position_embeddings.weight", (pos, H)),
                        (e + "token_type_embeddings.weight", (types, H)),
                        (e + "LayerNorm.weight", (H,)), (e + "LayerNorm.bias", (H,))]
    for l in range(L):
        p = f"bert.encoder.layer.{l}."
        for nm in ("query", "key", "value"):
            out += [(p + f"attention.self.{nm}.weight", (H, H)),
                    (p + f"attention.self.{nm}.bias", (H,))]
        out += [(p + "attention.output.dense.weight", (H, H)),
                (p + "attention.output.dense.bias", (H,)),
                (p + "attention.output.LayerNorm.weight", (H,)),
                (p + "attention.output.LayerNorm.bias", (H,)),
                (p + "intermediate.dense.weight", (I, H)),
                (p + "intermediate.dense.bias", (I,)),
                (p + "output.dense.weight", (H, I)),
                (p + "output.dense.bias", (H,)),
                (p + "output.LayerNorm.weight", (H,)),
                (p + "output.LayerNorm.bias", (H,))]
    out += [("bert.pooler.dense.weight", (H, H)), ("bert.pooler.dense.bias", (H,)),
            ("cls.predictions.bias", (vocab,)),
            ("cls.predictions.transform.dense.weight", (H, H)),
            ("cls.predictions.transform.dense.bias", (H,)),
            ("cls.predictions.transform.LayerNorm.weight", (H,)),
            ("cls.predictions.transform.LayerNorm.bias", (H,)),
            ("cls.seq_relationship.weight", (2, H)),
            ("cls.seq_relationship.bias", (2,))]
    return out


MODELS = ("resnet50", "resnet152", "bert-base", "bert-large")


def forward_params(model: str) -> List[Named]:
    if model in _RESNET_BLOCKS:
        return _resnet(_RESNET_BLOCKS[model])
    if model == "bert-base":
        return _bert(768, 3072, 12)
    if model == "bert-large":
        return _bert(1024, 4096, 24)
    raise ValueError(f"unknown model {model!r}; choose from {MODELS}")


def ready_order(model: str) -> List[Named]:
    """Gradient-ready order = reverse of forward order."""
    return list(reversed(forward_params(model)))


def numel(shape: Shape) -> int:
    n = 1
    for d in shape:
        n *= int(d)
    return n
