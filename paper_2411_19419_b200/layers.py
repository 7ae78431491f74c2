"""DenseNet121 single-channel layer table (the paper's Table 2) and its CSV
reader -- the workload of the reference's layer bench (inc/bench.hpp:36-111).

``densenet121_layers()`` generates the table from the architecture (stem
conv + pool, dense blocks of 6/12/24/16 bottleneck layers at 56/28/14/7 px,
transitions between blocks) and reproduces the reference's shipped
``proj/data/densenet121_layers.csv`` row for row, including the table's one
quirk (no 1x1 conv listed for block2.layer1), 123 rows in all;
tests/test_layers.py pins it against that file.  ``load_layer_table`` mirrors
the reference parser (inc/bench.hpp:68-111): same header check, field count,
integer parsing and ConvSpec validation, with the same messages.
"""
from __future__ import annotations

import os
import re
from dataclasses import dataclass
from typing import List


@dataclass(frozen=True)
class LayerConfig:
    """inc/bench.hpp:36-41."""
    name: str
    m: int
    n: int
    k: int
    s: int
    p: int

    def spec(self):
        from . import ConvSpec
        return ConvSpec(self.m, self.n, self.k, self.s, self.p)


def densenet121_layers() -> List[LayerConfig]:
    rows = [LayerConfig("conv0", 224, 224, 7, 2, 3), LayerConfig("pool0", 112, 112, 3, 2, 1)]
    for b, (size, count) in enumerate(zip((56, 28, 14, 7), (6, 12, 24, 16)), start=1):
        for layer in range(1, count + 1):
            if not (b == 2 and layer == 1):  # Table 2 lists no 1x1 conv for block2.layer1
                rows.append(LayerConfig(f"block{b}.layer{layer}.conv1", size, size, 1, 1, 0))
            rows.append(LayerConfig(f"block{b}.layer{layer}.conv2", size, size, 3, 1, 1))
        if b < 4:
            rows.append(LayerConfig(f"transition{b}.conv", size, size, 1, 1, 0))
            rows.append(LayerConfig(f"transition{b}.pool", size, size, 2, 2, 0))
    return rows


def _parse_count(s: str, context: str) -> int:
    """std::stoll with a full-consumption check (inc/bench.hpp:54-65): leading
    whitespace and a sign are accepted, anything after the digits is not."""
    if not re.fullmatch(r"[ \t\n\v\f\r]*[+-]?[0-9]+", s):
        raise RuntimeError(f"{context}: not an integer: '{s}'")
    return int(s.strip())


def load_layer_table(path: str) -> List[LayerConfig]:
    """Parses a ``name,m,n,k,s,p`` CSV; every row must form a valid ConvSpec."""
    if not os.path.exists(path):
        raise RuntimeError(f"cannot open layer table '{path}'")
    with open(path, newline="") as f:
        lines = f.read().split("\n")
    if not lines or (len(lines) == 1 and not lines[0]):
        raise RuntimeError(f"{path}: empty file")
    head = lines[0].rstrip("\r")
    if head != "name,m,n,k,s,p":
        raise RuntimeError(f"{path}:1: expected header 'name,m,n,k,s,p', got '{head}'")
    out = []
    for lineno, line in enumerate(lines[1:], start=2):
        line = line.rstrip("\r")
        if not line:
            continue
        where = f"{path}:{lineno}"
        fields = line.split(",")
        if len(fields) != 6:
            raise RuntimeError(f"{where}: expected 6 fields, got {len(fields)}")
        cfg = LayerConfig(fields[0], *(_parse_count(v, where) for v in fields[1:]))
        try:
            cfg.spec()
        except ValueError as e:
            raise RuntimeError(f"{where}: layer '{cfg.name}': {e}") from None
        out.append(cfg)
    return out
