"""Synthetic MoE-layer inputs from the ORACLE's generator — TEST / BASELINE
INFRASTRUCTURE ONLY.

The same keyed streams as paper_2603_06350_b200/workload.py (the product's
host/synth.cpp), restated in oracle/moe_oracle.c (orc_stream_key,
orc_synth_*), so the CPU reference arm of bench.py never loads the product
library.  tests/test_oracle.py checks both generators give identical bytes.
"""
from __future__ import annotations

import numpy as np

from . import orc, popularity, synth_expert, synth_gate, synth_tokens

TAG_TOKENS = 0x78746F6B  # "xtok"
TAG_GATE = 0x67617465    # "gate"
TAG_EXPERT = 0x65787074  # "expt"
TAG_NOISE = 0x6E6F6973   # "nois"


def stream_key(seed: int, a: int, b: int, tag: int) -> int:
    return int(orc().orc_stream_key(seed, a, b, tag))


def noise_permutation(E: int, seed: int, layer: int, iteration: int) -> np.ndarray:
    rng = np.random.default_rng(stream_key(seed, layer, iteration, TAG_NOISE))
    return rng.permutation(E).astype(np.int32)


def gate_weights(E: int, d: int, zipf_s: float, seed: int, layer: int, iteration: int,
                 drift_period: int = 0) -> np.ndarray:
    _, w = popularity(E, zipf_s, seed, layer, iteration, drift_period)
    return synth_gate(stream_key(seed, layer, 0, TAG_GATE), d, E, w, noise_permutation(E, seed, layer, iteration))


def tokens(T: int, d: int, E: int, seed: int, batch: int) -> np.ndarray:
    return synth_tokens(stream_key(seed, batch, 0, TAG_TOKENS), 0, T, d, E)


def expert_weights(d: int, ff: int, seed: int, layer: int, expert: int):
    return synth_expert(stream_key(seed, layer, expert, TAG_EXPERT), d, ff)
