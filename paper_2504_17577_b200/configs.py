"""Workload configurations (BASELINE.json ``configs`` + the north_star target T0).

C1..C5 are BASELINE.json configs[0..4]; T0 is the north_star's "D=128 non-causal
S=8192" target shape. FLOP convention
(R12): 4*B*Hq*Sq*Skv*D, halved when causal.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class AttnConfig:
    name: str
    B: int
    Hq: int
    Hkv: int
    Sq: int
    Skv: int
    D: int
    dtype: torch.dtype
    causal: bool
    seed: int
    note: str = ""

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.D)

    @property
    def dtype_name(self) -> str:
        return {torch.float16: "f16", torch.bfloat16: "bf16"}[self.dtype]

    def flops(self) -> float:
        """FA convention: 4*B*Hq*Sq*Skv*D, x1/2 if causal (R12)."""
        f = 4.0 * self.B * self.Hq * self.Sq * self.Skv * self.D
        return f / 2 if self.causal else f

    def flops_exact(self) -> float:
        """4*B*Hq*D*sum_i |J_i| — the count of allowed (query, key) pairs."""
        if not self.causal:
            pairs = self.Sq * self.Skv
        else:
            off = self.Skv - self.Sq
            pairs = 0
            # |J_i| = clamp(i + off + 1, 0, Skv); closed-form sum over i
            for i in range(self.Sq):
                pairs += max(0, min(self.Skv, i + off + 1))
        return 4.0 * self.B * self.Hq * self.D * pairs

    def hbm_bytes(self) -> float:
        """Algorithmic HBM bytes: Q, K, V read once, O written once, LSE written once."""
        e = 2
        return (e * self.B * self.Sq * self.Hq * self.D * 2          # Q + O
                + e * self.B * self.Skv * self.Hkv * self.D * 2      # K + V
                + 4 * self.B * self.Hq * self.Sq)                    # LSE

    def as_dict(self):
        return {"workload": self.name, "B": self.B, "Hq": self.Hq, "Hkv": self.Hkv,
                "Sq": self.Sq, "Skv": self.Skv, "D": self.D, "dtype": self.dtype_name,
                "causal": self.causal}


CONFIGS = {
    "C1": AttnConfig("C1", 1, 1, 1, 128, 128, 64, torch.float16, False, 1001,
                     "tiny oracle-checkable instance"),
    "C2": AttnConfig("C2", 8, 16, 16, 4096, 4096, 128, torch.bfloat16, False, 1002,
                     "paper-style FlashAttention benchmark"),
    "C3": AttnConfig("C3", 4, 32, 8, 8192, 8192, 128, torch.bfloat16, True, 1003,
                     "causal GQA 4:1"),
    "C4": AttnConfig("C4", 1, 32, 32, 16384, 16384, 64, torch.float16, True, 1004,
                     "causal long sequence"),
    "C5": AttnConfig("C5", 64, 32, 32, 2048, 2048, 128, torch.bfloat16, True, 1005,
                     "batch x head sharded across 1/2/4/8 B200"),
    "T0": AttnConfig("T0", 4, 32, 8, 8192, 8192, 128, torch.bfloat16, False, 1003,
                     "north_star target: D=128 non-causal S=8192 (C3 inputs, causal off)"),
}
