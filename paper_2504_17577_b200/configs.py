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

# D=64 non-causal companion of C4 (A/B timing of the D=64 kernel only; not a BASELINE config)
EXTRA = {
    "D64N": AttnConfig("D64N", 2, 32, 32, 8192, 8192, 64, torch.float16, False, 1020, "D=64 non-causal"),
}

# The paper's own FlashAttention shapes (Table 3: batch 1, 32 heads (R13),
# head dim 128, S in {512, 1024, 4096}); context set, SURVEY §8(d). dtype bf16 (R14).
PAPER_T3 = {
    "FA0": AttnConfig("FA0", 1, 32, 32, 512, 512, 128, torch.bfloat16, True, 1010, "Table 3 FA0"),
    "FA1": AttnConfig("FA1", 1, 32, 32, 512, 512, 128, torch.bfloat16, False, 1011, "Table 3 FA1"),
    "FA2": AttnConfig("FA2", 1, 32, 32, 1024, 1024, 128, torch.bfloat16, True, 1012, "Table 3 FA2"),
    "FA3": AttnConfig("FA3", 1, 32, 32, 1024, 1024, 128, torch.bfloat16, False, 1013, "Table 3 FA3"),
    "FA4": AttnConfig("FA4", 1, 32, 32, 4096, 4096, 128, torch.bfloat16, True, 1014, "Table 3 FA4"),
}


# ------------------------------------------------------------------ MLA decode
@dataclass(frozen=True)
class MlaConfig:
    """MLA decode workload (Fig. 18 / Fig. 14). The paper's Fig. 14 shapes are an
    image; these are DeepSeek-V3-style decode shapes (latent 512 + rope 64, one kv head),
    DESIGN.md "MLA workloads". ``ragged``: per-batch cache lengths uniform in [1, Skv]."""
    name: str
    B: int
    H: int
    Hkv: int
    Skv: int
    dtype: torch.dtype
    ragged: bool
    seed: int
    Dl: int = 512
    Dr: int = 64
    note: str = ""

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.Dl + self.Dr)

    @property
    def torch_dtype(self) -> torch.dtype:
        return self.dtype

    @property
    def dtype_name(self) -> str:
        return {torch.float16: "f16", torch.bfloat16: "bf16"}[self.dtype]

    def seqlens(self):
        from .inputs import gen_seqlens
        return gen_seqlens(self.B, self.Skv, self.seed) if self.ragged else None

    def total_keys(self) -> int:
        sl = self.seqlens()
        return int(sl.sum()) if sl is not None else self.B * self.Skv

    def flops(self) -> float:
        """2*H*n*(Dl+Dr) for the scores + 2*H*n*Dl for P.V, summed over batches."""
        return 2.0 * self.H * self.total_keys() * (2 * self.Dl + self.Dr)

    def hbm_bytes(self) -> float:
        """Algorithmic bytes: the latent cache (kv + k_pe) of every used key read once,
        q / q_pe read, o written (16-bit), lse written (fp32)."""
        e = 2
        return (e * self.total_keys() * self.Hkv * (self.Dl + self.Dr)
                + e * self.B * self.H * (2 * self.Dl + self.Dr) + 4 * self.B * self.H)

    def as_dict(self):
        return {"workload": self.name, "B": self.B, "H": self.H, "Hkv": self.Hkv,
                "Skv": self.Skv, "Dl": self.Dl, "Dr": self.Dr, "dtype": self.dtype_name,
                "ragged": self.ragged}


MLA_CONFIGS = [
    MlaConfig("MLA1", 64, 128, 1, 8192, torch.bfloat16, False, 2001,
              note="DeepSeek-V3 decode, 128 heads (TP1), 8K cache"),
    MlaConfig("MLA2", 128, 16, 1, 8192, torch.bfloat16, False, 2002,
              note="16 heads per GPU (TP8), 8K cache"),
    MlaConfig("MLA3", 32, 128, 1, 16384, torch.bfloat16, True, 2003,
              note="ragged cache lengths uniform in [1, 16384]"),
]


@dataclass(frozen=True)
class SsdConfig:
    """Mamba-2 SSD chunk kernels on the paper's Table 4 shapes:
    CC<i> = chunk_scan, CT<i> = chunk_state; nheads 64, head_dim 64, d_state 128; chunk
    length 256 and one group (readings L2, L3); bf16 (reading L8)."""
    name: str
    kind: str  # "scan" | "state"
    B: int
    L: int
    H: int = 64
    G: int = 1
    P: int = 64
    N: int = 128
    Q: int = 256
    dtype: torch.dtype = torch.bfloat16
    seed: int = 4000

    @property
    def nc(self) -> int:
        return (self.L + self.Q - 1) // self.Q

    def flops(self) -> float:
        """Multiply-adds x 2 of the definition: state 2 B nc H P N Q; scan 2 B L H P N
        (entering state) + 2 B H P sum_i (i + 1) per chunk (causal intra-chunk sum)."""
        if self.kind == "state":
            return 2.0 * self.B * self.nc * self.H * self.P * self.N * self.Q
        intra = sum(min(self.Q, self.L - c * self.Q) * (min(self.Q, self.L - c * self.Q) + 1) / 2
                    for c in range(self.nc))
        return 2.0 * self.B * self.L * self.H * self.P * self.N + 2.0 * self.B * self.H * self.P * intra

    def hbm_bytes(self) -> float:
        """Algorithmic HBM bytes: every input read once, the output written once."""
        e = 2
        x = e * self.B * self.L * self.H * self.P
        bc = e * self.B * self.L * self.G * self.N
        vec = 2 * 4 * self.B * self.H * self.nc * self.Q                 # dt, dA (fp32)
        states = e * self.B * self.nc * self.H * self.P * self.N
        if self.kind == "state":
            return x + bc + vec + states
        cb = e * self.B * self.nc * self.G * self.Q * self.Q
        return cb + x + bc + vec + states + x + 4 * self.H                # + out, D

    def as_dict(self):
        return {"workload": self.name, "kind": self.kind, "batch": self.B, "seqlen": self.L,
                "nheads": self.H, "ngroups": self.G, "headdim": self.P, "dstate": self.N,
                "chunk_size": self.Q, "dtype": {torch.float16: "f16", torch.bfloat16: "bf16"}[self.dtype]}


_T4 = {"0": (1, 1024), "1": (1, 2048), "2": (1, 8192), "3": (64, 1024), "4": (64, 2048),
       "5": (64, 8192)}
SSD_CONFIGS = {}
for _i, (_b, _l) in _T4.items():
    SSD_CONFIGS["CC" + _i] = SsdConfig("CC" + _i, "scan", _b, _l, seed=4000 + int(_i))
    SSD_CONFIGS["CT" + _i] = SsdConfig("CT" + _i, "state", _b, _l, seed=4100 + int(_i))
