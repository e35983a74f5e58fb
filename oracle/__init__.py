"""fp64 CPU oracle for the fused attention forward — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path
(``paper_2504_17577_b200``) never imports it and shares no code with it.
See ``oracle/oracle.h`` for the definitions and their citations (attention: PAPER.md
P:L424, Fig. 18; GEMM: Fig. 16; MLA: Fig. 18; Mamba-2 SSD chunk
kernels: Table 4). ``oracle.ssd`` holds the plain preprocessing steps of the SSD
pipeline (chunked cumulative decay, C B^T per chunk, state passing) used to pin the chunk
kernels against the recurrence.
"""
from .oracle import (  # noqa: F401
    build_oracle,
    widen,
    attn_rows,
    attn_rows_parallel,
    attn_full,
    brute_force,
    gemm_rows,
    gemm_rows_parallel,
    mla_decode,
    mla_decode_parallel,
    mla_brute,
    ssd_chunk_state,
    ssd_chunk_scan,
    ssd_recurrence,
    ssd_sample_chunks,
    ORACLE_F16,
    ORACLE_BF16,
)
