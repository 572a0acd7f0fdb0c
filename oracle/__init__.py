"""CPU oracle for the DSP hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything under `oracle/`. The
product path (`paper_2403_10266_b200/`) never imports it and shares no code,
headers, tables or helpers with it; both sides only share the seeded input
generator in `synth/`, which holds none of the method's arithmetic.

What it computes (PAPER.md = P:line, SPEC.md = S:line):
  * block.py   — the unsharded spatial-temporal block (P:40 pre-LN + residual
                 transformer block; P:17/P:46 attention "calculated separately for
                 the temporal and spatial dimensions"), float64 numpy.
  * switch.py  — split / gather / dynamic switch (§3.1, "a single AlltoAll
                 operation ... when transitioning between computation stages") as
                 explicit per-pair message copies between simulated ranks, with a
                 byte ledger (self-sends excluded S:173).
  * sharded.py — the DSP schedule over N simulated ranks (Fig. 1/2):
                 split -> spatial stage on T-shards -> switch T->S -> temporal stage
                 + MLP on S-shards -> switch S->T -> gather.
  * block_nd.py — the multi-dimensional block (attention along any list of dims)
                 and its DSP schedule with N-D switches (P:93 generalisation).
  * volume.py  — the communication-volume analysis of §3.2 / Table 1.

Pins (tests/test_oracle_*.py, `-m "not gpu"`) tie each function to something
other than itself: torch.nn library modules in float64, brute-force loops,
closed forms, the SPEC worked examples (tests/golden/), and invariants.
"""
