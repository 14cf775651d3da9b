"""CPU oracle for the STR / rSTR per-batch update — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 numpy implementation of what the hot path computes,
written from the paper (arXiv 2307.00719, ``/root/reference/PAPER.md``; cited as P:<line>).
Each function cites the passage it follows.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this package.
The product path (``paper_2307_00719_b200``) never imports it and shares no code with it.

Modules
  tensor   Def. 1 unfoldings, index linearization, TR reconstruction
  tralg    subchain (Def. 3), ⊠₂ (Def. 6), ⊡₂ (Def. 7), Gram tensors Z_n,
           ×_{2,4}^{1,3} (Def. 5), Gram chains H (Prop. 1), pseudo-inverse solve
  als      TR-ALS (Alg. 1) — init producer and pin for the STR step
  stream   STR (Alg. 4)
  sampler  SplitMix64 index draws, uniform / leverage distributions (ledger #11)
  rstream  rSTR-U / rSTR-L (Alg. 7, Alg. 8)
  ksrft    rSTR-K: KSRFT mixing (Def. 10, Alg. 5), Alg. 9
  fit      relative error

Parity status: every function is pinned by a -m "not gpu"
test except the noisy whole-trajectory results, which are pinned only through invariants
(the paper prints no numbers for them) and rSTR at m=2000 ("parity unpinned" vs theory;
pinned only by the exhaustive-enumeration degeneracy rSTR == STR).  rSTR-K (ksrft) likewise:
its mixing is pinned by numpy's FFT and brute force, its sketched normal equations by the
exhaustive-sketch identity and the exact-stream fixed point; at m=2000 it is "parity unpinned"
against Theorem 3.
"""
