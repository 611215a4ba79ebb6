"""CPU oracle for the NeuralPVS hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU reference.  The product path (``paper_2509_24677_b200``) never
imports it and fails loudly when its CUDA library is missing.

Contents
* ``oracle.sparse`` — numpy (float64) restatement of the reference hot path
  (pkg/src/froxelpvs/interleave.py:54-85, neural.py:151-399) in submanifold
  (masked) form, plus the pieces BASELINE.json needs that the reference lacks
  (kernel maps, k2s2 down/up convs, the U-Net, bf16 emulation, Kaiming-uniform
  init).  Every function cites the reference lines it follows.
* ``oracle.refbridge`` — imports the real reference from /root/reference when it
  is present (this container only) so tests can check the restatement against
  it and ``tests/golden/make_golden.py`` can write golden vectors.

Parity pinning: the reference's own tests do not cover the hot path (SURVEY.md
§4), so the restatement is pinned (a) against the reference itself, run here
by ``tests/golden/make_golden.py`` into committed fixtures, and (b) against the
SPEC known-answer examples.
"""
