"""fp64 CPU oracle for the pruned RNN-T hot path (arXiv 2206.13236).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2206_13236_b200``) never imports it, and it
never imports the product path: the two share no code.  The only common module
is ``synth`` (seeded input generation, no method arithmetic).

Citations: ``P:<line>`` = line of /root/reference/PAPER.md.  Readings of the
paper where it is silent or garbled are the D-numbers of DESIGN.md.

Parity pins (tests/test_oracle_*.py): brute-force path enumeration, the
uniform-lattice closed forms, finite differences, occupancy sum rules,
torchaudio's independent ``rnnt_loss`` (S >= U+1 identity and the linear
joiner identity), and brute-force least-feasible-sequence for the bound
adjustment.  Nothing here is "parity unpinned" except the time/memory
figures, which are not computed here.
"""
from .rnnt_oracle import *  # noqa: F401,F403
