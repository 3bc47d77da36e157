"""MAPA CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct brute force of what the MAPA hot path computes
(§3.2-§3.6, Eq. 1-3, Alg. 1; SPEC.md matcher/scoring/policies).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import, call, link or execute
anything under ``oracle/``.  The product path (``paper_2110_03214_b200``)
never imports it and shares no code with it.

* ``mapa_oracle`` — pure Python (itertools + fractions): the definition
  written out, exact rationals for Eq. 2.
* ``oracle.c`` → ``liboracle.so`` — the same definition in plain C (double for
  Eq. 2, pthreads over the first element of each device subset) for sizes the
  Python version cannot finish; cross-checked against ``mapa_oracle``.
* ``coracle`` — ctypes loader for ``liboracle.so``.
"""
