"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the CER/CSER hot path.

Nothing in the product package (``paper_1805_10692_b200``) imports this.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline (``cpu_baseline`` and ``--impl reference``) may call it, and only
as the checker / the timed reference arm — never as a fallback.

* ``numpy_port``  — restatement of the reference's vectorised numpy path
  (``lemt.formats.encode_cer/encode_cser`` formats.py:193-295 and
  ``lemt.kernels._dot_segmented`` kernels.py:117-125, 283-301).  Bitwise
  equal to the reference on every committed golden fixture.
* ``c_oracle``    — ctypes wrapper over ``cer_oracle.c``: a C restatement of
  the encoder and of the reference's sequential loop oracle
  (``tests/reference_kernels.py:144-203``), multi-threaded over rows, for
  configs the numpy path is too slow or too big for.

Parity is pinned: ``tests/test_oracle.py`` checks both against the
fixtures in ``tests/golden/`` that ``tests/golden/make_golden.py`` produced
by running the reference (`lemt`, /root/reference/pkg) in the build
container.
"""
