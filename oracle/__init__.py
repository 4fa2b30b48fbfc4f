"""TEST INFRASTRUCTURE ONLY — the parity oracle for the WaveHoltz explicit hot path.

Nothing in the product package (``paper_2504_03074_b200``) may import, call,
link or execute anything under ``oracle/``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs use it, and only as the checker / the timed CPU baseline.

Contents
--------
``waveholtz_oracle``   numpy restatement of the reference's explicit path in the
                       reference's exact operation order (bitwise identical to
                       ``waveholtz.timestep.wave_solve_filtered``; pinned against
                       the committed golden vectors in ``tests/golden``).
``whb_oracle.c``       the same algorithm in plain C (OpenMP), built with
                       ``-ffp-contract=off`` so it stays bitwise identical; used
                       where the numpy path is too slow (1025^3) and as the
                       multi-core CPU baseline.
``native``             ctypes loader for the C restatement.
``reference_harness``  helpers that import the real reference from
                       ``/root/reference`` (this container only) to generate and
                       check the golden fixtures.
"""
