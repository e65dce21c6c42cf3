"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the VPM-MPPI hot path.

Nothing in ``paper_2509_16079_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and its
``--impl reference`` arm) use it, and only as the checker / CPU baseline.

* :mod:`oracle.core` -- ctypes binding to ``liboracle.so`` (``vpm_oracle.c``,
  an FP64 C restatement of ``_accel/_core.pyx:175-745``) exposing the reference
  stepping-module contract (``step`` / ``rollout`` / ``batch_rollout`` /
  ``omp_threads``) plus per-rollout discrete-decision diagnostics.
* :mod:`oracle.planner` -- numpy restatement of ``mppi.py:19-84`` and
  ``policy.py:66-266`` driven by :mod:`oracle.core`.
* :mod:`oracle.refcore` -- loader for ``oracle/_ref/_core*.so``, the reference's
  own Cython core compiled by ``oracle/build_ref.sh``.
* :mod:`oracle.refpkg` -- imports the unmodified reference package staged under
  ``oracle/_ref/pkg`` and installs a stepping module as its compiled core (the
  drop-in tests run the reference's own API on the CUDA backend).
"""
