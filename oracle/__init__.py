"""CPU oracle for the flood-ensemble overlap path — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (``paper_2104_14667_b200``) imports, links or executes
anything under ``oracle/``.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` use it, and only as the
checker or the timed CPU baseline.

Contents
--------
* ``fs_oracle.py``  — NumPy restatement of the reference algorithm (each function cites
  the reference file:line it follows).  Pinned against the reference itself: the golden
  fixtures in ``tests/golden/`` were produced by importing /root/reference's
  ``floodstream`` (script ``tests/golden/make_golden.py``), and
  ``tests/test_oracle_golden.py`` checks this module reproduces every one of them.
* ``fs_oracle.c``   — the same primitives in plain C with pthreads, used as the
  multi-core CPU baseline at sizes NumPy cannot finish quickly.
* ``Makefile``      — builds ``_build/libfs_oracle.so`` and, when /root/reference is
  present, ``_ref/``: the reference's own native accelerator (``_accel.pyx``) cythonized
  and compiled from the sources where they lie (outputs only into ``_ref/``).
"""
