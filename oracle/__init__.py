"""TEST INFRASTRUCTURE ONLY.

The oracle package holds the checkers the product is compared against:

* ``oracle/_ref/ref_cli`` -- the reference pipeplan library itself, compiled
  from /root/reference/proj/src by ``oracle/Makefile`` and driven through a
  line-oriented JSON protocol (``ref_bridge.cpp``) in a separate process so it
  never shares an address space with the product library;
* ``oracle/schedule_ref.py`` -- a pure-Python restatement of the reference's
  schedule DAG (simulator.cpp:67-116) as a fixpoint sweep, the same
  independent check the reference's own tests use (test_support.hpp:51-85);
* ``oracle/executor_ref.py`` -- the CPU fp32/fp64 numerical executor of the
  DAPPLE training step (the reference has none; "parity unpinned" for loss and
  gradients, pinned internally by the sequential full-batch known-answer test).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.
"""
