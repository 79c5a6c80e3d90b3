"""dapple-b200: B200-native DAPPLE synchronous pipelined-DP training step.

* ``pipeplan``  -- the reference's planner / simulator API (bit-exact), via
  the C-ABI of libdapple.so;
* ``kernels``   -- the hand-written sm_100a stage kernels;
* ``runtime``   -- the per-GPU executor (one process per GPU) that runs a
  plan's early-backward 1F1B schedule with Split-Concat P2P and per-layer
  NCCL AllReduce and returns a measured Timeline.
"""
__version__ = "0.1.0"
