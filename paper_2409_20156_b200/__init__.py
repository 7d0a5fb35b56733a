"""B200-native ASTRA classifier hot path (drop-in for xcmix's refresh /
sampler / sampled-loss / classifier-update functions).

Layers:
  _lib      ctypes binding of the C-ABI (include/astra_b200.h, libastra_b200.so)
  ops       torch-tensor wrappers, one per C-ABI entry point
  anns, trainer, classifiers
            the reference-facing mirror: same names, signatures and error
            classes as xcmix.anns / xcmix.trainer / xcmix.classifiers
  engine    device-resident classifier state (W shard, optimizer state,
            hard-negative cache) and the full classifier step
  shard     label-range sharding over torch.distributed (NCCL)
  install   rebinding of the xcmix module globals to this package
"""

__version__ = "0.1.0"
