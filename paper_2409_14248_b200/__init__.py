"""B200-native (sm_100a) HRKAN physics-informed loss + gradient hot path (arXiv 2409.14248).

`hrkan`    ctypes binding of libhrkan.so (include/hrkan.h): create / forward_jet /
           pinn_loss_grad / adam_step / free.
`parallel` data-parallel step: contiguous point shards per rank, global normalisers and ONE
           allreduce of the flat [dL/dtheta | loss parts | flag] buffer (torch.distributed,
           NCCL on GPUs, gloo in the CPU tests).
"""
from .hrkan import (HRKANNet, HrkanError, HrkanPde, JET_HESSIAN, JET_TAYLOR5, jet_channels, load_library,  # noqa: F401
                    pde_struct)
