"""B200-native Woodpecker-DL hot path (arXiv 2008.04567): forward conv2d + fused bias/ReLU on
sm_100a kernels, and the per-layer GA / RL-search tuner, behind the C ABI of include/wpk.h."""
from . import _lib
from .conv import Conv2dPlan, DwPwPlan, make_options, output_dims

__all__ = ["Conv2dPlan", "DwPwPlan", "make_options", "output_dims", "_lib"]
