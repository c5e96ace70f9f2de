"""B200-native DCAT scoring path (PinFM, arxiv 2507.12704).

Drop-in for seqfm::rank_forward_batch (reference finetune.hpp:150-154) through
the C ABI in include/dcat_b200.h; kernels for sm_100a in csrc/.
"""
from .abi import Batch, FinetuneSpec, ModelSpec, Weights  # noqa: F401

__all__ = ["Batch", "FinetuneSpec", "ModelSpec", "Weights", "DcatModel", "build"]


def __getattr__(name):
    if name in ("DcatModel", "probs_from_logits", "lib"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)


def build(verbose: bool = False) -> str:
    """Compile csrc/ into libdcat_b200.so (sm_100a) in-tree."""
    import os
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(here, "csrc")], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
    return os.path.join(here, "libdcat_b200.so")
