"""Fixture loading shared by the CPU and GPU parity tests."""
from __future__ import annotations

import os

import numpy as np

from paper_2507_12704_b200.abi import Batch, FinetuneSpec, ModelSpec

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def batch_from(z, prefix: str = "") -> Batch:
    g = lambda f: z[prefix + f]  # noqa: E731
    aux = z[prefix + "aux"] if (prefix + "aux") in z.files else None
    return Batch(g("row_offset").astype(np.int64), g("row_valid").astype(np.int32), g("ev_ts").astype(np.uint64),
                 g("ev_action").astype(np.uint8), g("ev_surface").astype(np.uint8), g("ev_item").astype(np.uint64),
                 g("candidate").astype(np.uint64), g("age_seconds").astype(np.float64),
                 None if aux is None else aux.astype(np.float32))


def spec_from(z, prefix: str = "") -> ModelSpec:
    s = [int(x) for x in z[prefix + "spec"]]
    return ModelSpec(*s)


def weights_from(z, impl, prefix: str = ""):
    """Re-create the fixture's weights with `impl` (oracle or reference) init."""
    spec = spec_from(z, prefix)
    model_seed, J, R, d_sub, tseed, head_seed, hidden, d_aux, sel = [int(x) for x in z[prefix + "init"]]
    tau, std = [float(x) for x in z[prefix + "init_f"]]
    w = impl.init_weights(spec, model_seed, tau, table=(J, R, d_sub, tseed, std), head_seed=head_seed,
                          hidden=hidden, d_aux=d_aux, sel=sel)
    return spec, w


def apply_overrides(z, w, prefix: str = ""):
    """The fixture's post-init edits: lifted wq/wk and explicit aux_proj."""
    if (prefix + "lift") in z.files and float(z[prefix + "lift"][0]) != 1.0:
        lift = np.float32(z[prefix + "lift"][0])
        base = (4 if w.spec.pos_learned else 3) + 12
        for l in range(w.spec.n_layers):
            w.tensors[base + 16 * l + 2] *= lift
            w.tensors[base + 16 * l + 4] *= lift
    if (prefix + "aux_proj") in z.files:
        w.head["aux_proj"][:] = z[prefix + "aux_proj"]
    return w


def ft_from(z, prefix: str = "") -> FinetuneSpec:
    v, use, me, da = [int(x) for x in z[prefix + "ft"]]
    return FinetuneSpec(variant=VARIANT_NAMES[v], use_seq_module=bool(use), max_events=me, d_aux=da)


VARIANT_NAMES = ["base", "aux", "aux-lt", "lite-mean", "lite-last"]  # FusionVariant order (finetune.hpp:29)


def names(z):
    return [str(x) for x in z["names"]]
