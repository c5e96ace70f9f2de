"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/dcat_b200.h declares; struct layouts agree with the header;
host-side input builders behave like the reference's Segment rules."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2507_12704_b200 import abi
from paper_2507_12704_b200.synth import make_batch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dcat_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2507_12704_b200 import api
    if not os.path.exists(api.LIB_PATH):
        import paper_2507_12704_b200 as pkg
        pkg.build()
    return api.lib()


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dcat_\w+)\s*\(", text, re.M)))


def test_exports_every_declared_symbol(lib):
    from paper_2507_12704_b200 import api
    names = declared_functions()
    assert len(names) >= 8
    for n in names:
        assert hasattr(lib, n), f"libdcat_b200.so does not export {n}"
    assert set(names) == set(api.EXPORTS)
    assert lib.dcat_version().startswith(b"dcat_b200")


def test_struct_layouts_match_header(tmp_path):
    """Compile the real header with gcc and compare every field offset with ctypes."""
    structs = {"dcat_model_config": abi.ModelConfigC, "dcat_params": abi.ParamsC, "dcat_table": abi.TableC,
               "dcat_head": abi.HeadC, "dcat_finetune_config": abi.FinetuneConfigC, "dcat_batch": abi.BatchC,
               "dcat_call_stats": abi.CallStatsC}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    import subprocess
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l}
    for cname, cls in structs.items():
        assert got[(cname, "size")] == C.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert got[(cname, f)] == getattr(cls, f).offset, (cname, f)


def test_errors_without_gpu_are_reported_not_crashed(lib):
    # null arguments are validated before any CUDA call
    assert lib.dcat_rank_forward_batch(None, None, None, None, None, None, 0, None) == -1
    assert b"null" in lib.dcat_last_error()


def test_param_shapes_follow_all_params_order():
    spec = abi.ModelSpec(d_model=32, n_layers=2, n_heads=4, mlp_ratio=4, max_len=10, d_emb=16)
    shapes = spec.param_shapes()
    assert len(shapes) == 3 + 1 + 12 + 16 * 2
    assert shapes[4] == (16, 32)  # phi_in.w1: d_emb x d_model
    assert shapes[16 + 12] == (32, 128)  # layer0.fw1


def test_make_batch_layouts():
    b = make_batch(5, 3, 7, seed=1, layout="interleaved")
    assert b.n_rows == 15
    assert (b.row_offset[:5] == b.row_offset[5:10]).all()  # rep[b] = b % U shares storage
    g = make_batch(5, 3, 7, seed=1, layout="grouped", shared_storage=False)
    assert g.n_events == 15 * 7
    np.testing.assert_array_equal(g.ev_item[:7], g.ev_item[7:14])  # private copies, equal content
