"""Host-side checks that need no GPU: the C-ABI library builds for sm_100a, loads,
and exports every symbol include/hom2d.h declares; the header and the binding
agree on the config struct; the product never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1709_01619_b200 import build
    return build.build()


def header_functions():
    src = open(os.path.join(ROOT, "include", "hom2d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hom2d_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_binding_exports():
    import paper_1709_01619_b200 as P
    assert header_functions() == sorted(P.EXPORTS)


def test_library_exports_every_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    for name in header_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_config_struct_layout_matches_header():
    """The ctypes Config mirrors hom2d_config field by field (compiled probe)."""
    import paper_1709_01619_b200 as P
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "hom2d.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(hom2d_config), offsetof(hom2d_config, gamma),
         offsetof(hom2d_config, limiter_eps), offsetof(hom2d_config, record_decisions),
         offsetof(hom2d_config, limiter_per_step), offsetof(hom2d_config, limiter_characteristic),
         sizeof(hom2d_dist), offsetof(hom2d_dist, cuda_stream));
  printf("%zu %zu\n", offsetof(hom2d_config, fv_error_recon), offsetof(hom2d_config, dg_overintegrate));
  printf("%zu %zu %zu\n", sizeof(hom2d_peer_id_t), offsetof(hom2d_peer_id_t, offset), offsetof(hom2d_peer_id_t, rank));
  return 0;
}
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "p.c")
        exe = os.path.join(d, "p")
        open(src, "w").write(probe)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
        vals = [int(v) for v in subprocess.check_output([exe]).split()]
    C = P.Config
    D = P.Dist
    assert vals == [ctypes.sizeof(C), C.gamma.offset, C.limiter_eps.offset, C.record_decisions.offset,
                    C.limiter_per_step.offset, C.limiter_characteristic.offset, ctypes.sizeof(D), D.cuda_stream.offset,
                    C.fv_error_recon.offset, C.dg_overintegrate.offset,
                    ctypes.sizeof(P.PeerId), P.PeerId.offset.offset, P.PeerId.rank.offset]


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1709_01619_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "hom2d_oracle" not in txt, f


def test_missing_extension_fails_loudly(tmp_path):
    import paper_1709_01619_b200 as P
    saved = P._lib
    P._lib = None
    try:
        with pytest.raises(RuntimeError):
            P.load(str(tmp_path / "nope.so"))
    finally:
        P._lib = saved


@pytest.mark.parametrize("kw,status", [
    (dict(method="cpr", k=5), 3),                 # HOM2D_ERR_ORDER: k outside 1..4
    (dict(method="cpr", k=0), 3),
    (dict(method="fv", k=3), 3),                  # FV: 1 = MUSCL-2, 2 = MUSCL-3
    (dict(method=7, k=1), 1),                     # HOM2D_ERR_ARG: unknown method
    (dict(nx=1), 2),                              # HOM2D_ERR_MESH: nx < 2
    (dict(box=(1.0, 1.0, 0.0, 1.0)), 2),          # degenerate box
    (dict(gamma=1.0), 1),                         # gamma must exceed 1
    (dict(cfl=0.0), 1),
    (dict(bc=2), 1),
    (dict(limiter_per_step=2), 1),                # variant switches are 0/1
    (dict(fv_unlimited=5), 1),
    (dict(limiter_characteristic=-1), 1),
    (dict(fv_error_recon=2), 1),
    (dict(dg_overintegrate=3), 1),
])
def test_config_validation_status(kw, status):
    """hom2d_strip_plan validates the config on the host exactly as hom2d_create
    does: each bad field maps to its documented status (include/hom2d.h)."""
    import paper_1709_01619_b200 as P
    args = dict(nx=8, ny=8, method="cpr", k=1)
    args.update(kw)
    nx, ny = args.pop("nx"), args.pop("ny")
    cfg = P.make_config(nx, ny, **args)
    with pytest.raises(P.Hom2dError) as e:
        P.strip_plan(cfg, 0, 1)
    assert e.value.status == status
