"""C-ABI boundary checks that need no GPU: the library builds for sm_100a, loads, exports
every function include/mpcgemm.h declares, the structs match the header layout, argument
validation happens on the host before any CUDA call, and the slice rule agrees with the
oracle's independent implementation."""
import ctypes
import os
import re
import subprocess

import pytest

import mpgen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpcgemm.h")


@pytest.fixture(scope="module")
def P():
    import __graft_entry__ as g
    g.build_lib()
    import paper_2307_06072_b200 as P
    return P


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|void|size_t|char)\s*\*?\s*(mpc\w*)\s*\(", txt, flags=re.M)))


def test_exports_every_declared_symbol(P):
    names = declared_functions()
    assert len(names) >= 10
    lib = ctypes.CDLL(P.mpcgemm.LIB_PATH)
    for nm in names:
        assert hasattr(lib, nm), nm
    out = subprocess.run(["nm", "-D", "--defined-only", P.mpcgemm.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mpc\w*)", out))
    assert set(names) <= exported
    assert set(P.mpcgemm.SYMBOLS) == set(names)


def test_library_is_sm100a_with_tensor_core_code(P):
    sass = subprocess.run(["cuobjdump", "-sass", P.mpcgemm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", P.mpcgemm.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass            # tcgen05.mma kind::i8
    assert "UTMALDG" in sass            # TMA tensor loads
    assert "LDTM" in sass               # tcgen05.ld (TMEM -> registers)
    deps = subprocess.run(["ldd", P.mpcgemm.LIB_PATH], capture_output=True, text=True).stdout
    assert "libtorch" not in deps and "python" not in deps


def _c_layout(struct, fields):
    """sizeof and offsetof of a header struct, from a C program compiled against the header."""
    import subprocess
    import tempfile
    inc = os.path.join(ROOT, "include")
    body = "".join(f'printf("%zu\\n", offsetof({struct}, {f}));' for f in fields)
    src = (f'#include <stdio.h>\n#include <stddef.h>\n#include "mpcgemm.h"\n'
           f'int main(void) {{ printf("%zu\\n", sizeof({struct})); {body} return 0; }}\n')
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
        open(c, "w").write(src)
        subprocess.check_call(["gcc", "-I", inc, "-o", exe, c])
        vals = [int(x) for x in subprocess.check_output([exe]).split()]
    return vals[0], vals[1:]


@pytest.mark.parametrize("name", ["RMatC", "CMatC", "OptsC", "ReportC"])
def test_struct_layout_matches_header(P, name):
    """The binding's ctypes structs have the header's size and field offsets."""
    M = P.mpcgemm
    cls = getattr(M, name)
    cname = {"RMatC": "mpc_rmat", "CMatC": "mpc_cmat", "OptsC": "mpcgemm_opts", "ReportC": "mpcgemm_report"}[name]
    fields = [f for f, _ in cls._fields_]
    size, offs = _c_layout(cname, fields)
    assert ctypes.sizeof(cls) == size
    assert [getattr(cls, f).offset for f in fields] == offs


def test_version_and_strerror(P):
    assert P.mpcgemm_version() == 100
    for code in (0, -1, -2, -3, -4, -5, -6, -7, -8):
        assert P.mpcgemm_strerror(code) != "unknown status"


def test_host_validation_before_cuda(P):
    """Errors found on the host return without touching the GPU (works with no GPU)."""
    M = P.mpcgemm
    lib = M.lib()
    z = M.CMatC()
    rep = M.ReportC()
    opts = M.OptsC()
    assert lib.mpcgemm_ex(2, 2, 2, 128, None, None, None, 3, ctypes.byref(opts), ctypes.byref(rep)) == -1
    a = M.CMatC()
    for part in (a.re, a.im):
        part.sign, part.exp, part.limbs, part.ld = 16, 32, 64, 2
    assert lib.mpcgemm_ex(2, 2, 2, 5000, ctypes.byref(a), ctypes.byref(a), ctypes.byref(z), 3, None, None) == -2
    assert lib.mpcgemm_ex(2, 2, 2, 128, ctypes.byref(a), ctypes.byref(a), ctypes.byref(z), 5, None, None) == -1
    assert lib.mpcgemm_ex(-1, 2, 2, 128, ctypes.byref(a), ctypes.byref(a), ctypes.byref(z), 3, None, None) == -1
    c = M.CMatC()
    for part in (c.re, c.im):
        part.sign, part.exp, part.limbs, part.ld = 16, 32, 64, 1       # ld < cols
    assert lib.mpcgemm_ex(2, 2, 2, 128, ctypes.byref(a), ctypes.byref(a), ctypes.byref(c), 3, None, None) == -1
    for part in (c.re, c.im):
        part.ld = 2                                                      # C aliases A
    assert lib.mpcgemm_ex(2, 2, 2, 128, ctypes.byref(a), ctypes.byref(a), ctypes.byref(c), 3, None, None) == -5
    opts.slices = 5000
    d = M.CMatC()
    for q, part in enumerate((d.re, d.im)):
        part.sign, part.exp, part.limbs, part.ld = 1 << 40, 1 << 41, 1 << 42, 2
    assert lib.mpcgemm_ex(2, 2, 2, 128, ctypes.byref(a), ctypes.byref(a), ctypes.byref(d), 3, ctypes.byref(opts), None) == -8


def test_slice_rule_matches_oracle(P):
    for prec in (2, 53, 128, 256, 512, 768, 1024, 2048, 4096):
        for method in ("3M", "4M"):
            for k, trip in ((64, (64 * 127 * 60, None, -1)), (2048, (2048 * 3000, None, -1)), (12, (0, 5, 20)),
                            (12, (0, -1, 7)), (3, (-1, -1, -1)), (1 << 17, (1, None, -1))):
                minT, minT1, maxD2 = trip
                minT1 = minT if minT1 is None else minT1
                s_lib = P.mpcgemm_slices_for(prec, method, k, minT, minT1, maxD2)
                s_orc = oracle.slices_for(prec, method, k, minT, minT1, maxD2)[0]
                assert s_lib == s_orc, (prec, method, k, trip)


def test_workspace_size_positive(P):
    assert P.mpcgemm_workspace_size(2048, 2048, 2048, 1024, "3M", 129) > 3 * 129 * 2048 * 2048
