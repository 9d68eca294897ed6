"""C-ABI checks that need no GPU: libsks.so builds/loads, exports every symbol
include/sks.h declares, host-only entry points behave, and the product's partition
agrees with the input generator's."""
import ctypes as C
import os
import re

import pytest

from conftest import HAS_CUDA, ROOT

HDR = os.path.join(ROOT, "include", "sks.h")


def _declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"\b(sks_[a-z_]+)\s*\(", txt)))


def test_header_and_binding_agree():
    import paper_2111_00113_b200 as P
    assert sorted(P.EXPORTS) == _declared()


def test_library_exports_every_declared_symbol():
    import paper_2111_00113_b200 as P
    from paper_2111_00113_b200 import build
    build.build()
    lib = C.CDLL(P.LIBPATH)
    for name in _declared():
        assert hasattr(lib, name), name
    import re
    hdr = open(os.path.join(ROOT, "include", "sks.h")).read()
    assert P.load().sks_abi_version() == int(re.search(r"#define SKS_ABI_VERSION (\d+)", hdr).group(1))


def test_partition_matches_inputs_and_covers():
    import paper_2111_00113_b200 as P
    from inputs import partition_rows
    for kind, m, n in [("stencil2d", 2048, 2048 ** 2), ("stencil3d", 160, 160 ** 3), ("csr", 0, 2_000_000),
                       ("stencil2d", 33, 33 * 33)]:
        for nr in (1, 2, 3, 4, 8):
            prev = 0
            for r in range(nr):
                lo, hi = P.partition(kind, m, n, nr, r)
                assert (lo, hi) == partition_rows(kind, n, m, nr, r)
                assert lo == prev and hi > lo
                prev = hi
            assert prev == n


def test_unique_id_without_gpu():
    import paper_2111_00113_b200 as P
    uid = P.get_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128


@pytest.mark.skipif(HAS_CUDA, reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    import paper_2111_00113_b200 as P
    with pytest.raises(P.SksError) as e:
        P.Context(0)
    assert "SKS_ECUDA" in str(e.value)
