"""CPU-side checks of the C-ABI boundary: the library builds, loads, exports every
symbol include/gist.h declares, and refuses to run without a B200 (no fallback)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gist.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gist_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2102_10424_b200 import build, gist
    build.build()
    return gist.lib()


def test_header_declares_north_star_calls():
    names = declared_symbols()
    for n in ["gist_load_graph", "gist_partition", "gist_subtrain", "gist_aggregate", "gist_eval"]:
        assert n in names


def test_library_exports_every_declared_symbol(L):
    from paper_2102_10424_b200 import gist
    names = declared_symbols()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(gist.EXPORTS) == names


def test_no_cpu_fallback_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2102_10424_b200.gist import Gist, GistError
    with pytest.raises(GistError, match="UNSUPPORTED"):
        Gist("gcn", [4, 8, 3])


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2102_10424_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
