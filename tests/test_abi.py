"""CPU-side checks of the boundary: the library builds, loads and exports every
symbol include/lcp.h declares; the product path fails loudly without a GPU;
the product package never imports the oracle."""
import ast
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_build_and_exports():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2512_12442_b200 import EXPORTS, load_library
    L = load_library()
    header = open(os.path.join(ROOT, "include", "lcp.h")).read()
    declared = set(re.findall(r"^\s*(?:lcp_status_t|void|const char\*|int32_t)\s+(lcp_\w+)\s*\(", header, re.M))
    assert declared == set(EXPORTS), declared ^ set(EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


def test_no_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2512_12442_b200 import Context, LcpError
    with pytest.raises((LcpError, RuntimeError, AssertionError)):
        Context(0)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2512_12442_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), p
            if f.endswith((".cu", ".cuh", ".h", ".py")):
                src = open(p).read()
                assert "lcp_oracle" not in src and "orc_" not in src, p


def test_oracle_and_cuda_share_no_source():
    csrc = os.path.join(ROOT, "paper_2512_12442_b200", "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f)).read()
        incs = re.findall(r"#include\s+[\"<]([^\">]+)", src)
        assert not any("oracle" in i for i in incs), (f, incs)
    osrc = open(os.path.join(ROOT, "oracle", "lcp_oracle.c")).read()
    assert "lcp.h" not in osrc and "csrc" not in osrc
