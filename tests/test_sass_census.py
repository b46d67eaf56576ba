"""The built library is Blackwell-native (CPU test: cuobjdump reads the sm_100a
cubins without a GPU). The hot kernels' SASS holds the instructions that prove
it -- UTCHMMA (tcgen05.mma), UTMALDG (TMA tensor loads), LDTM (tcgen05.ld),
UBLKCP (cp.async.bulk), SYNCS (mbarriers) -- and no legacy HMMA tensor path;
the PageRank gather's exchange epilogue holds the system-scope store
(`multimem.st` compiles to STG.E.STRONG.SYS on the multicast address).
Skipped when the library is not built or cuobjdump is absent."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2005_08466_b200", "_lib", "libhaocl_b200.so")


@pytest.fixture(scope="module")
def sass():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(tool):
        pytest.skip("library not built or cuobjdump missing")
    out = subprocess.run([tool, "-sass", LIB], capture_output=True, text=True, timeout=600).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return funcs


def census(funcs, pattern):
    hits = {k: v for k, v in funcs.items() if re.search(pattern, k)}
    assert hits, f"no kernel matches {pattern}"
    ops = {}
    for lines in hits.values():
        for line in lines:
            m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
            if m:
                ops[m.group(1)] = ops.get(m.group(1), 0) + 1
    return ops


@pytest.mark.parametrize("kernel,need", [
    ("gemm_tc_kernel", ("UTCHMMA", "UTMALDG", "LDTM", "SYNCS")),
    ("conv3x3_v3_kernel", ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM")),
    ("kmeans_assign_tc_kernel", ("UTCHMMA", "UTMALDG", "LDTM", "FMNMX3")),
    ("pr_bin_scatter_kernel", ("UBLKCP", "SYNCS")),
    ("pr_bin_gather_kernel", ("UBLKCP", "ATOMS")),
    ("kmeans_accumulate32_bulk_kernel", ("UBLKCP", "ATOMS")),
])
def test_hot_kernels_are_blackwell_native(sass, kernel, need):
    ops = census(sass, kernel)
    for op in need:
        assert ops.get(op, 0) > 0, f"{kernel}: no {op} in its SASS ({sorted(ops)[:40]})"
    assert ops.get("HMMA", 0) == 0, f"{kernel}: legacy HMMA tensor path"


def test_pagerank_exchange_store_is_system_scope(sass):
    lines = [l for k, v in sass.items() if "pr_bin_gather_kernel" in k for l in v]
    assert any("STG.E.STRONG.SYS" in l for l in lines), "no system-scope (multicast / peer) store in the gather"
