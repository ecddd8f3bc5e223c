"""Register-spill guard for the hot kernels (CPU; reads the ptxas -v log of the in-tree build).

The depth sweep and the backward sweep run at the 80-register cap of 3 CTAs x 256 threads per SM, where a
small unrelated change (a field inserted into RasterArgs, one more compare in a shared helper) has flipped
ptxas into hundreds of bytes of local-memory spills (profiles/r01/evolution.md)."""
import os
import re

import pytest

from paper_2110_06635_b200 import build as B

LOG = os.path.join(B.PKG, "build", "ptxas.log")
HOT = B.HOT


def _spills():
    out, cur = {}, None
    for line in open(LOG):
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores", line)
        if m and cur:
            out[cur] = int(m.group(1))
    return out


@pytest.mark.skipif(not os.path.exists(LOG), reason="no in-tree build log (python -m paper_2110_06635_b200.build)")
def test_hot_kernels_do_not_spill():
    sp = _spills()
    for fn, limit in HOT.items():
        assert fn in sp, fn
        assert sp[fn] <= limit, f"{fn}: {sp[fn]} bytes of spill stores (limit {limit})"
