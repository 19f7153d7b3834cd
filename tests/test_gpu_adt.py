"""The paper's transfer model, Eq. 1 (SPEC S:L371-409
sdt_makespan / adt_makespan), on the library's host pipeline
(hamming_decode_host): stage times measured per chunk
predict the measured SDT (1 stream) and ADT (3 streams) makespans within
30 %, and ADT beats SDT (overlap never hurts).  The band is wide
because host-link timings move from box to box (SDT measured from 2 % above
to 23 % below the model of its own stage times), and the three-stage pipeline
model takes the H2D and D2H engines as independent full-rate links
while concurrent they share the host's PCIe/memory path (ADT 8-16 % above the
model, profiles/r02_adt_eq1.md).  The full table is
tools/adt_eq1.py -> profiles/r02_adt_eq1.md."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.mark.parametrize("m,chunk,n_chunks", [(6, 1 << 22, 12), (4, 1 << 23, 12)])
def test_eq1_makespans_match_measured_stages(m, chunk, n_chunks):
    """Host-link timings vary from box to box and call to call (the stage times are medians of
    single-stage runs, the makespans wall clock): up to three measurements, the first inside the
    bands counts; the structural claims must hold on every one."""
    import adt_eq1
    rs = []
    for _ in range(3):
        r = adt_eq1.model(m, chunk, n_chunks)
        assert r["adt"] < r["sdt"] and r["speedup"] > 1.3, r
        # the link dominates (the paper's own regime: T_PS + T_PR >= T_DKE)
        assert r["t_ps"] + r["t_pr"] >= r["t_dke"], r
        rs.append(r)
        if abs(r["sdt"] / r["sdt_pred"] - 1) < 0.30 and abs(r["adt"] / r["adt_pred"] - 1) < 0.30:
            return
    raise AssertionError(f"Eq. 1 predictions off by more than 30 % in three measurements: {rs}")
