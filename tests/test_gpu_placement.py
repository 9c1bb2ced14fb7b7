"""GPU-offloaded placements of the paper's CT (§4
L320-330): CT^u (device update, host filter), CT^f (host update, device
filter), CT^uf (both on the device, the paper's per-call transfers) -- every
call vs the oracle, bit-exact, plus their transfer accounting."""
import numpy as np
import pytest

from paper_2507_18413_b200 import CT_OK, HostTable
from test_host_ct import host_walk, table1_exhaustive, POLICIES
from workloads import random_table, banded_table, table1, knapsack_table

pytestmark = pytest.mark.gpu
PLACES = ["u", "f", "uf"]


@pytest.mark.parametrize("place", PLACES)
def test_placement_table1_exhaustive(place):
    p = table1()
    tab = HostTable(p.lo, p.d, p.tuples, placement=place)
    table1_exhaustive(tab, p)
    tab.close()


@pytest.mark.parametrize("place", PLACES)
@pytest.mark.parametrize("shape", [(5, 12, 3000, -4), (1, 9, 40, 0), (2, 70, 700, 3), (3, 130, 5000, 0),
                                   (4, 20, 4096 * 5 + 17, 1), (6, 16, 300_077, 0)])
def test_placement_walks(shape, place):
    n, d, t, lo = shape
    p = random_table(n, d, t, seed=n * 1000 + d, lo=lo)
    tab = HostTable(p.lo, p.d, p.tuples, placement=place)
    host_walk(tab, p, calls=120, seed=3)
    tab.close()


@pytest.mark.parametrize("place", PLACES)
@pytest.mark.parametrize("pol", ["dom", "delta"])
def test_placement_policies(place, pol):
    p = random_table(5, 20, 20_000, seed=17)
    tab = HostTable(p.lo, p.d, p.tuples, placement=place, **POLICIES[pol])
    host_walk(tab, p, calls=100, seed=5)
    tab.close()


@pytest.mark.parametrize("place", PLACES)
def test_placement_config2_lin_banded(place):
    p = random_table(5, 20, 100_000, seed=1)
    tab = HostTable(p.lo, p.d, p.tuples, placement=place)
    assert host_walk(tab, p, calls=300, seed=2) > 0
    st = tab.stats()
    assert st["calls"] > 0 and st["h2d_bytes"] > 0 and st["d2h_bytes"] > 0 and st["kernel_launches"] > 0
    assert st["kernel_ms"] > 0 and st["h2d_ms"] > 0
    tab.close()
    from workloads import LIN_PRESETS
    p = knapsack_table(seed=21, **LIN_PRESETS["lin_b"])
    tab = HostTable(p.lo, p.d, p.tuples, placement=place)
    host_walk(tab, p, calls=100, seed=31)
    tab.close()
    p = banded_table(5, 30, 20000, seed=4)
    tab = HostTable(p.lo, p.d, p.tuples, placement=place)
    host_walk(tab, p, calls=100, seed=8, m=1, q=0.8)
    tab.close()
