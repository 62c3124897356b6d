"""Parity helpers: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs. Tolerances (DESIGN.md §2 A25): pool, CSIP ip and NAT bit-exact;
estimates within 1e-6 relative (+1e-9 absolute near 0); the ABOVE_THETA flag equal
unless |est - theta| / theta < 1e-12 (tie band)."""
import numpy as np
import torch

from paper_1807_01527_b200 import asse

REL_TOL = 1e-6
ABS_TOL = 1e-9


def to_device(pk, offset_packets=0):
    """Host (n,2) uint32 -> device int32 tensor; optional leading pad to misalign."""
    t = torch.from_numpy(pk.view(np.int32).reshape(-1))
    if offset_packets:
        pad = torch.zeros(2 * offset_packets, dtype=torch.int32)
        t = torch.cat([pad, t])
    d = t.cuda()
    return d, d.data_ptr() + 8 * offset_packets


def compare_reports(dev, ora, theta, ctx=""):
    assert len(dev) == len(ora), "%s |CSIP| %d vs oracle %d" % (ctx, len(dev), len(ora))
    if len(ora) == 0:
        return
    assert (dev["ip"] == ora["ip"]).all(), ctx + " CSIP ip differ"
    assert (dev["nat"] == ora["nat"]).all(), ctx + " NAT differ"
    e1, e2 = dev["estimate"], ora["estimate"]
    inf = np.isinf(e2)
    assert (np.isinf(e1) == inf).all(), ctx + " saturation differs"
    f = ~inf
    err = np.abs(e1[f] - e2[f])
    assert (err <= REL_TOL * np.abs(e2[f]) + ABS_TOL).all(), ctx + " estimate max err %g" % err.max()
    sat1, sat2 = dev["flags"] & 1, ora["flags"] & 1
    assert (sat1 == sat2).all()
    ab1, ab2 = dev["flags"] & 2, ora["flags"] & 2
    tie = np.zeros(len(ora), bool)
    tie[f] = np.abs(e2[f] - theta) / theta < 1e-12
    assert ((ab1 == ab2) | tie).all(), ctx + " theta flag differs"


def compare_pool(dev_pool, ora_pool, ctx=""):
    if not (dev_pool == ora_pool).all():
        bad = np.argwhere(dev_pool != ora_pool)
        y, z, x, i = bad[0]
        raise AssertionError("%s pool differs at %d ATs, first [y=%d z=%d x=%d i=%d]: dev %d oracle %d"
                             % (ctx, len(bad), y, z, x, i, dev_pool[y, z, x, i], ora_pool[y, z, x, i]))


def step_both(dev, ora, pk, theta, ctx, check_pool=True, mode=1, split=1, offset=0):
    """Scan one slice on both sides, close it, compare reports and the post-advance pool."""
    d_pk, ptr = to_device(pk, offset)
    n = len(pk)
    if split <= 1:
        dev.scan_slice(ptr, n)
    else:
        cuts = np.linspace(0, n, split + 1).astype(np.int64)
        for a, b in zip(cuts[:-1], cuts[1:]):
            dev.scan_slice(ptr + 8 * int(a), int(b - a))
    ora.scan(pk)
    rep_o = ora.end_slice(mode)
    rep_d = dev.end_slice(mode)
    torch.cuda.synchronize()
    del d_pk
    compare_reports(rep_d, rep_o, theta, ctx)
    if check_pool:
        compare_pool(dev.pool(), ora.pool(), ctx)
    return rep_d, rep_o
