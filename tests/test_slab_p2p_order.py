"""Host-side ordering of the fused slab's p2p exchange (no GPU).

In the p2p mode PK and MF store straight into the owning ranks' Y buffers, so
the host driver must put a cross-rank barrier between every rank's own writes to
a buffer and the first remote store into it, and between the stores and the
consuming pass (``slab.FusedSlabStokes``).  A recording backend and communicator
check that order for a cold start and two iterations."""

import numpy as np
import torch

import paper_2312_15554_b200 as pf
from paper_2312_15554_b200.slab import FusedSlabStokes


class _Rec:
    def __init__(self):
        self.log = []


class _Backend:
    def __init__(self, rec):
        self.rec = rec

    def __getattr__(self, name):  # every other device call: record and do nothing
        def call(*a, **k):
            self.rec.log.append(name)
        return call

    def fused_sizes(self):
        return (6, 2)

    def alloc_real(self, count):
        return torch.zeros(count, dtype=torch.float64)

    def alloc_complex(self, count):
        return torch.zeros(2 * count, dtype=torch.float64)

    def read(self):
        self.rec.log.append("read")
        return {"done": False, "iter": 0}


class _Comm:
    def __init__(self, rec, world=2):
        self.rec, self.world = rec, world

    def get_world_size(self, group=None):
        return self.world

    def get_rank(self, group=None):
        return 0

    def p2p_alloc(self, numel, device):
        return torch.zeros(numel, dtype=torch.float64)

    def p2p_ptrs(self, buf):
        return [buf.data_ptr()] * self.world

    def p2p_barrier(self):
        self.rec.log.append("barrier")

    def all_reduce(self, t, group=None):
        self.rec.log.append("all_reduce")

    def all_to_all_single(self, out, inp, group=None, async_op=False):
        self.rec.log.append("all_to_all")


def test_p2p_cold_start_and_iteration_order():
    rec = _Rec()
    n = 8
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0), max_iter=4)
    z3 = torch.zeros((3, n // 2, n, n), dtype=torch.float64)
    state = {"u": z3.clone(), "u_tilde": z3.clone(), "q": torch.zeros((n // 2, n, n), dtype=torch.float64),
             "a": z3.clone(), "lam": z3.clone()}
    solid = torch.zeros((n // 2, n, n), dtype=torch.uint8)
    s = FusedSlabStokes(_Backend(rec), (n, n, n), cfg, None, solid, state, comm=_Comm(rec), exchange="p2p")
    assert s.p2p
    s.begin()
    s.iterate(2, poll=False)
    log = [e for e in rec.log if e in ("fused_setup_zero", "fused_pk", "fused_rs", "finalize", "fused_mf",
                                       "barrier", "all_reduce")]
    z = log.index("fused_setup_zero")
    first_pk = log.index("fused_pk")
    assert "barrier" in log[z:first_pk], log  # owners' zeroing before any remote PK store
    body = log[first_pk:]
    assert body == ["fused_pk", "barrier", "fused_rs", "all_reduce", "finalize", "fused_mf", "barrier"] * 2, body
    assert np.isfinite(float(s.totals.sum()))
