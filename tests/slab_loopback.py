"""In-process loopback communicator: P slab ranks as P host threads on ONE GPU.

Each rank thread drives its own device backend (plan, buffers); the collectives
are host-synchronised -- every rank finishes its device work (stream sync) and
meets at a barrier, the exchange is done with device-to-device copies in a fixed
order, and a second barrier releases the ranks.  No kernel ever waits on another
rank's kernel, so this is a faithful single-GPU test of the per-rank device
logic (slab offsets, zero-mode ownership, pack/unpack) at P > 1, not a stand-in
for multi-GPU timing.  Test infrastructure only.
"""

import threading


class LoopbackHub:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.error = None

    def rank(self, r):
        return _RankComm(self, r)


class _RankComm:
    def __init__(self, hub, rank):
        self.hub, self.r = hub, rank

    def get_world_size(self, group=None):
        return self.hub.world

    def get_rank(self, group=None):
        return self.r

    def is_initialized(self):
        return True

    def _meet(self):
        self.hub.barrier.wait(timeout=300)

    def all_to_all_single(self, recv, send, group=None, async_op=False):
        import torch

        h, w = self.hub, self.hub.world
        torch.cuda.synchronize()
        h.slots[self.r] = send
        self._meet()
        k = send.numel() // w
        for s in range(w):  # block s of my recv = block r of rank s's send
            recv[s * k:(s + 1) * k].copy_(h.slots[s][self.r * k:(self.r + 1) * k])
        torch.cuda.synchronize()
        self._meet()
        return _Done() if async_op else None

    # peer-memory exchange: every rank's buffers live on the one GPU, so their
    # plain device addresses serve as the P2P-mapped peer addresses
    def p2p_alloc(self, numel, device):
        import torch

        return torch.empty(numel, dtype=torch.float64, device=device)

    def p2p_ptrs(self, buf):
        h = self.hub
        h.slots[self.r] = buf.data_ptr()
        self._meet()
        ptrs = list(h.slots)
        self._meet()
        return ptrs

    def p2p_barrier(self):
        import torch

        torch.cuda.synchronize()
        self._meet()

    def all_reduce(self, t, group=None):
        import torch

        h = self.hub
        torch.cuda.synchronize()
        h.slots[self.r] = t.clone()
        self._meet()
        tot = h.slots[0].clone()
        for s in range(1, h.world):  # fixed order: identical totals on every rank
            tot += h.slots[s]
        self._meet()
        t.copy_(tot)
        torch.cuda.synchronize()


class _Done:
    """Handle of an exchange the loopback already completed (async_op=True)."""

    def wait(self):
        return True


def run_ranks(world, fn):
    """Run fn(rank, comm) on ``world`` threads; returns the per-rank results."""
    hub = LoopbackHub(world)
    out, errs = [None] * world, [None] * world

    def body(r):
        try:
            out[r] = fn(r, hub.rank(r))
        except BaseException as e:  # noqa: BLE001  (re-raised below)
            errs[r] = e
            hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errs:
        if e is not None:
            raise e
    return out


class SoloComm:
    """Rank ``rank`` of a ``world``-rank slab decomposition run ALONE: the other
    ranks' exchange blocks arrive as zeros and contribute nothing to the
    all-reduce.  Both device slab pipelines then compute the same well-defined
    map (the iteration with the other ranks' fields held at zero), so comparing
    them validates the per-rank kernels of a decomposition whose full cell does
    not fit one GPU (1024^3), and the rank's compute time is the per-GPU share
    of that decomposition.  Test / measurement infrastructure only."""

    def __init__(self, world, rank=0):
        self.world, self.r = world, rank

    def get_world_size(self, group=None):
        return self.world

    def get_rank(self, group=None):
        return self.r

    def is_initialized(self):
        return True

    def all_to_all_single(self, recv, send, group=None, async_op=False):
        k = send.numel() // self.world
        recv.zero_()
        recv[self.r * k:(self.r + 1) * k].copy_(send[self.r * k:(self.r + 1) * k])
        return _Done() if async_op else None

    def all_reduce(self, t, group=None):
        return None
