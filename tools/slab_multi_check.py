"""Multi-GPU check of the slab-decomposed Stokes solve on real NVLink peers
(torchrun, one rank per GPU, NCCL): the fused slab with the all_to_all exchange
and with the peer-memory exchange (torch symmetric memory rendezvous + its
device barrier; slab.SymmetricMemoryExchange) — cold start, then a warm start
from the first result — must agree with each other and with the single-GPU
fused solve of the whole cell (gathered on rank 0).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/slab_multi_check.py [--n 64] [--iters 30]

Exits 0 and prints one JSON line on rank 0 when everything matches."""

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=64)
    ap.add_argument("--iters", type=int, default=30)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2312_15554_b200 as pf
    from paper_2312_15554_b200 import slab as S
    from paper_2312_15554_b200.grid import rasterize_packing_slab, random_sphere_packing

    n = args.size
    dims = (n, n, n)
    lo, hi = S.slab_range(n, world, rank)
    solid = rasterize_packing_slab(random_sphere_packing(0), dims, lo, hi)
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0), max_iter=args.iters)
    out = {}
    for ex in ("a2a", "p2p"):
        st, rep = S.solve_stokes_slab(solid, dims, cfg, device=dev, fused=True, exchange=ex)
        host = {k: v.cpu().numpy() for k, v in st.items()}
        st2, rep2 = S.solve_stokes_slab(solid, dims, cfg, init_local=host, device=dev, fused=True, exchange=ex)
        out[ex] = (host, rep, {k: v.cpu().numpy() for k, v in st2.items()}, rep2)
    worst = 0.0
    for phase in (0, 2):
        for k in ("u", "u_tilde", "q", "a", "lam"):
            a, b = out["a2a"][phase][k], out["p2p"][phase][k]
            worst = max(worst, float(np.abs(a - b).max() / max(1e-300, np.abs(a).max())))
    same_hist = all(np.array_equal(out["a2a"][i].history, out["p2p"][i].history) for i in (1, 3))
    # gather u on rank 0 and compare with the single-GPU fused solve of the whole cell
    u_loc = torch.as_tensor(out["p2p"][0]["u"]).to(dev).contiguous()
    parts = [torch.empty_like(u_loc) for _ in range(world)]
    dist.all_gather(parts, u_loc)
    ok = worst <= 1e-13 and same_hist
    line = None
    if rank == 0:
        u_slab = np.concatenate([p.cpu().numpy() for p in parts], axis=1)
        ind = pf.random_packing_geometry(n, seed=0)
        st1, rep1 = pf.solve_stokes(ind, cfg)
        rel = float(np.linalg.norm(u_slab - st1.u) / np.linalg.norm(st1.u))
        ok = ok and rel <= 1e-11 and rep1.iterations == out["p2p"][1].iterations
        line = {"ranks": world, "n": n, "iters": args.iters, "p2p_vs_a2a_max_rel": worst,
                "history_bitwise_equal": same_hist, "slab_vs_single_gpu_rel_l2": rel, "ok": bool(ok)}
        print(json.dumps(line), flush=True)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    return 0 if int(flag.item()) else 1


if __name__ == "__main__":
    sys.exit(main())
