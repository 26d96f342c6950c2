"""Worker for the multi-rank GPU test (launched by torch.distributed.run).

Every rank runs the slab-partitioned CUDA engine on its slab (host-callback
transport over gloo, so several ranks can share one GPU without any kernel
waiting on another rank); rank 0 also runs the same integration on one rank
and writes both results to ``--out``.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="burgers")
    ap.add_argument("--shape", default="64,64")
    ap.add_argument("--family", default="gauss")
    ap.add_argument("--stages", type=int, default=3)
    ap.add_argument("--dt", type=float, default=5e-4)
    ap.add_argument("--nsteps", type=int, default=2)
    ap.add_argument("--transport", default="callback")
    ap.add_argument("--inner", type=int, default=4)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_2101_01776_b200 as pk
    from paper_2101_01776_b200.distributed import SlabContext, gather, scatter

    rank = int(os.environ["RANK"])
    ws = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    backend = "gloo" if args.transport == "callback" else "nccl"
    dist.init_process_group(backend)
    shape = tuple(int(x) for x in args.shape.split(","))
    dae = args.kind == "arakawa"
    if dae:
        # vorticity/streamfunction DAE (configs[4] form): state [omega; psi],
        # each slab-partitioned; the constraint solve is a slab -> pencil transpose FFT
        prob = pk.VorticityProblem(shape, nu=1e-3)
        w0, p0 = pk.vorticity_initial_state(prob, seed=3)
        u0 = np.concatenate([w0, p0])
    else:
        params = {"burgers": dict(nu=1e-2), "nldiff": {}, "rad": dict(nu=0.01, c=0.3, lam=-0.2)}
        prob = pk.GridProblem(args.kind, shape, **params[args.kind])
        u0 = pk.fourier_u0(shape, 1, 4, 0.5 if args.kind == "burgers" else 0.1, 0)
    n_glob = int(np.prod(shape))

    def local_of(vec):
        if not dae:
            return scatter(vec, shape, rank, ws)
        return np.concatenate([scatter(vec[:n_glob], shape, rank, ws),
                               scatter(vec[n_glob:], shape, rank, ws)])

    def global_of(parts):
        if not dae:
            return gather(parts, shape)
        halves = [np.split(p, 2) for p in parts]
        return np.concatenate([gather([h[0] for h in halves], shape),
                               gather([h[1] for h in halves], shape)])

    def advance(c, x, t):
        return c.dae_step_device(x, t, args.dt) if dae else c.step_device(x, t, args.dt)

    tab = pk.make_tableau(args.family, args.stages)
    prep = pk.prepare_stages(tab)
    cfg = pk.SolverConfig(krylov_maxit=5000, precond=pk.PrecondSpec(inner=args.inner))

    ctx = SlabContext(prob, rank, ws, transport=args.transport)
    ctx.set_prep(prep)
    ctx.set_config(cfg)
    u = torch.from_numpy(np.ascontiguousarray(local_of(u0))).cuda()
    stats = []
    for j in range(args.nsteps):
        st = advance(ctx, u, j * args.dt)
        stats.append([st.newton_iterations, st.krylov_iterations,
                      {str(k): v for k, v in st.block_iterations.items()}])
    local = u.cpu().numpy()
    parts = [None] * ws
    dist.all_gather_object(parts, local)
    halos = ctx.counters()["halo_exchanges"]
    ctx.close()
    if rank == 0:
        uglob = global_of(parts)
        from paper_2101_01776_b200.engine import Context

        single = Context(prob)
        single.set_prep(prep)
        single.set_config(cfg)
        us = torch.from_numpy(u0).cuda()
        sstats = []
        for j in range(args.nsteps):
            st = advance(single, us, j * args.dt)
            sstats.append([st.newton_iterations, st.krylov_iterations,
                           {str(k): v for k, v in st.block_iterations.items()}])
        ref = us.cpu().numpy()
        rel = float(np.linalg.norm(uglob - ref) / np.linalg.norm(ref))
        with open(args.out, "w") as fh:
            json.dump({"rel": rel, "stats": stats, "single_stats": sstats, "halos": halos,
                       "world": ws}, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
