"""The slab-partitioned CUDA engine (csrc/comm.cu, halo exchange + global
sums) on several ranks reproduces the single-rank run: same Newton/Krylov
counts and the same final state to rounding.  Ranks share one GPU through the
host-callback transport (gloo), so no kernel waits on another rank."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(tmp_path, nproc, *args, env=None):
    out = tmp_path / "mr.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "multirank_worker.py"),
           "--out", str(out), *args]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=dict(os.environ, **(env or {})))
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    with open(out) as fh:
        return json.load(fh)


@pytest.mark.parametrize("nproc,args", [
    (2, ["--kind", "burgers", "--shape", "64,64", "--family", "gauss", "--stages", "3"]),
    (2, ["--kind", "nldiff", "--shape", "48,40", "--family", "radau_iia", "--stages", "3",
         "--dt", "2e-4"]),
    (3, ["--kind", "nldiff", "--shape", "16,14,24", "--family", "gauss", "--stages", "2",
         "--dt", "1e-3"]),
    # nx >= 64: the communication-avoiding step (one v_j halo of depth 2(K-1)+1, the chains
    # compute the ghost rows of z1 / z2 themselves); ragged slabs of 17 / 17 / 16 rows
    (3, ["--kind", "burgers", "--shape", "64,50", "--family", "gauss", "--stages", "3"]),
    (3, ["--kind", "nldiff", "--shape", "96,50", "--family", "radau_iia", "--stages", "2",
         "--dt", "2e-4"]),
    # other sweep counts: K = 2 (v_j halo of 3 planes) and K = 6 (2(K-1)+1 = 11 planes exceed the
    # ghost buffers: the step falls back to exchanging z1 / z2)
    (2, ["--kind", "burgers", "--shape", "64,48", "--family", "gauss", "--stages", "2",
         "--inner", "2"]),
    (2, ["--kind", "burgers", "--shape", "64,48", "--family", "gauss", "--stages", "2",
         "--inner", "1"]),
    (2, ["--kind", "nldiff", "--shape", "64,48", "--family", "gauss", "--stages", "2",
         "--dt", "2e-4", "--inner", "6"]),
    # in-plane extents >= 32: the 3.5-D blocked chain (csrc/jacobi3d.cu) on z-slabs with ghost planes
    (2, ["--kind", "nldiff", "--shape", "32,34,16", "--family", "gauss", "--stages", "2",
         "--dt", "1e-3"]),
    # the vorticity DAE: 9-point stencils on slabs + the gathered constraint solve
    (2, ["--kind", "arakawa", "--shape", "40,40", "--family", "gauss", "--stages", "2",
         "--dt", "2e-3"]),
    (3, ["--kind", "arakawa", "--shape", "32,36", "--family", "gauss", "--stages", "4",
         "--dt", "2e-3"]),
    # nx >= 64: the warp-strip Arakawa chain (csrc/arachain.cu k_ara_sp2d) on slabs with ghost rows
    (2, ["--kind", "arakawa", "--shape", "64,48", "--family", "gauss", "--stages", "2",
         "--dt", "2e-3"]),
])
def test_slab_partition_matches_single_rank(tmp_path, nproc, args):
    r = _run(tmp_path, nproc, *args)
    assert r["rel"] <= 1e-12, r
    assert len(r["stats"]) == len(r["single_stats"])
    for got, want in zip(r["stats"], r["single_stats"]):
        assert got[0] == want[0], (got, want)
        assert abs(got[1] - want[1]) <= 1, (got, want)
    assert r["halos"] > 0


def test_nccl_transport_single_gpu_ring(tmp_path):
    """The native NCCL transport (dlopen'ed libnccl, grouped send/recv halos,
    ncclAllReduce) on a 1-rank ring: slab mode forced, ghost planes arrive
    through NCCL self send/recv; must equal the plain periodic run."""
    r = _run(tmp_path, 1, "--kind", "burgers", "--shape", "64,64", "--transport", "nccl",
             env={"IRKG_FORCE_SLAB": "1"})
    assert r["rel"] <= 1e-12, r
    assert [s[0] for s in r["stats"]] == [s[0] for s in r["single_stats"]]
    assert r["halos"] > 0


def test_slab_step_with_exchanged_z_halos_matches(tmp_path):
    """IRKG_EXT_HALO=0: the step that exchanges the halos of z1 and z2 instead of
    computing their ghost rows (the path 3-D grids and narrow 2-D grids take)."""
    r = _run(tmp_path, 2, "--kind", "burgers", "--shape", "64,64", "--family", "gauss",
             "--stages", "3", env={"IRKG_EXT_HALO": "0"})
    assert r["rel"] <= 1e-12, r
    assert all(abs(a[1] - b[1]) <= 1 for a, b in zip(r["stats"], r["single_stats"]))


def test_nccl_ring_with_halo_overlap_matches(tmp_path):
    """The interior/edge band split with the halos on a side stream
    (IRKG_HALO_OVERLAP=1: fork/join inside the captured step graph) gives the
    same step as the plain periodic run (forced 1-rank NCCL ring)."""
    r = _run(tmp_path, 1, "--kind", "burgers", "--shape", "128,96", "--transport", "nccl",
             env={"IRKG_FORCE_SLAB": "1", "IRKG_HALO_OVERLAP": "1"})
    assert r["rel"] <= 1e-12, r
    assert [s[0] for s in r["stats"]] == [s[0] for s in r["single_stats"]]
    assert all(abs(a[1] - b[1]) <= 1 for a, b in zip(r["stats"], r["single_stats"]))
    assert r["halos"] > 0


def test_nccl_ring_dae_transposed_constraint_solve(tmp_path):
    """The DAE step over the native NCCL transport on a forced 1-rank slab:
    9-point stencils through NCCL ghost planes and the constraint solve's
    slab -> pencil transposes through NcclComm::alltoall (grouped self
    send/recv); must equal the plain single-rank run (2-D cuFFT solve)."""
    r = _run(tmp_path, 1, "--kind", "arakawa", "--shape", "40,36", "--family", "gauss",
             "--stages", "2", "--dt", "2e-3", "--transport", "nccl",
             env={"IRKG_FORCE_SLAB": "1"})
    assert r["rel"] <= 1e-12, r
    assert [s[0] for s in r["stats"]] == [s[0] for s in r["single_stats"]]
    assert all(abs(a[1] - b[1]) <= 1 for a, b in zip(r["stats"], r["single_stats"]))
    assert r["halos"] > 0
