"""Two real processes, one GPU: the row-distributed setup and solve of
libpmgr (pmgr_dist_setup / pmgr_dist_gmres) driven end to end over a
torch.distributed gloo group through the host-staged transport
(dist.host_transport), checked against the CPU oracle.

The transport stages every exchange through host memory and synchronises
the stream, so no kernel ever waits on the other process; the exchange
pattern (halo point-to-point, all-gather of the collapsed coarse right-hand
side, all-reduces of the Krylov projections, the setup's status exchanges and
row fetches) is the one the NCCL transport runs on a multi-GPU node."""

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import os, sys, json
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch
import torch.distributed as tdist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
tdist.init_process_group("gloo")
torch.cuda.set_device(0)
from paper_1904_05960_b200 import dist as D, krylov, mgr, problems, sparse
name = sys.argv[2]
if name == "C5":
    base = problems.make_c5(seed=4, nxy=10, nz_per_gpu=5, gpus=2)
elif name == "C3":
    base = problems.make("C3", seed=4, n=8)
else:
    base = problems.make_c4(seed=4, n=8)
pb, bounds = problems.rank_major(base, world)
opts = problems.solver_options(name, pb)
cfg = mgr.config_from_options(opts)
A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
tr = D.host_transport(rank, world, tdist)
lo, hi = int(bounds[rank]), int(bounds[rank + 1])
if name == "C3":
    # ILU(1) global smoother level: sliced from a hierarchy built whole in every process
    h_whole = mgr.mgr_setup(A, lay, cfg)
    solver = D.DeviceDistSolver(h_whole, bounds, rank, world, tr)
else:
    solver = D.DeviceDistSetupSolver(D.row_slice(A, lo, hi), lay, cfg, bounds, rank, world, tr)
assert (solver.lo, solver.n_own) == (lo, hi - lo)
v = np.random.default_rng(11).standard_normal(pb.n)
z_own = solver.apply(v[lo:hi]).cpu()
gcfg = krylov.GmresConfig(restart=opts["restart"], max_iters=opts["max_iters"], rtol=1e-6)
x_own, st = solver.gmres(pb.rhs[lo:hi], gcfg)
parts = [None] * world
tdist.all_gather_object(parts, (lo, z_own.numpy(), x_own.cpu().numpy(), st.iterations, st.converged))
if rank == 0:
    z = np.zeros(pb.n); x = np.zeros(pb.n)
    for lo_p, zp, xp, _, _ in parts:
        z[lo_p:lo_p + len(zp)] = zp
        x[lo_p:lo_p + len(xp)] = xp
    its = {p[3] for p in parts}
    conv = all(p[4] for p in parts)
    # single-GPU hierarchy of the same problem: the distributed application is bitwise equal
    h = mgr.mgr_setup(A, lay, cfg)
    z1 = h.apply(v)
    # the CPU oracle (pinned to the reference, tests/test_oracle_golden.py)
    from oracle import oracle as O
    oA = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    oh = O.mgr_setup(oA, pb.field_of, pb.entity_of, O.config_from_options(opts))
    zo = oh.apply(v)
    xo, its_o, _, conv_o = O.gmres(lambda y: O.spmv(oA, y), oh.apply, pb.rhs, restart=opts["restart"],
                                   max_iters=opts["max_iters"], rtol=1e-6)
    print("RESULT", json.dumps(dict(
        bitwise_apply=bool(np.array_equal(z, z1)),
        apply_rel_oracle=float(np.linalg.norm(z - zo) / np.linalg.norm(zo)),
        its=sorted(its), its_oracle=int(its_o), conv=bool(conv and conv_o),
        x_rel_oracle=float(np.linalg.norm(x - xo) / np.linalg.norm(xo)))), flush=True)
tdist.barrier()
tdist.destroy_process_group()
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name", ["C5", "C4", "C3"])
def test_two_processes_host_transport_vs_oracle(name):
    import json

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    port = _free_port()
    procs = []
    for r in range(2):
        # coarse levels kept distributed down to 300 rows, as in
        # test_gpu_dist.py::test_distributed_setup_is_bitwise (at the default
        # thresholds the redundantly set-up small levels agree to ~1e-13, not
        # bitwise: DESIGN.md §7)
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), PMGR_COLLAPSE_ROWS="300", PMGR_DIST_REPLICATE_ROWS="300")
        procs.append(subprocess.Popen([sys.executable, "-c", _SCRIPT, REPO, name], env=env, cwd=REPO,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        try:
            out, err = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            p.kill()
            out, err = p.communicate()
        outs.append((p.returncode, out, err))
    for r, (rc, out, err) in enumerate(outs):
        if os.environ.get("PMGR_TEST_LOGDIR"):
            with open(os.path.join(os.environ["PMGR_TEST_LOGDIR"], f"multiproc_{name}_rank{r}.log"), "w") as f:
                f.write(f"rc={rc}\n--- stdout\n{out}\n--- stderr\n{err}\n")
    for rc, out, err in outs:
        assert rc == 0, (out[-2000:], err[-4000:])
    line = [ln for ln in outs[0][1].splitlines() if ln.startswith("RESULT")]
    assert line, outs[0]
    res = json.loads(line[0][len("RESULT "):])
    print(name, res)
    assert res["bitwise_apply"]
    assert res["apply_rel_oracle"] <= 1e-10
    assert res["conv"] and len(res["its"]) == 1 and abs(res["its"][0] - res["its_oracle"]) <= 1
    assert res["x_rel_oracle"] <= (1e-10 if res["its"][0] == res["its_oracle"] else 1e-5)
