"""The library's multi-GPU code path with SEVERAL RANKS on the one test GPU: each rank is a
thread with its own dc_ctx, joined through dc_comm_attach, but the NCCL transport is the
in-process stand-in tests/fake_nccl (real NCCL refuses two ranks on one device). Everything
the library does at N > 1 runs: the partition check, the (c_i, zeta_i) exchange with
per-rank counts at the IEWPF barrier, the analysis split around it (pulls on the second
stream), the drifter gather to rank 0 for the forecast statistics. The result must equal
one context holding every member, bit for bit."""
import json
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import json, sys, threading
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1910_01031_b200 as pkg
parts = json.loads(sys.argv[2])           # members per rank
total = sum(parts)
cfg = pkg.Config(nx=100, ny=60)
_, S = pkg.precompute_S(cfg)
_, usig = pkg.precompute_local_svd(cfg, S)
rng = np.random.default_rng(3)
lx, ly = 100 * 2220.0, 60 * 2220.0
pos0 = rng.uniform(0, 1, (5, 2)) * [lx, ly]
obs = [np.hstack([rng.uniform(0, 1, (6, 2)) * [lx, ly], rng.normal(0, 20, (6, 2))]) for _ in range(3)]
truth = [pos0 + 100.0 * (c + 1) for c in range(3)]

def run(M, base, rank, world, nid, out):
    ens = pkg.Ensemble(cfg, M, member_base=base)
    if nid is not None:
        ens.comm_attach(nid, rank, world, total)
    ens.init_double_jet()
    ens.drifters_set(pos0[None].repeat(M, 0))
    res = []
    for c in range(3):
        ens.da_cycle(5, obs[c], S, usig, c)
        ens.readback_enqueue(c % 2, truth_xy=truth[c])
        if c:
            r = ens.readback_wait((c - 1) % 2)
            res.append((float(r["E"]), float(r["RMSE"])))
    r = ens.readback_wait(0)
    res.append((float(r["E"]), float(r["RMSE"])))
    e, u, v, t = ens.download()
    d, wb = ens.iewpf_diagnostics()
    E, R, _, _ = ens.forecast_error(truth[2])   # the synchronous gathered form
    out[rank] = {"stats": res, "sync": [float(E), float(R)], "diag": d.tolist(), "wb": wb.tolist(),
                 "e": e.tobytes().hex(), "u": u.tobytes().hex(), "v": v.tobytes().hex(),
                 "t": t.tolist()}
    ens.close()

world = len(parts)
nid = pkg.comm_unique_id()
out = [None] * world
ths, base = [], 0
for r, M in enumerate(parts):
    ths.append(threading.Thread(target=run, args=(M, base, r, world, nid, out)))
    base += M
for t in ths: t.start()
for t in ths: t.join()
one = [None]
run(total, 0, 0, 1, None, one)
print(json.dumps({"ranks": out, "one": one[0]}))
'''


# [3, 3], [2, 2, 3]: even / uneven slices; the eight-rank partition of configs[3]
# (1000 members over 8 GPUs), scaled down, with uneven slices
@pytest.mark.parametrize("parts", [[3, 3], [2, 2, 3], [2, 1, 2, 2, 1, 2, 2, 2]])
def test_comm_ranks_on_one_gpu_equal_one_context(tmp_path, parts):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    lib = str(tmp_path / "libfake_nccl.so")
    subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", f"-I{cuda}/include",
                    os.path.join(ROOT, "tests", "fake_nccl", "fake_nccl.cpp"), f"-L{cuda}/lib64",
                    "-lcudart", f"-Wl,-rpath,{cuda}/lib64", "-o", lib], check=True)
    env = dict(os.environ, DC_NCCL_LIB=lib)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, json.dumps(parts)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    one, ranks = res["one"], res["ranks"]
    # rank 0 holds the forecast statistics of the whole ensemble (gathered drifters)
    assert ranks[0]["stats"] == one["stats"] and ranks[0]["sync"] == one["sync"]
    nx, ny = 100, 60
    cell = nx * ny * 4 * 2  # hex chars per member field
    base = 0
    for k, M in enumerate(parts):
        rk = ranks[k]
        assert rk["wb"] == one["wb"]
        assert rk["diag"] == one["diag"][base:base + M]
        for f in ("e", "u", "v"):
            assert rk[f] == one[f][base * cell:(base + M) * cell], (k, f)
        assert rk["t"] == one["t"][base:base + M]
        base += M
