"""TEST INFRASTRUCTURE: run N ranks of libpf as threads of one process on one
GPU over the in-process NCCL stand-in (nccl_fake.cu), and the same global
problem as one context holding all blocks (nranks = 1, halos as device
copies).  Prints one JSON line: per-rank bitwise agreement of the state, the
window shifts, and (optionally) checkpoint / mesh agreement.

usage: PF_LIB=build/libpf_fakenccl.so python run_ranks.py '<json spec>'"""
import json
import os
import sys
import tempfile
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from inputs import gen  # noqa: E402
from paper_1506_01684_b200 import pf  # noqa: E402

spec = json.loads(sys.argv[1])
NX, NY, NZ = spec["grid"]
px, py, pz = spec["blocks"]
N = px * py * pz
cfg = gen.load_config(spec.get("config", "c2"))
pd = gen.load_params("v1")
lh = spec.get("layer_height", NZ / 2)
prm = pf.make_params(pd, cfg, layer_height=lh, window=spec.get("window", False), overlap=spec.get("overlap", 0),
                     aniso=spec.get("aniso"))
steps = spec.get("steps", 10)
gs = gen.spec_from_config(cfg, NX, NY)
gs.layer_height = lh
gs.n_seeds = spec.get("n_seeds", 7)
phi, mu = gen.generate(gs, NX, NY, NZ)

# reference: one context, all blocks on the GPU
with pf.Context(NX, NY, NZ, prm, px, py, pz) as ref:
    ref.write(phi, mu)
    ref.step(steps)
    rphi, rmu = ref.read()
    rshifts = ref.info().shifts
    rmesh = [ref.mesh(a) for a in range(4)] if spec.get("mesh") else None

nid = pf.nccl_unique_id()
ctxs = [None] * N
errs = []
results = [None] * N
ckdir = tempfile.mkdtemp()


def rank_main(r):
    try:
        c = pf.Context(NX, NY, NZ, prm, px, py, pz, rank=r, nranks=N, device=0, nccl_id=nid)
        ctxs[r] = c
        if spec.get("fusion"):   # fused mu(n) + phi(n+1) kernels; the reference runs the separate sweeps
            c.set_fusion(True)
        inf = c.info()
        x0, y0, z0 = int(inf.x0), int(inf.y0), int(inf.z0)
        nz, ny, nx = c.shape
        c.write(np.ascontiguousarray(phi[:, z0:z0 + nz, y0:y0 + ny, x0:x0 + nx]),
                np.ascontiguousarray(mu[:, z0:z0 + nz, y0:y0 + ny, x0:x0 + nx]))
        if spec.get("checkpoint"):
            half = steps // 2
            c.step(half)
            c.save(os.path.join(ckdir, "ck.bin"))
            c.step(steps - half)
            gphi, gmu = c.read()
            mesh = [c.mesh(a) for a in range(4)] if spec.get("mesh") else None
            c.load(os.path.join(ckdir, "ck.bin"))       # collective
            c.step(steps - half)
            lphi, lmu = c.read()
            res = {"resumed_equal_cast": True, "lphi": lphi, "lmu": lmu}
        else:
            if spec.get("step_io"):    # the last step through pf_step_io (collective; multi-rank: the plain calls)
                c.step(steps - 1)
                gphi, gmu = c.step_io(*c.read())
            else:
                c.step(steps)
                gphi, gmu = c.read()
            mesh = [c.mesh(a) for a in range(4)] if spec.get("mesh") else None
            res = {}
        res.update(box=(x0, y0, z0, nx, ny, nz), phi=gphi, mu=gmu, shifts=int(c.info().shifts))
        res["mesh"] = mesh       # of the state compared with the reference
        results[r] = res
    except Exception as e:  # noqa: BLE001
        errs.append(f"rank {r}: {e!r}")


threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(N)]
for t in threads:
    t.start()
for t in threads:
    t.join(timeout=600)
out = {"ranks": N, "errors": errs, "alive": [t.is_alive() for t in threads]}
if not errs and all(r is not None for r in results):
    eq_phi = eq_mu = True
    for res in results:
        x0, y0, z0, nx, ny, nz = res["box"]
        eq_phi &= bool(np.array_equal(res["phi"], rphi[:, z0:z0 + nz, y0:y0 + ny, x0:x0 + nx]))
        eq_mu &= bool(np.array_equal(res["mu"], rmu[:, z0:z0 + nz, y0:y0 + ny, x0:x0 + nx]))
    out.update(equal_phi=eq_phi, equal_mu=eq_mu, shifts=[res["shifts"] for res in results], ref_shifts=int(rshifts),
               moved=float(np.abs(rphi - phi).max()))
    if spec.get("checkpoint"):
        # the resumed run continues from the binary32 cast of the step-half state:
        # all ranks' resumed states must assemble into what one context resumed
        # from the same file produces
        with pf.Context(NX, NY, NZ, prm, px, py, pz) as one:
            one.load(os.path.join(ckdir, "ck.bin"))
            one.step(steps - steps // 2)
            ophi, omu = one.read()
        ok = True
        for res in results:
            x0, y0, z0, nx, ny, nz = res["box"]
            ok &= bool(np.array_equal(res["lphi"], ophi[:, z0:z0 + nz, y0:y0 + ny, x0:x0 + nx]))
            ok &= bool(np.array_equal(res["lmu"], omu[:, z0:z0 + nz, y0:y0 + ny, x0:x0 + nx]))
        out["checkpoint_equal"] = ok
    if spec.get("mesh"):
        from oracle import mesh as MC
        ok = True
        for a in range(4):
            ids = np.concatenate([res["mesh"][a][0] for res in results])
            ok &= bool(np.array_equal(MC.canonical(ids), MC.canonical(rmesh[a][0])))
        out["mesh_equal"] = ok
for c in ctxs:
    if c is not None:
        c.close()
print(json.dumps(out))
