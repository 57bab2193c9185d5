"""Hash of the fields after a few steps with one libpf build (PF_LIB), for bitwise A/B checks of kernel variants.
usage: PF_LIB=build/libpf_X.so python tools/ab_hash.py [aniso] — prints one hash per grid (ragged and 256^3)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01684_b200.pf as pfm
from inputs import gen
aniso = "aniso" in sys.argv[1:]
cfg = gen.load_config("c5" if aniso else "c4"); pd = gen.load_params("v1")
out = []
for (nx, ny, nz) in [(37, 29, 23), (256, 256, 256)]:
    prm = pfm.make_params(pd, cfg, nx=nx, ny=ny, window=False)
    with pfm.Context(nx, ny, nz, prm) as ctx:
        ctx.init(cfg["seed"]); ctx.step(5)
        phi, mu = ctx.read()
        out.append(hashlib.sha1(phi.tobytes() + mu.tobytes()).hexdigest()[:16])
print(os.environ.get("PF_LIB", "default"), " ".join(out))
