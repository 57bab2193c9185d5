"""Time pf_mesh (marching cubes, NEXT-4) on the C4 state (512^3, one B200):
per phase, the count-only pass and the full count+emit into device buffers."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import gen
from paper_1506_01684_b200 import pf

n = int(os.environ.get("N", 512))
cfg = gen.load_config("c4")
prm = pf.make_params(gen.load_params("v1"), cfg, nx=n, ny=n)
L = pf.lib()
with pf.Context(n, n, n, prm) as ctx:
    ctx.init(cfg["seed"])
    ctx.step(10)
    torch.cuda.synchronize()
    for a in range(4):
        cnt = ctypes.c_int64(0)
        L.pf_mesh(ctx._c, a, 0.5, 0, None, None, ctypes.byref(cnt))
        T = cnt.value
        ids = torch.empty((max(T, 1), 3), dtype=torch.int64, device="cuda")
        pos = torch.empty((max(T, 1), 3, 3), dtype=torch.float64, device="cuda")
        for cap, what in ((0, "count"), (T, "count+emit")):
            L.pf_mesh(ctx._c, a, 0.5, cap, ids.data_ptr(), pos.data_ptr(), ctypes.byref(cnt))
            t0 = time.perf_counter()
            reps = 5
            for _ in range(reps):
                L.pf_mesh(ctx._c, a, 0.5, cap, ids.data_ptr(), pos.data_ptr(), ctypes.byref(cnt))
            dt = (time.perf_counter() - t0) / reps
            cubes = n * n * (n - 1)
            print(f"phase {a}: {T} triangles, {what}: {dt * 1e3:.3f} ms/call, {cubes / dt / 1e9:.2f} G cubes/s")
