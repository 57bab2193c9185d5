"""Small run that launches every kernel of libpf once or more, for
compute-sanitizer (one tool per run: memcheck / racecheck / synccheck / initcheck).
C1-sized states, several decompositions, all overlap modes, the moving window
(forced shift), the NaN watchdog, checkpoints, marching cubes, read/write."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import gen  # noqa: E402
from paper_1506_01684_b200 import pf  # noqa: E402

pd = gen.load_params("v1")
for cfg_name, n, blocks, ov, window, lh in (("c1", 32, (1, 1, 1), 0, False, 8),
                                            ("c2", 24, (2, 2, 2), 3, True, 15.5),
                                            ("c5", 20, (2, 1, 2), 2, True, 13.5)):
    cfg = gen.load_config(cfg_name)
    spec = gen.spec_from_config(cfg, n, n)
    spec.layer_height = lh
    phi, mu = gen.generate(spec, n, n, n)
    prm = pf.make_params(pd, cfg, layer_height=lh, overlap=ov, window=window, nan_check_every=2)
    with pf.Context(n, n, n, prm, *blocks) as ctx:
        ctx.write(phi, mu)
        ctx.step(4)
        ctx.init(3)
        ctx.step(2)
        gp, gm = ctx.read()
        for a in range(4):
            ctx.mesh(a)
        with tempfile.TemporaryDirectory() as d:
            ctx.save(os.path.join(d, "c.bin"))
            ctx.load(os.path.join(d, "c.bin"))
        ctx.step(1)
        print(cfg_name, blocks, "ok", ctx.info().shifts)
print("sanitize run done")
