"""CUDA-graph replay of the time step (pf_params.graph = 1, single-rank runs
without per-sweep timing) against launching the kernels one by one: bitwise identical states, the same launch counts, the time level
carried on the device across graph replays, graphs re-captured after window
shifts, origin changes and new states."""
import numpy as np
import pytest

from inputs import gen

pytestmark = pytest.mark.gpu


def _pf():
    from paper_1506_01684_b200 import pf
    return pf


def _state(cfg_name, n, lh):
    cfg = gen.load_config(cfg_name)
    spec = gen.spec_from_config(cfg, n, n)
    spec.layer_height = lh
    spec.n_seeds = 9
    return cfg, gen.generate(spec, n, n, n)


def _run(cfg, phi, mu, steps, graph, blocks=(1, 1, 1), chunks=None, **kw):
    pf = _pf()
    n = phi.shape[-1]
    prm = pf.make_params(gen.load_params("v1"), cfg, graph=graph, **kw)
    with pf.Context(n, n, n, prm, *blocks) as ctx:
        ctx.write(phi, mu)
        for c in (chunks or [steps]):
            ctx.step(c)
        out = ctx.read()
        inf = ctx.info()
        return out[0], out[1], int(inf.launches), int(inf.shifts), int(inf.step)


@pytest.mark.parametrize("overlap", [0, 3])
@pytest.mark.parametrize("blocks", [(1, 1, 1), (2, 2, 2)])
def test_graph_bitwise_equal_eager(overlap, blocks):
    cfg, (phi, mu) = _state("c2", 24, 10.5)
    a = _run(cfg, phi, mu, 25, False, blocks, overlap=overlap, layer_height=10.5, window=False)
    b = _run(cfg, phi, mu, 25, True, blocks, chunks=[1, 7, 1, 16], overlap=overlap, layer_height=10.5,
             window=False)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert b[2] == a[2] + 25 and a[4] == b[4] == 25   # the graph adds the device step-counter kernel


def test_graph_window_shifts_and_nan_watchdog():
    # anisotropic C5 model, forced window shifts (graphs re-captured after each)
    cfg, (phi, mu) = _state("c5", 24, 17.5)
    kw = dict(layer_height=17.5, window=True, nan_check_every=4)
    a = _run(cfg, phi, mu, 30, False, **kw)
    b = _run(cfg, phi, mu, 30, True, chunks=[3, 27], **kw)
    assert a[3] > 0 and a[3] == b[3]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_graph_time_level_and_origin():
    # pf_set_time between steps: the table of the replayed graph must follow
    pf = _pf()
    cfg, (phi, mu) = _state("c2", 16, 6.5)
    outs = []
    for graph in (False, True):
        prm = pf.make_params(gen.load_params("v1"), cfg, graph=graph, layer_height=6.5, window=False)
        with pf.Context(16, 16, 16, prm) as ctx:
            ctx.write(phi, mu)
            ctx.step(3)
            ctx.set_time(500, 7)
            ctx.step(4)
            outs.append(ctx.read())
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_timing_runs_eagerly_and_matches():
    pf = _pf()
    cfg, (phi, mu) = _state("c2", 16, 6.5)
    res = []
    for timing in (False, True):
        prm = pf.make_params(gen.load_params("v1"), cfg, layer_height=6.5, window=False, graph=True)
        with pf.Context(16, 16, 16, prm) as ctx:
            ctx.write(phi, mu)
            ctx.set_timing(timing)
            ctx.step(5)
            inf = ctx.info()
            res.append((ctx.read(), inf.phi_launches))
    assert res[0][1] == 0 and res[1][1] == 5
    assert np.array_equal(res[0][0][0], res[1][0][0]) and np.array_equal(res[0][0][1], res[1][0][1])
