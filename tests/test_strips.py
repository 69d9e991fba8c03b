"""Strip decomposition: host logic on CPU with gloo.

The decomposition driver (paper_2204_07921_b200.strips) is backend-agnostic;
here it drives a CPU backend built on the pinned oracle (test infrastructure)
over torch.distributed/gloo with world sizes 2 and 3, and the union of the
owned rows must equal the single-image oracle solve BIT FOR BIT.
"""

import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_07921_b200 import strips as S
from paper_2204_07921_b200.driver import SolverConfig


class OracleStrip:
    """CPU strip backend: the reference algorithm (oracle) run on the window."""

    is_cuda = False

    def __init__(self, geom, cfg, f_full, ref_full=None):
        self.geom, self.cfg = geom, cfg
        w = slice(geom.w0, geom.w1)
        self.buf = {i: np.array(f_full[w], dtype=np.float64) for i in range(3)}
        self.buf[3] = np.array(f_full[w], dtype=np.float64)
        self.buf[4] = None if ref_full is None else np.array(ref_full[w], dtype=np.float64)

    def level_step(self, layer, cur, out):
        self.buf[out][...] = O.sweep_layer(self.buf[cur], self.buf[3], layer, self.cfg.mode,
                                           self.cfg.inner_iters, self.cfg.alpha)

    def energy_partials(self, cur, prev, use_ref):
        g = self.geom
        lo, hi = g.local(g.g0), g.local(g.g1)
        u, up, f = self.buf[cur], self.buf[prev], self.buf[3]
        curv = O.curvature_field(u, self.cfg.mode)[lo:hi]
        out = np.array([curv.sum(), ((u[lo:hi] - f[lo:hi]) ** 2).sum(), np.abs(u[lo:hi] - up[lo:hi]).sum(),
                        np.abs(u[lo:hi]).sum(), 0.0])
        if use_ref:
            out[4] = ((u[lo:hi] - self.buf[4][lo:hi]) ** 2).sum()
        return out

    # asynchronous protocol (strips.solve_strips): begin / partials tensor with the
    # non-finite flag appended
    def begin(self):
        pass

    def energy_partials_async(self, cur, prev, use_ref):
        import torch

        return torch.from_numpy(np.append(self.energy_partials(cur, prev, use_ref), 0.0))

    def rows(self, index, g_lo, g_hi):
        import torch

        return torch.from_numpy(self.buf[index][self.geom.local(g_lo):self.geom.local(g_hi)])

    def download(self, index):
        return self.buf[index]


def _image(m, n, seed=3):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:m, 0:n]
    clean = np.clip(0.4 + 0.3 * np.sin(y / 9.0) * np.cos(x / 7.0) + 0.2 * ((y - m / 2) ** 2 + (x - n / 3) ** 2 < 300),
                    0, 1)
    return clean + 0.06 * rng.standard_normal((m, n)), clean


def test_geometry():
    assert S.row_align(3) == 42 and S.ghost_rows(3) == 42
    assert S.row_align(1) == 2 and S.ghost_rows(1) == 6
    assert S.ghost_rows(2) == 18
    parts = S.partition_rows(16384, 8, 3)
    assert parts[0] == (0, 2058) and parts[-1][1] == 16384
    assert all(g0 % 42 == 0 for g0, _ in parts)
    assert all(b[0] == a[1] for a, b in zip(parts, parts[1:]))
    with pytest.raises(ValueError):
        S.check_strippable(100, 100, 4, 3)
    with pytest.raises(ValueError):
        S.check_strippable(4000, 100, 2, 4)


@pytest.mark.parametrize("parts,mode,layers", [(2, "mean", 3), (3, "gaussian", 3), (4, "mean", 2), (2, "mean", 1)])
def test_local_strips_equal_single_image(parts, mode, layers):
    m, n = 42 * 3 * parts + 17, 71
    f, clean = _image(m, n)
    cfg = SolverConfig(mode=mode, layers=layers, max_outer=5, epsilon=1e-300, inner_iters=1)
    G = S.ghost_rows(layers)
    geoms = [S.StripGeometry(m, n, g0, g1, G) for g0, g1 in S.partition_rows(m, parts, layers)]
    strips = [OracleStrip(g, cfg, f, clean) for g in geoms]
    ex = S.LocalExchange(strips)
    cur, tr = S.solve_strips(strips, ex, cfg, m * n, True, 1.0)
    u = np.concatenate(ex.gather_owned(cur))
    ref = O.denoise(f, mode=mode, layers=layers, max_outer=5, epsilon=1e-300, reference=clean, peak=1.0)
    assert np.array_equal(u, ref["u"])
    assert tr.iterations == ref["iterations"]
    assert np.allclose(tr.energies(), ref["energies"], rtol=1e-13, atol=0)
    assert np.allclose([r.psnr for r in tr.records], ref["psnr"], rtol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, m, n, mode, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        f, clean = _image(m, n)
        cfg = SolverConfig(mode=mode, layers=3, max_outer=30, epsilon=1e-5)
        G = S.ghost_rows(3)
        geoms = [S.StripGeometry(m, n, g0, g1, G) for g0, g1 in S.partition_rows(m, ws, 3)]
        st = OracleStrip(geoms[rank], cfg, f, clean)
        ex = S.DistExchange(st, geoms, rank)
        cur, tr = S.solve_strips([st], ex, cfg, m * n, True, 1.0)
        parts = ex.gather_owned(cur)  # tensor all-gather of every rank's owned rows
        if rank == 0:
            q.put((np.concatenate(parts), tr.energies(), tr.iterations, tr.converged))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws,mode", [(2, "mean"), (3, "gaussian")])
def test_gloo_strips_equal_single_image(ws, mode):
    import torch.multiprocessing as mp

    m, n = 42 * 2 * ws + 29, 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, m, n, mode, q)) for r in range(ws)]
    for p in procs:
        p.start()
    u, energies, iters, conv = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    f, clean = _image(m, n)
    ref = O.denoise(f, mode=mode, layers=3, max_outer=30, epsilon=1e-5)
    assert iters == ref["iterations"] and conv == ref["converged"]
    assert np.array_equal(u, ref["u"])
    assert np.allclose(energies, ref["energies"], rtol=1e-13, atol=0)
