"""GPU parity of the point sensors (Table 2) through the
C ABI: dg_sensors_sample vs the oracle's locate + Lagrange evaluation (oracle/sensors.py)
on the same seeded pulse state; per-step recording inside dg_rk_step; sensors off the mesh."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1710_03887_b200 as dg  # noqa: E402
from oracle import sensors  # noqa: E402
from oracle.refelem import reference_element  # noqa: E402
from synth import configs  # noqa: E402
from oracle import geom  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _solver(cfg):
    m = cfg.mesh
    return dg.Solver(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma, q_inf=cfg.q_inf)


def _points(cfg, n, seed):
    m = cfg.mesh
    rng = np.random.default_rng(seed)
    V = m.vxyz[m.etov]
    ks = rng.choice(m.K, n, replace=False)
    lam = rng.dirichlet(np.ones(4), size=n)
    return np.einsum("nv,nvd->nd", lam, V[ks])


@pytest.mark.parametrize("name,scale", [("C2", 0.25), ("C4", 0.1), ("C5", 0.1)])
def test_sensor_sample_parity(name, scale):
    cfg = configs.make(name, scale=scale)
    m = cfg.mesh
    R = reference_element(cfg.order)
    x = geom.node_coordinates(m.vxyz, m.etov, R.r, R.s, R.t)
    Q = configs.initial_state(cfg, x)
    s = _solver(cfg)
    s.set_state(Q)
    pts = np.concatenate([_points(cfg, 12, 1), [[1e3, 1e3, 1e3]]])   # the last one is off the mesh
    el = s.set_sensors(pts)
    got = s.sample_sensors()
    assert el[-1] == -1 and np.all(np.isnan(got[-1]))
    scale_q = np.array([1.4, 1.4, 1.4, 1.4, 2.5, 1.0])
    for i, p in enumerate(pts[:-1]):
        k, r, ss, t = sensors.locate(m.vxyz, m.etov, p)
        assert el[i] == k
        want = sensors.sample(cfg.order, Q, k, r, ss, t, cfg.gamma)
        assert np.all(np.abs(got[i] - want) <= 1e-13 * scale_q), (i, got[i], want)
    s.close()


def test_sensor_recording_matches_sampling():
    cfg = configs.make("C2", scale=0.25)
    m = cfg.mesh
    s = _solver(cfg)
    s.set_state(configs.initial_state(cfg, s.nodes()))
    dt = s.stable_dt(0.5)
    s.set_sensors(_points(cfg, 5, 2))
    s.record_sensors(4)
    n0 = dg.dg_launch_count(s.ctx)
    s.step(dt, 3)
    rec = s.sensor_record()
    assert rec.shape == (3, 5, 6)
    assert dg.dg_launch_count(s.ctx) - n0 == 3 * 5 + 3   # 5 stage launches + 1 sampler per step
    assert np.array_equal(rec[-1], s.sample_sensors())
    s.step(dt, 3)                                         # capacity 4: one more sample, then full
    assert dg.dg_sensors_recorded(s.ctx) == 4
    s.close()


def test_recorded_pressure_spectrum_on_device():
    """N4 pipeline on a device record: torch.fft on the GPU vs the oracle's DFT sums."""
    from oracle import analysis as oan
    from paper_1710_03887_b200 import analysis as pan
    cfg = configs.make("C2", scale=0.25)
    s = _solver(cfg)
    s.set_state(configs.initial_state(cfg, s.nodes()))
    dt = s.stable_dt(0.5)
    s.set_sensors(_points(cfg, 3, 4))
    s.record_sensors(16)
    s.step(dt, 16)
    torch.cuda.synchronize()
    p = s._rec[:, :, 5]                          # (16, 3) pressure, on the device
    f, db, a = pan.spectrum(p, dt)
    assert a.is_cuda
    for i in range(3):
        f0, db0, a0 = oan.dft_amplitude(p[:, i].cpu().numpy(), dt)
        assert np.abs(a[:, i].cpu().numpy() - a0).max() < 1e-15 + 1e-12 * a0.max()
    s.close()
