"""Microscopy particle registration (GMM / Bhattacharyya) kernel vs the float64 oracle (1e-4 rel)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import gmm as ogmm  # noqa: E402


def test_gmm_engine_matches_oracle():
    from paper_2009_04755_b200.apps import ParticleFusionApp
    from paper_2009_04755_b200.engine import AllPairsEngine
    n = 20
    app = ParticleFusionApp(n, seed=3, angles=24)
    res = AllPairsEngine(app, leaf_block=4, device_slots=9).run()
    parts = [app.points(k) for k in range(n)]
    want = [ogmm.compare(parts[i], parts[j], angles=24) for i in range(n) for j in range(i + 1, n)]
    np.testing.assert_allclose(res.values, want, rtol=1e-4)
    assert res.stats["pairs_done"] == n * (n - 1) // 2


def test_gmm_rotated_copy_known_answer():
    from paper_2009_04755_b200.apps import ParticleFusionApp, ItemData, Stage
    base = ogmm.particle(5, 1)
    t = 2 * np.pi * 7 / 36                       # on the rotation grid
    c, s = np.cos(t), np.sin(t)
    rot = base.copy()
    rot[:, 0] = c * base[:, 0] - s * base[:, 1] + 40.0
    rot[:, 1] = s * base[:, 0] + c * base[:, 1] - 25.0
    other = ogmm.particle(9, 1)
    app = ParticleFusionApp(3, particles=[rot, base, other], angles=36)
    pre = {}
    for k in range(3):
        raw = ItemData(Stage.RAW_FILE, app.fetch_raw(app.path_for_key(k)))
        pre[k] = app.preprocess(k, app.parse(k, raw))
    import struct
    v01 = struct.unpack("<d", app.compare((0, pre[0]), (1, pre[1])))[0]
    self_overlap = ogmm.compare(base, base, angles=36)
    assert v01 == pytest.approx(self_overlap, rel=1e-4)       # perfect registration found
    v12 = struct.unpack("<d", app.compare((1, pre[1]), (2, pre[2])))[0]
    assert v12 == pytest.approx(ogmm.compare(base, other, angles=36), rel=1e-4)
