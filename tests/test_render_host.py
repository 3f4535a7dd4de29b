"""Host logic without a GPU: estimate -> renderer parameter mapping, strong
ray sharding, and the NCCL entry points of the C ABI (argument checks, the
lazily resolved libnccl)."""
import ctypes

import numpy as np
import pytest

from paper_1803_00430_b200 import _lib, distributed, render, workloads
from paper_1803_00430_b200.analysis import ReverbParams


def _estimate(nb, rt, gain, direct, predelay, silent=None):
    nk = 16
    L = np.stack([np.eye(nk) * (1.0 + b) for b in range(nb)])
    return ReverbParams(rt60=np.asarray(rt, float), reverb_gain=np.asarray(gain, float),
                        drr_db=np.zeros(nb), total_intensity=np.ones(nb),
                        direct_intensity=np.asarray(direct, float),
                        silent_bands=np.zeros(nb, bool) if silent is None else np.asarray(silent),
                        predelay=predelay, mean_free_path=5.0, avg_directivity=np.zeros((nb, nk)),
                        loudness=L, silent=False)


def test_params_from_estimates_folds_bands_and_geometry():
    e = [_estimate(8, [0.4, 0.6, 1.0, 1.2, 0.8, 0.8, 2.0, 4.0], [1, 1, 2, 2, 3, 5, 0, 0],
                   [4, 4, 0, 0, 1, 9, 0, 0], 0.02, silent=[0, 0, 0, 0, 0, 0, 1, 1]),
         _estimate(8, [1.0] * 8, [1.0] * 8, [1.0] * 8, -1.0)]
    src = np.array([[3.0, 4.0, 0.0], [0.0, 0.0, 6.86]])
    p0 = workloads.c4_params(n_sources=2)
    p = render.params_from_estimates(e, src, [0.0, 0.0, 0.0], p0["fdn_delay"], p0["hrtf"])
    assert p["rt60"].shape == (2, 4)
    np.testing.assert_allclose(p["rt60"][0], [0.5, 1.1, 0.8, 1.0])          # silent pair -> fallback 1.0
    np.testing.assert_allclose(p["g_reverb"][0], [1.0, 2.0, np.sqrt(17.0), 0.0])
    np.testing.assert_allclose(p["gain_direct"][0], [2.0, 0.0, np.sqrt(5.0), 0.0])
    np.testing.assert_allclose(p["dir_direct"], [[0.6, 0.8, 0.0], [0.0, 0.0, 1.0]])
    np.testing.assert_allclose(p["delay_direct"], [5.0 / 343.0 * 48000.0, 6.86 / 343.0 * 48000.0])
    assert p["predelay"][0] == pytest.approx(0.02 * 48000.0)
    assert p["predelay"][1] == pytest.approx(p["delay_direct"][1])          # silent -> direct delay
    np.testing.assert_allclose(p["D"][0, 1], np.eye(16) * 3.5)              # mean of bands 2, 3
    with pytest.raises(ValueError):
        render.params_from_estimates(e, np.zeros((2, 3)), [0.0, 0.0, 0.0], p0["fdn_delay"], p0["hrtf"])
    with pytest.raises(ValueError):
        render.params_from_estimates([_estimate(6, [1] * 6, [1] * 6, [1] * 6, 0.0)], src[:1], [0, 0, 0],
                                     p0["fdn_delay"][:1], p0["hrtf"])


def test_shard_rays_strong():
    assert [distributed.shard_rays(1 << 20, g, 8) for g in (0, 3, 7)] == [
        (0, 1 << 17), (3 << 17, 1 << 17), (7 << 17, 1 << 17)]
    with pytest.raises(ValueError):
        distributed.shard_rays(10, 0, 3)
    with pytest.raises(ValueError):
        distributed.shard_rays(8, 2, 2)


def test_nccl_entry_points_validate():
    L = _lib.lib()
    assert L.ef_nccl_reduce_hist(None, None, None, 0, 0, None) == _lib.EF_EINVAL
    assert "null communicator" in _lib.last_error()
    assert L.ef_nccl_reduce_hist(ctypes.c_void_p(8), ctypes.c_void_p(8), ctypes.c_void_p(8), 1, 7,
                                 None) == _lib.EF_EINVAL
    assert "mode" in _lib.last_error()
    comm = ctypes.c_void_p()
    uid = (ctypes.c_uint8 * 128)()
    assert L.ef_nccl_comm_create(2, 5, uid, -1, ctypes.byref(comm)) == _lib.EF_EINVAL
    assert L.ef_nccl_comm_destroy(None) == _lib.EF_OK
    rc = L.ef_nccl_unique_id(uid)          # libnccl resolved lazily; no GPU needed for an id
    assert rc in (_lib.EF_OK, _lib.EF_ENCCL)
    if rc == _lib.EF_OK:
        assert any(bytes(uid))
