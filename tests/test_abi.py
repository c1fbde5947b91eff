"""C ABI surface (CPU): the library loads and exports every symbol gnb.h declares;
argument validation that happens before any CUDA call."""

import ctypes

import numpy as np
import pytest

from paper_1905_13746_b200 import _native as N


def test_every_declared_symbol_is_exported():
    names = N.declared_symbols()
    assert len(names) >= 12
    for name in names:
        assert hasattr(N.lib, name), name


def test_version_and_strerror():
    assert N.lib.gnb_abi_version() == 3
    assert N.lib.gnb_strerror(0) == b"ok"


@pytest.mark.parametrize("F,ldx,width,limit,S,C", [
    (0, 4, 10, 10, 1, 2), (4, 3, 10, 10, 1, 2), (4, 4, 0, 10, 1, 2), (4, 4, 3, 10, 1, 2),
    (4, 4, 10, 10, 0, 2), (4, 4, 10, 10, 1, 1), (4, 4, 10, 10, 1, 17)])
def test_predict_rejects_bad_geometry(F, ldx, width, limit, S, C):
    rc = N.lib.gnb_predict(None, 0, F, ldx, None, width, limit, 1, S, C, 1, None, None, 0)
    assert rc == N.GNB_EINVAL
    assert N.lib.gnb_last_error()


def test_packed_table_bytes():
    # prior [S][CP] + log-lik [S][NB][32][CP], NB = ceil(F/32) padded to a multiple of 4
    assert N.lib.gnb_packed_table_bytes(1, 2, 32) == 1 * 2 * 8 + 1 * 4 * 32 * 2 * 8
    assert N.lib.gnb_packed_table_bytes(3, 5, 200) == 3 * 8 * 8 + 3 * 8 * 32 * 8 * 8
    assert N.lib.gnb_packed_table_bytes(0, 2, 32) == 0
    assert N.lib.gnb_packed_table_bytes(1, 17, 32) == 0


def test_fit_rejects_bad_arguments():
    assert N.lib.gnb_fit_stats(None, 0, 0, 0, None, None, 10, 10, 2, None, None, None, None, 0,
                               0) == N.GNB_EINVAL
    assert N.lib.gnb_fit_stats(None, 0, 4, 4, None, None, 10, 10, 1, 1, None, 1, None, 0,
                               0) == N.GNB_EINVAL


def test_check_maps_errors():
    from paper_1905_13746_b200.errors import InvalidConfigError
    N.lib.gnb_predict(None, 0, 0, 0, None, 1, 1, 1, 1, 2, 1, None, None, 0)
    with pytest.raises(InvalidConfigError):
        N.check(N.GNB_EINVAL, "x")
    with pytest.raises(N.NativeError):
        N.check(N.GNB_ECUDA, "x")


def test_comms_argument_validation():
    """gnb_comms_* reject bad arguments before touching NCCL or CUDA."""
    h = ctypes.c_void_p()
    assert N.lib.gnb_comms_init(ctypes.byref(h), 0, None) == N.GNB_EINVAL
    assert N.lib.gnb_comms_init_rank(ctypes.byref(h), 2, 2, None, 0) == N.GNB_EINVAL
    assert N.lib.gnb_fit_allreduce(None, None, 0, None) == N.GNB_EINVAL
    assert N.lib.gnb_comms_size(None) == 0
    N.lib.gnb_comms_destroy(None)


def test_pack_u4_layout_and_odd_ldx():
    """pack_u4: feature 2j in the low nibble of byte j, rows padded to 8 bytes;
    out-of-range counts refused; GNB_X_U4 with an odd ldx rejected before CUDA."""
    import numpy as np
    import torch
    from paper_1905_13746_b200 import dense
    x = np.random.default_rng(0).integers(0, 16, size=(5, 19))
    p = dense.pack_u4(torch.from_numpy(x)).numpy()
    assert p.shape == (5, 16)
    un = np.stack([p & 15, p >> 4], axis=2).reshape(5, 32)
    assert (un[:, :19] == x).all() and (un[:, 19:] == 0).all()
    with pytest.raises(ValueError):
        dense.pack_u4(torch.tensor([[16]]))
    with pytest.raises(ValueError):
        dense.pack_u4(torch.tensor([[-1]]))
    assert N.lib.gnb_predict_host_typed(None, N.X_U4, 1, 3, 3, None, 1, 1, None, 1, 2, None,
                                        None, None, None, 0, None) == N.GNB_EINVAL
    assert N.lib.gnb_predict_host_typed(None, 9, 1, 3, 3, None, 1, 1, None, 1, 2, None,
                                        None, None, None, 0, None) == N.GNB_EINVAL


def test_mixed_rows_kernel_choice():
    """gnb_predict_mixed_rows (host-only shape logic): the mixed-slot kernel takes
    C = 2 batches of >= 2 slots whose tables fit next to >= 3 ring stages, and
    never short rows (row-box kernel) or bad arguments."""
    f = N.lib.gnb_predict_mixed_rows
    assert f(200, N.X_I32, 2, 29) == 256          # cfg3: 29 x 200 features = 93 KB of tables
    assert f(300, N.X_U8, 2, 20) == 256          # uint8 rows of 300 features (not row-box)
    assert f(200, N.X_U8, 2, 29) == 0             # uint8 F=200 is 13 quads: row-box kernel
    assert f(200, N.X_I32, 2, 1) == 0             # one slot: uniform tiles
    assert f(200, N.X_I32, 4, 29) == 0            # class pad 4
    assert f(50, N.X_I32, 2, 8) == 0              # short rows: row-box kernel
    assert f(2000, N.X_I32, 2, 64) == 0           # 2 MB of tables
    assert f(200, N.X_I32, 2, 40) == 256          # 129 KB of tables + 3 stages fit
    assert f(200, N.X_I32, 2, 45) == 0            # 145 KB: fewer than 3 stages fit
    assert f(0, N.X_I32, 2, 4) == 0 and f(200, 7, 2, 4) == 0 and f(200, N.X_I32, 17, 4) == 0
