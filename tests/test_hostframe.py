"""HostFrame's host-side views of the compact downloads (CPU only): the dense
chart_of_triangle from the sparse chart ids, and the (n_visible, 6) float32
UV rows from the per-visible-vertex UVs (NaN rows where a corner is NaN)."""

import numpy as np

from paper_2502_17712_b200 import HostFrame


def _frame():
    tris = np.array([[0, 1, 2], [2, 1, 3], [3, 4, 5], [5, 6, 7], [6, 8, 9]], np.int64)
    hf = HostFrame(0, n_triangles=len(tris), triangles=tris, n_vertices=10)
    hf.visible = np.array([0, 1, 3, 4], np.int32)
    hf.visible_chart = np.array([0, 0, 3, 3], np.int32)
    hf.visible_vertices = np.array([0, 1, 2, 3, 5, 6, 7, 8, 9], np.int32)
    uv = np.arange(18, dtype=np.float32).reshape(9, 2) + 0.25
    uv[6] = np.nan  # vertex 7: at/behind the camera plane
    hf.vertex_uv = uv
    return hf, tris, uv


def test_dense_chart_ids():
    hf, _, _ = _frame()
    assert hf.chart_of_triangle.tolist() == [0, 0, -1, 3, 3]


def test_uv_rows_from_vertex_uvs():
    hf, tris, uv = _frame()
    full = np.full((10, 2), np.nan, np.float32)
    full[hf.visible_vertices] = uv
    rows = hf.uv
    assert rows.dtype == np.float32 and rows.shape == (4, 6)
    for k, t in enumerate(hf.visible):
        want = full[tris[t]].reshape(6)
        if np.isnan(want).any():
            assert np.isnan(rows[k]).all()  # the whole row, as cli.py:433-435
        else:
            assert np.array_equal(rows[k], want)
    assert np.isnan(rows[2]).all() and not np.isnan(rows[0]).any()
    assert hf.uv is rows  # built once


def test_d2h_bytes_counts_copies_only():
    hf, _, _ = _frame()
    hf.placements = np.zeros((2, 8), np.int64)
    n = hf.d2h_bytes()
    _ = hf.uv, hf.chart_of_triangle  # host-side rebuilds are not copies
    assert hf.d2h_bytes() == n == 4 * 4 + 4 * 4 + 9 * 4 + 9 * 8 + 2 * 64
