"""Host-arithmetic probe.

The reference's only non-IEEE-sequential float64 arithmetic runs inside
OpenBLAS through numpy: the projection `homo @ cam.view_proj.T`
(charts.py:273-274) and the shoelace `np.dot` of `_signed_area2`
(charts.py:251-253).  OpenBLAS picks its kernels by CPU at run time, so the
reference's bits are host dependent.  The oracle (and the CUDA kernels)
restate the FMA chains of the kernels found in the build container; this
probe checks, on whatever host it runs on, that numpy still produces exactly
those bits.  The un-marked test runs in the build container (where the
goldens were made); the `gpu`-marked twin runs on the GPU box's host, where
the reference itself cannot run (tests/golden stores the camera matrices, so
the GPU tests never depend on the box's BLAS).
"""

import json
import os

import numpy as np
import pytest

import oracle


def blas_config() -> dict:
    info = {"numpy": np.__version__}
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "architecture", "num_threads")}
                        for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception as e:  # pragma: no cover - informational only
        info["blas"] = repr(e)
    return info


def probe(n_tris: int = 20000, n_polys: int = 3000, seed: int = 5) -> dict:
    from paper_2502_17712_b200.geometry import CameraFrame
    rng = np.random.default_rng(seed)
    cam = CameraFrame.from_params(1.0471975511965976, 16 / 9, 0.1, 1000.0, position=(0.3, 1.0, 0.2),
                                  look_at=(0.0, -0.2, -6.0))
    vp = cam.view_proj
    corners = rng.uniform(-10, 10, size=(n_tris, 3, 3))
    homo = np.concatenate([corners, np.ones((n_tris, 3, 1))], axis=2)
    batched = homo @ vp.T                                  # charts.py:274 (batched matmul)
    flat = np.concatenate([corners.reshape(-1, 3), np.ones((3 * n_tris, 1))], axis=1) @ vp.T  # geometry.py:301
    fma_chain = oracle.project(corners.reshape(-1, 3), vp)
    proj_bad = int(np.count_nonzero(batched.reshape(-1, 4).view(np.uint64) != fma_chain.view(np.uint64)))
    flat_bad = int(np.count_nonzero(flat.view(np.uint64) != fma_chain.view(np.uint64)))
    area_bad = 0
    sign_bad = 0
    for k in range(n_polys):
        n = 3 + k % 7
        poly = rng.uniform(-2000, 2000, size=(n, 3))
        x, y = poly[:, 0], poly[:, 1]
        ref = float(np.dot(x, np.roll(y, -1)) - np.dot(y, np.roll(x, -1)))  # charts.py:253
        got = oracle.signed_area2(x, y)
        area_bad += np.float64(ref).view(np.uint64) != np.float64(got).view(np.uint64)
        sign_bad += (ref > 0) != (got > 0) or (ref == 0) != (got == 0)
    return dict(projection_mismatches=proj_bad, projection_2d_mismatches=flat_bad, projection_values=12 * n_tris,
                area_mismatches=int(area_bad), area_sign_mismatches=int(sign_bad), areas=n_polys,
                config=blas_config())


def _check(tag):
    r = probe()
    out = os.environ.get("FA_HOST_PROBE_OUT")
    if out:
        with open(out, "w") as fh:
            json.dump(dict(r, host=tag), fh, indent=1)
    print(json.dumps(r))
    assert r["projection_mismatches"] == 0 and r["projection_2d_mismatches"] == 0, r
    assert r["area_mismatches"] == 0, r


def test_build_host_blas_matches_oracle_chains():
    _check("build container")


@pytest.mark.gpu
def test_gpu_box_host_blas_matches_oracle_chains():
    _check("gpu box")
