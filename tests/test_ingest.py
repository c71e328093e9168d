"""§8(f) row 2: device ingest (decimate + image_pair_to_cloud,
ingest.cpp:27-75) against the host restatement, bit-exact."""
import numpy as np
import pytest


def host_image_pair_to_cloud(depth, inten, intr, inv_max=1 / 255.0, depth_scale=1000.0, f=1):
    """ingest.cpp:27-75 restated in numpy (row-major, zero depths dropped)."""
    fx, fy, cx, cy = intr
    d = depth[::f, ::f][: depth.shape[0] // f, : depth.shape[1] // f]
    it = inten[::f, ::f][: depth.shape[0] // f, : depth.shape[1] // f]
    fx, fy, cx, cy = fx / f, fy / f, cx / f, cy / f
    v, u = np.nonzero(d > 0)
    z = d[v, u] * (1.0 / depth_scale)
    return np.column_stack([(u - cx) * z / fx, (v - cy) * z / fy, z, it[v, u] * inv_max])


def test_synthetic_images_match_cloud(gm):
    dep, inten, intr = gm.synthetic_frame_images()
    ref = gm.synthetic_frame_cloud()
    assert np.array_equal(host_image_pair_to_cloud(dep, inten, intr), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("factor", [1, 2, 3])
def test_device_ingest_bit_exact(gm, ctx, factor):
    dep, inten, intr = gm.synthetic_frame_images()
    dep = dep.copy()
    dep[100:140, 200:260] = 0  # holes are dropped
    n, pts = ctx.ingest_images(dep, inten, intr, factor=factor, want_points=True)
    ref = host_image_pair_to_cloud(dep, inten, intr, f=factor)
    assert n == len(ref)
    assert np.array_equal(pts, ref)


@pytest.mark.gpu
def test_ingest_then_fit_equals_fit(gm, ctx):
    dep, inten, intr = gm.synthetic_frame_images(160, 120)
    ctx.ingest_images(dep, inten, intr)
    em = gm.EmParams(30, 1e-3, 1e-6, 0)
    a = ctx.fit_k_resident(16, em)
    b = gm.fit_k(gm.synthetic_frame_cloud(160, 120), 16, em, ctx=ctx)
    assert a.em_iterations == b.em_iterations
    assert np.array_equal(a.model.weights, b.model.weights)


@pytest.mark.gpu
def test_ingest_errors(gm, ctx):
    dep, inten, intr = gm.synthetic_frame_images(64, 48)
    with pytest.raises(gm.NumericalError, match="empty cloud"):
        ctx.ingest_images(np.zeros_like(dep), inten, intr)
    with pytest.raises(ValueError, match="decimation factor"):
        ctx.ingest_images(dep, inten, intr, factor=0)
    with pytest.raises(ValueError, match="principal point"):
        ctx.ingest_images(dep, inten, (50.0, 50.0, -1.0, 10.0))
