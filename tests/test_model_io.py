"""§8(f) row 4: model wire format (gmm_io.cpp) — binary SGMM4D01 and the
JSON mirror, round trips and the reference's load-time checks. Host code
only (no GPU)."""
import struct

import numpy as np
import pytest


def model(gm, m=5, seed=0):
    rng = np.random.default_rng(seed)
    w = rng.random(m) + 0.1
    w /= w.sum()
    mu = rng.normal(size=(m, 4))
    cov = np.zeros((m, 10))
    for b in range(m):
        a = rng.normal(size=(4, 4))
        s = a @ a.T + 0.5 * np.eye(4)
        cov[b] = [s[i, j] for i in range(4) for j in range(i + 1)]
    return gm.Gmm(w, mu, cov)


def test_binary_round_trip_is_f32(gm, tmp_path):
    md = model(gm)
    p = str(tmp_path / "m.sgmm")
    gm.save_gmm(md, p)
    raw = open(p, "rb").read()
    assert raw[:8] == b"SGMM4D01" and struct.unpack("<I", raw[8:12])[0] == 5
    assert len(raw) == 12 + 4 * 5 * 15
    back = gm.load_gmm(p)
    assert np.allclose(back.means, np.float32(md.means), atol=0)
    assert np.allclose(back.covariances, np.float32(md.covariances), atol=0)
    assert abs(back.weights.sum() - 1.0) < 1e-15  # renormalised after the f32 narrowing
    w32 = np.float32(md.weights).astype(np.float64)
    assert np.allclose(back.weights, w32 / w32.sum(), rtol=1e-15)


def test_json_round_trip_exact(gm, tmp_path):
    md = model(gm, 7, 3)
    p = str(tmp_path / "m.json")
    gm.save_gmm(md, p, json=True)
    back = gm.load_gmm(p, json=True)
    assert np.array_equal(back.means, md.means) and np.array_equal(back.covariances, md.covariances)
    assert np.allclose(back.weights, md.weights, rtol=1e-15)


def test_load_errors(gm, tmp_path):
    md = model(gm)
    p = tmp_path / "m.sgmm"
    gm.save_gmm(md, str(p))
    raw = bytearray(p.read_bytes())
    bad = tmp_path / "bad.sgmm"
    bad.write_bytes(b"XGMM4D01" + raw[8:])
    with pytest.raises(gm.GmmFormatError, match="bad magic"):
        gm.load_gmm(str(bad))
    bad.write_bytes(raw[:40])
    with pytest.raises(gm.GmmFormatError, match="truncated"):
        gm.load_gmm(str(bad))
    zero = bytearray(raw)
    zero[8:12] = struct.pack("<I", 0)
    bad.write_bytes(zero)
    with pytest.raises(gm.GmmFormatError, match="zero components"):
        gm.load_gmm(str(bad))
    wsum = bytearray(raw)
    wsum[12:16] = struct.pack("<f", 0.9)
    bad.write_bytes(wsum)
    with pytest.raises(gm.NumericalError, match="beyond the 1e-6"):
        gm.load_gmm(str(bad))
    nspd = gm.Gmm(md.weights, md.means, md.covariances.copy())
    nspd.covariances[2, :] = [1, 2, 1, 0, 0, 1, 0, 0, 0, 1]
    gm.save_gmm(nspd, str(bad))
    with pytest.raises(gm.NumericalError, match="component 2 is not positive definite"):
        gm.load_gmm(str(bad))
    with pytest.raises(gm.IoError):
        gm.load_gmm(str(tmp_path / "missing.sgmm"))
    (tmp_path / "x.json").write_text('{"weights": [1.0], "means": [[0,0,0]]}')
    with pytest.raises(gm.GmmFormatError):
        gm.load_gmm(str(tmp_path / "x.json"), json=True)


def test_json_rejects_non_numeric_elements(gm, tmp_path):
    """A string or nested array inside a mean / covariance row is a format
    error (the reference's get<double>() raises GmmFormatError), not 0.0."""
    import json
    md = model(gm, 3, 1)
    p = str(tmp_path / "m.json")
    gm.save_gmm(md, p, json=True)
    doc = json.load(open(p))
    for field, bad in (("means", "x"), ("covariances_packed", [1.0])):
        d = json.loads(json.dumps(doc))
        d[field][1][2] = bad
        q = str(tmp_path / f"bad_{field}.json")
        json.dump(d, open(q, "w"))
        with pytest.raises(gm.IoError, match="malformed"):
            gm.load_gmm(q, json=True)
