"""Native OBJ reader/writer (sbr_obj_*) vs the reference-equivalent Python
loops (geometry.py:190-265 restated in geometry._load_mesh_py/_save_obj_py):
same vertices, triangles, face labels, error messages and exceptions.
Host-only: needs libsbr200.so but no GPU."""

import warnings

import numpy as np
import pytest

import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import geometry as G
from paper_2604_09243_b200 import _native as nat


def _write(tmp_path, name, text, binary=False):
    p = tmp_path / name
    if binary:
        p.write_bytes(text)
    else:
        p.write_bytes(text.encode("utf-8"))
    return p


def _same_mesh(a, b):
    for k in ("v0", "v1", "v2", "normals"):
        assert np.array_equal(getattr(a, k), getattr(b, k), equal_nan=True), k
    assert np.array_equal(a.aabb.min, b.aabb.min) and np.array_equal(a.aabb.max, b.aabb.max)


GOOD = [
    "# header\nv 0 0 0\nv 1 0 0\nv 0 1 0\nv 1 1 0\n\nf 1 2 3\nf 2 4 3\n",
    "v 0 0 0\r\nv 1 0 0\r\nv 0 1 0\r\nv 1 1 0.5\r\nf 1 2 3 4\r\n",          # CRLF, quad
    "v 0 0 0\rv 1 0 0\rv 0 1 0\rf 1 2 3\r",                                  # lone CR
    "v\t0 0 0\nv 1e0 0 0\x0c\nv 0 +1 -0\nvn 0 0 1\nvt 0 0\nf 1/1/1 2//1 3/2\n",
    "v 0 0 0 1\nv 1 0 0 1\nv 0 1 0 1\nv -.5 .5 5.\nf -4 -3 -2\nf 1 2 3 4\ng x\no y\n",
    "v 0 0 0\nv 2.5e-3 0 0\nv 0 1E+2 0\nv 3 3 3\nv 3 4 3\nf 1 2 3\nf 4 5 1 2 3\n",
    "  # indented comment\n#f 1 2 3\nv 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n",
]


@pytest.mark.parametrize("text", GOOD)
def test_native_reader_matches_python_loop(tmp_path, text):
    p = _write(tmp_path, "m.obj", text)
    assert nat.obj_read(p) is not None          # took the native path
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _same_mesh(sbr.load_mesh(p), G._load_mesh_py(p))


def test_native_reader_labels_and_fans(tmp_path):
    p = _write(tmp_path, "m.obj", GOOD[5])
    v, f, lab = nat.obj_read(p)
    assert f.tolist() == [[0, 1, 2], [3, 4, 0], [3, 0, 1], [3, 1, 2]]
    assert lab.tolist() == [0, 1, 1, 1]
    assert v[1, 0] == 2.5e-3 and v[2, 1] == 100.0


BAD = [
    ("v 0 0\nf 1 2 3\n", "malformed vertex record"),
    ("v 0 0 0\nv 1 0 0\nf 1 2\n", "face with <3 vertices"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n", "zero vertex index in face 0"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\nf 1 2 4\n", "vertex index 4 out of range in face 1"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf -4 1 2\n", "vertex index -4 out of range in face 0"),
    ("v 0 0 0\n# only vertices\n", "no faces found"),
]


@pytest.mark.parametrize("text,msg", BAD)
def test_native_reader_errors_match(tmp_path, text, msg):
    p = _write(tmp_path, "bad.obj", text)
    with pytest.raises(sbr.ValidationError) as e_nat:
        sbr.load_mesh(p)
    with pytest.raises(sbr.ValidationError) as e_py:
        G._load_mesh_py(p)
    assert str(e_nat.value) == str(e_py.value)
    assert msg in str(e_nat.value)


@pytest.mark.parametrize("text", [
    "v 1_0 0 0\nv 0 1 0\nv 0 0 1\nf 1 2 3\n",       # Python float() accepts underscores
    "v 0x1p3 0 0\nv 0 1 0\nv 0 0 1\nf 1 2 3\n",      # Python float() rejects hex
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 +0_3\n",      # int() with underscore
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 /3\n",        # empty index
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3 # tail\n",  # int('#') raises in the reference
])
def test_unusual_syntax_defers_to_python(tmp_path, text):
    p = _write(tmp_path, "odd.obj", text)
    assert nat.obj_read(p) is None
    try:
        ref = G._load_mesh_py(p)
    except Exception as e:   # the reference raises whatever Python raises
        with pytest.raises(type(e)):
            sbr.load_mesh(p)
    else:
        _same_mesh(sbr.load_mesh(p), ref)


def test_non_ascii_and_missing_file(tmp_path):
    p = _write(tmp_path, "u.obj", b"# caf\xe9\nv 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n", binary=True)
    assert nat.obj_read(p) is None
    _same_mesh(sbr.load_mesh(p), G._load_mesh_py(p))
    with pytest.raises(FileNotFoundError):
        sbr.load_mesh(tmp_path / "missing.obj")


def test_degenerate_drop_and_strict(tmp_path):
    p = _write(tmp_path, "d.obj", "v 0 0 0\nv 1 0 0\nv 2 0 0\nv 0 1 0\nf 1 2 3\nf 1 2 4\n")
    with pytest.warns(UserWarning, match="dropping 1 zero-area"):
        m = sbr.load_mesh(p)
    assert m.triangle_count == 1
    with pytest.raises(sbr.ValidationError, match="face index \\[0\\]"):
        sbr.load_mesh(p, strict=True)


def test_writer_matches_python_loop(tmp_path):
    m = sbr.generate_icosphere(1.0, 2)
    tri = np.stack([m.v0, m.v1, m.v2], 1).copy()
    tri[0, 0] = [0.0, -0.0, 1e-300]            # -0.0 shares with 0.0 like a tuple key
    tri[1, 0] = [-0.0, 0.0, 1e-300]
    m2 = sbr.mesh_from_soup(tri)
    a, b = tmp_path / "native.obj", tmp_path / "py.obj"
    sbr.save_obj(m2, a)
    G._save_obj_py(m2, b)
    assert a.read_bytes() == b.read_bytes()
    _same_mesh(sbr.load_mesh(a), m2)


def test_large_mesh_roundtrip(tmp_path):
    from paper_2604_09243_b200 import meshgen
    m = meshgen.generate_aircraft(density=0.05)
    p = tmp_path / "air.obj"
    sbr.save_obj(m, p)
    back = sbr.load_mesh(p)
    assert np.array_equal(back.v0, m.v0) and np.array_equal(back.v2, m.v2)


def test_number_parsing_is_correctly_rounded(tmp_path):
    """Every coordinate equals Python's float() of the same text: random
    magnitudes 1e-300..1e300, subnormals, 5- to 21-digit mantissas, signs."""
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.standard_normal(9000) * 10.0 ** rng.integers(-300, 300, 9000),
                           rng.random(9000), np.array([5e-324, 2.2250738585072014e-308,
                                                       1.7976931348623157e308, 0.1, 0.3])])
    vals = vals[: len(vals) // 3 * 3]
    fmts = [lambda x: repr(float(x)), lambda x: "%.20e" % x, lambda x: "%.5g" % x,
            lambda x: "+%r" % abs(float(x)), lambda x: "%.17f" % x]
    lines = ["v " + " ".join(fmts[(i + j) % len(fmts)](x) for j, x in enumerate(vals[i:i + 3]))
             for i in range(0, len(vals), 3)]
    p = _write(tmp_path, "r.obj", "\n".join(lines) + "\nf 1 2 3\n")
    got = nat.obj_read(p)
    assert got is not None
    ref = np.array([[float(t) for t in ln.split()[1:4]] for ln in lines])
    assert np.array_equal(got[0], ref)


def test_dump_hits_csv_matches_python_loop(tmp_path):
    from paper_2604_09243_b200 import transport as TR
    rng = np.random.default_rng(5)
    n_u, n_v = 37, 53
    n = n_u * n_v
    rec = sbr.HitRecords(valid=rng.random(n) < 0.4,
                         normal0=np.where(rng.random((n, 1)) < 0.5, 0.0,
                                          rng.standard_normal((n, 3))) * np.array([1, -1, 1e-7]),
                         path=rng.random(n) * 1e3, bounces=rng.integers(0, 6, n).astype(np.int32),
                         escaped=rng.random(n) < 0.5, out_dir=rng.standard_normal((n, 3)))
    rec.normal0[3] = [-0.0, np.inf, -np.inf]
    rec.path[4] = np.nan

    class G:
        pass
    g = G()
    g.n_u, g.n_v = n_u, n_v
    a, b = tmp_path / "nat.csv", tmp_path / "py.csv"
    TR.dump_hits_csv(rec, g, a)
    TR._dump_hits_csv_py(rec, g, b)
    assert a.read_bytes() == b.read_bytes()
