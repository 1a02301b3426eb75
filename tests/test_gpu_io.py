"""§8f row 4: Matrix Market and VTK output of device data in the reference's formats
(linsolve.cpp:478-490, postproc.cpp:111-167).  The Matrix Market text is compared byte for byte
with the reference's format string; the VTK file is parsed back (ASCII and BINARY) and checked
against the oracle's cell order and vertex coordinates."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    import paper_1806_09924_b200 as cf
    return cf


def _state(P, seed):
    rng = np.random.default_rng(seed)
    x = np.zeros(P.n_total)
    x[:P.n_u] = 1e-2 * rng.uniform(-1, 1, P.n_u)
    x[P.n_u:] = rng.uniform(0, 1, P.n_vertices)
    return x, rng.uniform(0, 1, P.n_vertices)


@pytest.mark.parametrize("d,n0,r", [(2, 3, 1), (3, 2, 1)])
def test_matrix_market_reference_text(cf, tmp_path, d, n0, r):
    P = cf.Problem(d, 1.0, n0, r)
    x, pt = _state(P, 5)
    J = cf.assemble_jacobian(P, cf.build_constraints(P), cf.Material(), cf.Regularization(0.3, 1e-6), x, pt)
    for w in range(3):
        path = tmp_path / f"J{w}.mtx"
        J.write_matrix_market(w, str(path))
        A = J.csr(w)
        lines = ["%%MatrixMarket matrix coordinate real general", f"{A.rows} {A.cols} {A.nnz}"]
        for i in range(A.rows):
            for k in range(A.ptr[i], A.ptr[i + 1]):
                lines.append("%d %d %.17g" % (i + 1, A.col[k] + 1, A.val[k]))
        assert path.read_text() == "\n".join(lines) + "\n"
        import scipy.io
        M = scipy.io.mmread(str(path), spmatrix=False).tocsr()
        assert np.array_equal(M.toarray(), A.to_scipy().toarray())


def _parse_vtk(path, binary):
    raw = open(path, "rb").read()
    pos = 0

    def line():
        nonlocal pos
        e = raw.index(b"\n", pos)
        s = raw[pos:e].decode()
        pos = e + 1
        return s

    head = [line() for _ in range(4)]
    out = {"head": head}

    def block(count, dtype, width):
        nonlocal pos
        if binary:
            n = count * width
            a = np.frombuffer(raw, dtype=np.dtype(dtype).newbyteorder(">"), count=n, offset=pos)
            pos += n * np.dtype(dtype).itemsize + 1  # trailing newline
            return a.reshape(count, width).astype(dtype)
        rows = [line().split() for _ in range(count)]
        return np.array(rows, dtype=dtype).reshape(count, -1)

    t = line().split()
    nv = int(t[1])
    out["points"] = block(nv, np.float64, 3)
    t = line().split()
    nc, tot = int(t[1]), int(t[2])
    out["cells"] = block(nc, np.int32, tot // nc)
    t = line().split()
    out["types"] = block(nc, np.int32, 1)
    line()  # POINT_DATA
    line()  # VECTORS u double
    out["u"] = block(nv, np.float64, 3)
    line()
    line()
    out["phi"] = block(nv, np.float64, 1)[:, 0]
    if pos < len(raw):
        line()
        line()
        out["phi_old"] = block(nv, np.float64, 1)[:, 0]
    return out


@pytest.mark.parametrize("binary", [False, True])
@pytest.mark.parametrize("d,n0,r", [(2, 3, 2), (3, 2, 1)])
def test_vtk_against_oracle_mesh(cf, orc, tmp_path, d, n0, r, binary):
    P = cf.Problem(d, 2.0, n0, r)
    O = orc.Problem(d, 2.0, n0, r)
    x, po = _state(P, 9)
    path = tmp_path / "sol.vtk"
    cf.write_vtk(str(path), P, x, po, binary=binary)
    v = _parse_vtk(path, binary)
    assert v["head"][2] == ("BINARY" if binary else "ASCII") and v["head"][3] == "DATASET UNSTRUCTURED_GRID"
    assert np.array_equal(v["points"], O.coords())
    nc = P.n_cells
    npc = 1 << d
    perm = [0, 1, 3, 2] if d == 2 else [0, 1, 3, 2, 4, 5, 7, 6]
    order = O.cell_order()  # reference active-cell order as lexicographic cell indices
    nc1 = (n0 << r)
    exp = np.zeros((nc, npc + 1), dtype=np.int64)
    exp[:, 0] = npc
    for t, c in enumerate(order):
        cx, cy, cz = c % nc1, (c // nc1) % nc1, c // (nc1 * nc1)
        for k, corner in enumerate(perm):
            exp[t, 1 + k] = (cx + (corner & 1)) + (nc1 + 1) * ((cy + ((corner >> 1) & 1)) + (nc1 + 1) * (cz + ((corner >> 2) & 1)))
    assert np.array_equal(v["cells"], exp)
    assert np.all(v["types"] == (9 if d == 2 else 12))
    u = np.zeros((P.n_vertices, 3))
    u[:, :d] = x[:P.n_u].reshape(-1, d)
    assert np.array_equal(v["u"], u)
    assert np.array_equal(v["phi"], x[P.n_u:])
    assert np.array_equal(v["phi_old"], po)
