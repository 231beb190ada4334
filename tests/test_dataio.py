"""Dataset ingestion (dataio.py:1-457) and sparse factor matrices (row 4).

CPU: the generators write byte-identical files to the reference's (committed under
tests/golden/dataio/ by oracle/gen_golden_dataio.py), schema / triplet / CSV parsing and the
reference's error behaviour. GPU: ``load`` through the device constructors reproduces the
reference's materialized T and target bit for bit, and ``fb_csr_expand`` (scipy CSR factor
matrices) is bit-exact against scipy's own densification.
"""
import filecmp
import json
import os

import numpy as np
import pytest

import golden_io

from paper_1612_07448_b200 import dataio
from paper_1612_07448_b200.exceptions import DataError

DIR = os.path.join(golden_io.GOLDEN, "dataio")
CASES = ["pkfk_dense", "pkfk_sparse", "mn", "star_strings"]
GEN = {
    "pkfk_dense": lambda d: dataio.gen_pkfk(dataio.SynthParams(n_s=40, n_r=8, d_s=3, d_r=4, seed=3), d),
    "pkfk_sparse": lambda d: dataio.gen_pkfk(
        dataio.SynthParams(n_s=60, n_r=10, d_s=40, d_r=30, density=0.03, seed=5), d),
    "mn": lambda d: dataio.gen_mn(dataio.SynthParams(n_s=30, n_r=12, d_s=2, d_r=3, n_u=5, seed=9), d),
}


def _golden(name):
    with np.load(os.path.join(DIR, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


# --------------------------------------------------------------------------- CPU
@pytest.mark.parametrize("name", sorted(GEN))
def test_generators_byte_identical(name, tmp_path):
    out = tmp_path / name
    schema = GEN[name](str(out))
    assert os.path.basename(schema) == "schema.json"
    ref = os.path.join(DIR, name)
    files = sorted(os.listdir(ref))
    assert sorted(os.listdir(out)) == files
    for f in files:
        assert filecmp.cmp(out / f, os.path.join(ref, f), shallow=False), f


def test_load_schema_roundtrip():
    sd = dataio.load_schema(os.path.join(DIR, "star_strings", "schema.json"))
    assert sd.entity_path == "entity.csv" and sd.target == "y"
    assert [k.column for k in sd.keys] == ["ka", "kb"] and {k.kind for k in sd.keys} == {"pkfk"}
    assert [(t.id, t.pk) for t in sd.tables] == [("A", "name"), ("B", None)]
    doc = json.load(open(os.path.join(DIR, "star_strings", "schema.json")))
    assert sd.to_json_dict() == doc


def test_schema_validation(tmp_path):
    t = (dataio.TableDef("0", "t.csv"),)
    with pytest.raises(DataError, match="duplicate"):
        dataio.SchemaDescriptor("e.csv", (), t + t)
    with pytest.raises(DataError, match="undeclared"):
        dataio.SchemaDescriptor("e.csv", (dataio.SchemaKey("k", "9"),), t)
    with pytest.raises(DataError, match="unknown join kind"):
        dataio.SchemaDescriptor("e.csv", (dataio.SchemaKey("k", "0", "fk"),), t)
    with pytest.raises(DataError, match="not found"):
        dataio.load_schema(tmp_path / "nope.json")
    (tmp_path / "bad.json").write_text('{"entity": {}}')
    with pytest.raises(DataError, match="malformed"):
        dataio.load_schema(tmp_path / "bad.json")


def test_synth_params_validation():
    with pytest.raises(DataError):
        dataio.SynthParams(n_s=0, n_r=1, d_s=1, d_r=1)
    with pytest.raises(DataError):
        dataio.SynthParams(n_s=4, n_r=1, d_s=1, d_r=1, density=0.0)
    with pytest.raises(DataError):
        dataio.SynthParams(n_s=4, n_r=1, d_s=1, d_r=1, n_u=5)
    with pytest.raises(DataError, match="n_s >= n_r"):
        dataio.gen_pkfk(dataio.SynthParams(n_s=2, n_r=3, d_s=1, d_r=1), "/nonexistent")
    with pytest.raises(DataError, match="n_u"):
        dataio.gen_mn(dataio.SynthParams(n_s=2, n_r=3, d_s=1, d_r=1), "/nonexistent")


def test_read_triplet_matches_file_lines():
    path = os.path.join(DIR, "pkfk_sparse", "table_0.triplet")
    m = dataio.read_triplet(path)
    lines = open(path).read().split("\n")
    rows, cols = (int(v) for v in lines[0].split(","))
    want = np.zeros((rows, cols))
    for ln in lines[2:]:
        if ln:
            r, c, v = ln.split(",")
            want[int(r), int(c)] += float(v)
    assert m.shape == (rows, cols) and m.nnz == int(lines[1])
    np.testing.assert_array_equal(m.toarray(), want)
    g = _golden("pkfk_sparse")
    assert m.shape[1] == g["t"].shape[1] - 40


def test_triplet_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(0)
    a = np.where(rng.random((9, 7)) < 0.2, rng.standard_normal((9, 7)), 0.0)
    dataio.write_triplet(tmp_path / "a.triplet", a)
    np.testing.assert_array_equal(dataio.read_triplet(tmp_path / "a.triplet").toarray(), a)
    dataio.write_triplet(tmp_path / "z.triplet", np.zeros((3, 2)))
    assert dataio.read_triplet(tmp_path / "z.triplet").shape == (3, 2)
    (tmp_path / "h.triplet").write_text("3;2\n1\n0,0,1\n")
    with pytest.raises(DataError, match="header"):
        dataio.read_triplet(tmp_path / "h.triplet")
    (tmp_path / "n.triplet").write_text("3,2\n2\n0,0,1\n")
    with pytest.raises(DataError, match="claims 2"):
        dataio.read_triplet(tmp_path / "n.triplet")
    with pytest.raises(DataError, match="not found"):
        dataio.read_triplet(tmp_path / "missing.triplet")


def test_csv_errors(tmp_path):
    (tmp_path / "e.csv").write_text("")
    with pytest.raises(DataError, match="empty file"):
        dataio._CsvTable(tmp_path / "e.csv")
    (tmp_path / "h.csv").write_text("a,b\n")
    with pytest.raises(DataError, match="no data rows"):
        dataio._CsvTable(tmp_path / "h.csv")
    (tmp_path / "v.csv").write_text("a,b\n1,2\n3,x7\n")
    with pytest.raises(DataError, match=r"v.csv:3: column 'b' has unparseable value 'x7'"):
        dataio._CsvTable(tmp_path / "v.csv")
    (tmp_path / "w.csv").write_text("a,b\n1,2\n3,4,5\n")
    with pytest.raises(DataError, match="columns"):
        dataio._CsvTable(tmp_path / "w.csv")
    t = dataio._CsvTable(os.path.join(DIR, "pkfk_dense", "entity.csv"), string_cols=("k_0",))
    assert t.names[:2] == ["target", "k_0"] and t.rows == 40
    assert t.strings("k_0").to_pylist()[:8] == [str(i) for i in range(1, 9)]


def test_positional_keys():
    import pyarrow as pa

    pk = pa.array(["b", "a", "c"])
    np.testing.assert_array_equal(dataio._positional_keys(pa.array(["a", "c", "a", "b"]), pk, "p", "k"),
                                  [2, 3, 2, 1])
    with pytest.raises(DataError, match="dangling key: entity row 1 value 'q'"):
        dataio._positional_keys(pa.array(["a", "q"]), pk, "p", "k")
    with pytest.raises(DataError, match="duplicate primary-key"):
        dataio._positional_keys(pa.array(["a"]), pa.array(["a", "a"]), "p", "k")


def test_join_codes_equal_iff_strings_equal():
    import pyarrow as pa

    a, b = dataio._join_codes(pa.array(["3", "1", "3", "7"]), pa.array(["1", "7", "9", "3.0"]))
    assert a[0] == a[2] and a[1] == b[0] and a[3] == b[1]
    assert b[3] not in set(a.tolist()) and b[2] not in set(a.tolist())


def test_maybe_sparse():
    d = np.eye(30)  # 3.3 % nonzero
    assert hasattr(dataio._maybe_sparse(d, None), "tocsr")
    assert isinstance(dataio._maybe_sparse(d, "dense"), np.ndarray)
    assert hasattr(dataio._maybe_sparse(np.ones((2, 2)), "sparse"), "tocsr")
    assert isinstance(dataio._maybe_sparse(np.ones((2, 2)), None), np.ndarray)


def test_load_rejects_mixed_and_multi_mn(tmp_path):
    sd = dataio.SchemaDescriptor("entity.csv", (dataio.SchemaKey("k_0", "0", "pkfk"),
                                                dataio.SchemaKey("k_0", "0", "mn")),
                                 (dataio.TableDef("0", "table_0.csv"),), base_dir=os.path.join(DIR, "pkfk_dense"))
    with pytest.raises(DataError, match="mixing"):
        dataio.load(sd)


# --------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_load_bit_exact_vs_reference(name):
    import paper_1612_07448_b200 as fb

    g = _golden(name)
    nm, y = dataio.load(os.path.join(DIR, name, "schema.json"))
    assert nm.variant == str(g["variant"])
    t = fb.materialize(nm)
    assert t.shape == tuple(g["shape"])
    np.testing.assert_array_equal(t, g["t"])
    np.testing.assert_array_equal(y, g["y"])
    # the loaded matrix runs through the operators
    x = np.random.default_rng(1).standard_normal((t.shape[1], 2))
    np.testing.assert_allclose(fb.lmm(nm, x), t @ x, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(fb.col_sums(nm).ravel(), t.sum(axis=0), rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_load_dangling_positional_key(tmp_path):
    import shutil

    d = tmp_path / "ds"
    shutil.copytree(os.path.join(DIR, "pkfk_dense"), d)
    lines = (d / "entity.csv").read_text().split("\n")
    f = lines[5].split(",")
    f[1] = "99"
    lines[5] = ",".join(f)
    (d / "entity.csv").write_text("\n".join(lines))
    with pytest.raises(DataError, match="nonexistent attribute row 99"):
        dataio.load(d / "schema.json")


@pytest.mark.gpu
def test_csr_expand_bit_exact():
    import torch
    from scipy import sparse

    from paper_1612_07448_b200 import _device as D

    rng = np.random.default_rng(4)
    for n, d, dens in [(1, 1, 1.0), (1000, 37, 0.05), (4099, 300, 0.01), (64, 5, 0.0)]:
        a = sparse.random(n, d, density=dens, format="coo", random_state=rng, data_rvs=rng.standard_normal)
        # duplicate entries are summed, as scipy does
        dup = sparse.coo_matrix((a.data[: a.nnz // 3], (a.row[: a.nnz // 3], a.col[: a.nnz // 3])), shape=a.shape)
        m = sparse.coo_matrix((np.r_[a.data, dup.data], (np.r_[a.row, dup.row], np.r_[a.col, dup.col])), shape=a.shape)
        t = D.as_matrix(m.tocsr())
        assert t.is_cuda and t.dtype == torch.float64
        np.testing.assert_array_equal(t.cpu().numpy(), m.toarray())
    assert D.as_matrix(sparse.csr_matrix((0, 4))).shape == (0, 4)


@pytest.mark.gpu
def test_sparse_factors_through_builders():
    from scipy import sparse

    import paper_1612_07448_b200 as fb

    rng = np.random.default_rng(8)
    s = sparse.random(500, 20, density=0.04, format="csr", random_state=rng)
    r = sparse.random(40, 60, density=0.03, format="csr", random_state=rng)
    keys = rng.integers(1, 41, size=500)
    nm_sp = fb.build_pkfk(s, keys, r)
    nm_d = fb.build_pkfk(s.toarray(), keys, r.toarray())
    np.testing.assert_array_equal(fb.materialize(nm_sp), fb.materialize(nm_d))
    x = rng.standard_normal((80, 3))
    # factors at <= 5 % density stay CSR and the LMM reads them natively (csr_ops): the same
    # products, summed in CSR order instead of the dense kernels' order
    assert nm_sp.has_csr
    np.testing.assert_allclose(fb.lmm(nm_sp, x), fb.lmm(nm_d, x), rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(fb.crossprod(nm_sp), fb.crossprod(nm_d))  # dense expansion


def test_sparse_input_fails_loudly_without_gpu():
    """No CPU fallback: a CSR factor needs the device expansion kernel."""
    import torch
    from scipy import sparse

    from paper_1612_07448_b200 import _device as D
    from paper_1612_07448_b200.exceptions import ExtensionMissingError

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by test_csr_expand_bit_exact")
    with pytest.raises(ExtensionMissingError):
        D.as_matrix(sparse.eye(3, format="csr"))
    with pytest.raises(ExtensionMissingError):
        dataio.load(os.path.join(DIR, "pkfk_sparse", "schema.json"))
