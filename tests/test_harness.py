"""CPU: the native harness of libmlg_b200.so (csrc/harness.cu, csrc/errors.cu
make_reference) against the compiled reference's harness (harness.cpp) on the
same inputs -- strict config parsing (same status class and message), order
estimation, reference tables, the CSV writer (byte-identical) and the table
printer (identical text).  Mirrors /root/reference/proj/tests/test_harness.cpp;
no device calls."""
import math

import numpy as np
import pytest

GOOD = """{
  "domain": {"x_min": -1.0, "x_max": 1.0, "y_min": -1.0, "y_max": 1.0},
  "H": 0.5, "delta": 0.5, "m": 1, "n_levels": 2, "degree": 1, "nev": 2,
  "example": "laplace", "cg_tol": 1e-10, "workers": 1, "deterministic": true
}"""


def variant(**kw):
    import json
    j = json.loads(GOOD)
    for k, v in kw.items():
        if v is None:
            j.pop(k)
        else:
            j[k] = v
    return json.dumps(j)


BAD = [
    GOOD.replace('"deterministic": true', '"deterministic": true, "bogus": 1'),  # unknown key
    '{"H": 0.5}',                                                                 # missing keys
    GOOD.replace('"m": 1', '"m": 1.5'),                                           # wrong type
    GOOD.replace('"y_max": 1.0}', '"y_max": 1.0, "z": 0}'),                       # domain key
    "{",                                                                          # invalid JSON
    "[1, 2]",                                                                     # not an object
    GOOD.replace('"laplace"', '"poisson"'),                                       # unknown example
    GOOD.replace('"degree": 1', '"degree": 3'),                                   # validate_config
    GOOD.replace('"nev": 2', '"nev": 0'),
    GOOD.replace('"H": 0.5', '"H": -0.5'),
    GOOD.replace('"x_max": 1.0', '"x_max": -2.0'),
    GOOD.replace('"cg_tol": 1e-10', '"cg_tol": 0'),
    GOOD.replace('"workers": 1', '"workers": 0'),
    GOOD.replace('"deterministic": true', '"deterministic": 1'),
    GOOD.replace('"example": "laplace"', '"example": 1'),
    GOOD.replace('"m": 1', '"m": "1"'),
    GOOD.replace('"domain": {', '"domain": 3, "x": {'),
    GOOD.replace('"n_levels": 2', '"n_levels": 2.0'),
    GOOD + "x",                                                                   # trailing garbage
]

GOODS = [
    GOOD,
    GOOD.replace('"laplace"', '"variable"'),
    GOOD.replace('"H": 0.5', '"H": 1'),                  # integer literal where a number is due
    GOOD.replace('"cg_tol": 1e-10', '"cg_tol": 1E-12'),
    GOOD.replace('"deterministic": true', '"deterministic": false'),
    GOOD.replace('"degree": 1', '"degree": 2'),          # valid for the reference's parser
    '{"workers":3,"nev":1,"n_levels":4,"m":4,"H":0.25,"example":"laplace","delta":0.1,'
    '"degree":1,"domain":{"y_max":1,"y_min":0,"x_max":1,"x_min":0},"cg_tol":1e-8,'
    '"deterministic":true}',
]


@pytest.fixture(scope="module")
def H(mlg):
    from paper_1401_4969_b200 import harness
    return harness


def c_fields(cfg):
    d = cfg.domain
    ex = {"laplace": 0, "variable": 1}[cfg.example]
    return dict(x_min=d.x_min, x_max=d.x_max, y_min=d.y_min, y_max=d.y_max, H=cfg.H,
                delta=cfg.delta, m=cfg.m, n_levels=cfg.n_levels, degree=cfg.degree, nev=cfg.nev,
                example=ex, workers=cfg.workers, cg_tol=cfg.cg_tol,
                deterministic=int(cfg.deterministic))


@pytest.mark.parametrize("text", GOODS)
def test_parse_config_accepts_like_reference(H, oracle_ref, text):
    st, msg, ref_cfg = oracle_ref.parse_config_json(text)
    assert st == 0, msg
    assert c_fields(H.parse_config_json(text)) == ref_cfg


@pytest.mark.parametrize("text", BAD)
def test_parse_config_rejects_like_reference(H, mlg, oracle_ref, text):
    st, msg, _ = oracle_ref.parse_config_json(text)
    assert st == 2
    with pytest.raises(mlg.ConfigError) as e:
        H.parse_config_json(text)
    if msg.startswith("config is not valid JSON"):  # parser diagnostics differ by library
        assert str(e.value).startswith("config is not valid JSON")
    else:
        assert str(e.value) == msg


def test_parse_config_file(H, mlg, oracle_ref, tmp_path):
    p = tmp_path / "c.json"
    p.write_text(GOOD)
    assert c_fields(H.parse_config_file(str(p))) == oracle_ref.parse_config_file(str(p))[2]
    with pytest.raises(mlg.IoError, match="cannot open config file"):
        H.parse_config_file("/nonexistent/config.json")
    assert oracle_ref.parse_config_file("/nonexistent/config.json")[0] == 4


def test_estimate_orders(H, mlg, oracle_ref):  # test_harness.cpp:38-49
    o = H.estimate_orders([0.073555, 0.018534], 2.0)
    assert len(o) == 1 and abs(o[0] - 1.988649) <= 1e-6 * 1.988649
    assert H.estimate_orders([0.5, 0.5], 2.0) == [0.0]
    assert abs(H.estimate_orders([0.4, 0.1], 2.0)[0] - 2.0) <= 2e-14
    rng = np.random.default_rng(5)
    e = rng.uniform(1e-6, 1.0, 9)
    assert np.array_equal(np.array(H.estimate_orders(e, 2.0)), oracle_ref.estimate_orders(e, 2.0))
    assert H.estimate_orders([0.3], 2.0) == []
    for errs, beta in (([0.1, 0.0], 2.0), ([0.1, -0.5], 2.0), ([0.1, 0.05], 1.0)):
        with pytest.raises(mlg.ConfigError):
            H.estimate_orders(errs, beta)


def test_make_reference_matches_reference_table(H, mlg, oracle_ref):
    pts = np.array([[0.0, 0.0], [0.3, -0.7], [-0.9, 0.25], [0.61, 0.61]])
    for nev in (1, 5, 12):
        lam_r, has_r, vals_r = oracle_ref.make_reference("laplace", nev, pts)
        for dom in (None, H.DomainRect(-1.0, 1.0, -1.0, 1.0)):
            refs = H.make_reference("laplace", nev, dom)
            assert np.array_equal(np.array(refs.lambdas), lam_r)  # bitwise
            assert [i in refs.eigenfunctions for i in range(nev)] == has_r.tolist()
            for i, fn in refs.eigenfunctions.items():
                assert (fn.amp, fn.x0, fn.lx) == (1.0, -1.0, 2.0)
                for k, (x, y) in enumerate(pts):
                    gx, gy = fn.gradient(x, y)
                    np.testing.assert_allclose([fn.value(x, y), gx, gy], vals_r[i, k],
                                               rtol=1e-13, atol=1e-15)
    # test_harness.cpp:51-69
    refs = H.make_reference("laplace", 5)
    want = [4.934802200544679, 12.337005501361698, 12.337005501361698, 19.739208802178716,
            24.674011002723397]
    np.testing.assert_allclose(refs.lambdas, want, rtol=1e-14)
    assert sorted(refs.eigenfunctions) == [0, 3]
    assert abs(refs.eigenfunctions[0].value(0.0, 0.0) - 1.0) <= 1e-14
    # variable table (test_harness.cpp:71-77)
    lam_v, has_v, _ = oracle_ref.make_reference("variable", 6)
    rv = H.make_reference("variable", 6)
    assert rv.lambdas == lam_v.tolist() and not rv.eigenfunctions and not has_v.any()
    with pytest.raises(mlg.ConfigError, match="6 modes only"):
        H.make_reference("variable", 7)


def test_make_reference_unit_square(H):
    """The generalised table: unit square -> lambda = pi^2 (m^2 + n^2), b-normalised
    modes (amplitude 2); a 2x1 rectangle orders modes by mx^2/4 + my^2."""
    refs = H.make_reference("laplace", 4, H.DomainRect(0.0, 1.0, 0.0, 1.0))
    pi2 = math.pi ** 2
    np.testing.assert_allclose(refs.lambdas, [2 * pi2, 5 * pi2, 5 * pi2, 8 * pi2], rtol=1e-15)
    assert sorted(refs.eigenfunctions) == [0, 3]
    f = refs.eigenfunctions[0]
    xs = (np.arange(400) + 0.5) / 400
    X, Y = np.meshgrid(xs, xs)
    assert abs(np.mean(f.value(X, Y) ** 2) - 1.0) <= 1e-9
    r = H.make_reference("laplace", 3, H.DomainRect(0.0, 2.0, 0.0, 1.0))
    np.testing.assert_allclose(r.lambdas, [pi2 * (0.25 + 1), pi2 * (1 + 1), pi2 * (2.25 + 1)],
                               rtol=1e-15)
    assert (r.eigenfunctions[0].mx, r.eigenfunctions[1].mx) == (1, 2)


@pytest.fixture(scope="module")
def ref_csv(oracle_ref, tmp_path_factory):
    d = tmp_path_factory.mktemp("csv")
    p = d / "ref.csv"
    oracle_ref.run_experiment(p, domain=(-1.0, 1.0, -1.0, 1.0), H=0.5, delta=0.5, m=1,
                              n_levels=3, nev=2)
    return p


def test_write_csv_byte_identical(H, ref_csv, tmp_path):
    """Rows read back from the reference's CSV, rewritten by the native writer."""
    text = ref_csv.read_text()
    rows = []
    for ln in text.splitlines()[1:]:
        f = ln.split(",")
        rows.append(H.ReportRow(int(f[0]), float(f[1]), int(f[2]), int(f[3]), float(f[4]),
                                float(f[5]), float(f[6]) if f[6] else None,
                                float(f[7]) if f[7] else None, float(f[8]), float(f[9]),
                                float(f[10])))
    out = tmp_path / "ours.csv"
    H.write_csv(H.ExperimentReport(None, rows), str(out))
    assert out.read_bytes() == ref_csv.read_bytes()


def test_print_table_identical(H, mlg, oracle_ref, ref_csv, tmp_path):
    assert H.print_table(str(ref_csv)) == oracle_ref.print_table(ref_csv)
    assert "eigenvalue 1:" in H.print_table(str(ref_csv))
    with pytest.raises(mlg.IoError):
        H.print_table("/nonexistent.csv")
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b\n")
    with pytest.raises(mlg.ConfigError, match="unexpected CSV header"):
        H.print_table(str(bad))
    with pytest.raises(mlg.IoError, match="cannot open output file"):
        H.write_csv(H.ExperimentReport(None, []), "/nonexistent/dir/x.csv")


def test_reaction_seed_key_only_with_reaction(H, mlg):
    """"seed" is the one key beyond the reference's schema, accepted only for the
    B200 extension example "reaction" (BASELINE config 4)."""
    txt = GOOD.replace('"laplace"', '"reaction"').replace('"workers": 1', '"workers": 1, "seed": 5')
    cfg = H.parse_config_json(txt)
    assert cfg.example == "reaction" and cfg.seed == 5
    assert H.parse_config_json(GOOD.replace('"laplace"', '"reaction"')).seed == 0
    with pytest.raises(mlg.ConfigError, match='unknown config field "seed"'):
        H.parse_config_json(GOOD.replace('"workers": 1', '"workers": 1, "seed": 5'))
    with pytest.raises(mlg.ConfigError, match="seed"):
        H.parse_config_json(txt.replace('"seed": 5', '"seed": -1'))
