"""ReducedModel store: round trip bit-exact, byte-stable rewrite, corruption → StoreError."""

import json

import numpy as np
import pytest

from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import store, synthetic
from paper_1807_11866_b200.errors import StoreError


def _files(path):
    return {p.name: p.read_bytes() for p in sorted(path.iterdir())}


@pytest.mark.parametrize("kind", ["cfg4", "lifted"])
def test_round_trip_bit_exact(tmp_path, kind):
    m = (synthetic.make_model(9, 3, "trig3", n_p=5, name="cfg-like") if kind == "cfg4"
         else synthetic.make_lifted_model(8, 2, n_p=4))
    a = store.save_model(m, tmp_path / "a.rbm")
    r = store.load_model(a)
    for name in ("A", "C", "f", "Mp", "Bq"):
        assert np.array_equal(getattr(r, name), getattr(m, name))
    for fam in ("linear", "quadratic", "load", "coupling"):
        assert getattr(r, f"theta_{fam}") == getattr(m, f"theta_{fam}")   # scales bit-exact via hex
    assert r.nu_linear == m.nu_linear and r.name == m.name
    b = store.save_model(r, tmp_path / "b.rbm")
    assert _files(a) == _files(b)                                          # write→read→write byte-identical
    mu = (synthetic.make_mu(4, 200.0) if kind == "cfg4" else synthetic.make_lifted_mu(4))
    u1 = oracle.solve_batch(m, mu)[0]
    u2 = oracle.solve_batch(store.load_model(b, mmap=True), mu)[0]
    assert np.array_equal(u1, u2)


def test_manifest_contents(tmp_path):
    m = synthetic.make_lifted_model(6, 1)
    p = store.save_model(m, tmp_path / "m.rbm")
    man = json.loads((p / "manifest.json").read_text())
    assert man["format"] == "rbflow-reduced-model" and man["basis"] == {"n_velocity": 6, "n_pressure": 0, "n_attached_pressure": 0}
    assert set(man["families"]) == {"linear", "quadratic", "load"}
    assert len(man["families"]["linear"]["terms"]) == 4 * 1 + 3 + 4 * 1 + 1
    assert man["arrays"]["C"]["shape"] == [5, 6, 6, 6]
    assert (p / "C.f64").stat().st_size == 5 * 6 ** 3 * 8
    assert man["provenance"]["form"] == "lifted-piola"


def test_corruption_detected(tmp_path):
    m = synthetic.make_lifted_model(6, 1)
    p = store.save_model(m, tmp_path / "m.rbm")
    raw = bytearray((p / "A.f64").read_bytes())
    raw[17] ^= 1
    (p / "A.f64").write_bytes(bytes(raw))
    with pytest.raises(StoreError, match="sha256"):
        store.load_model(p)
    store.save_model(m, p)
    (p / "C.f64").write_bytes((p / "C.f64").read_bytes()[:-8])
    with pytest.raises(StoreError, match="bytes"):
        store.load_model(p)
    store.save_model(m, p)
    man = json.loads((p / "manifest.json").read_text())
    man["families"]["load"]["terms"][0]["scale_hex"] = float(2.0).hex()
    (p / "manifest.json").write_text(json.dumps(man))
    with pytest.raises(StoreError, match="hash"):
        store.load_model(p)
    with pytest.raises(StoreError, match="manifest"):
        store.load_model(tmp_path / "missing.rbm")


@pytest.mark.gpu
def test_store_to_device(tmp_path):
    """Ingestion path: store → (mmap) ReducedModel → rbns_model_create2 → solve equals the in-memory model's."""
    torch = pytest.importorskip("torch")
    from paper_1807_11866_b200 import online

    m = synthetic.make_lifted_model(20, 3, n_p=6)
    p = store.save_model(m, tmp_path / "m.rbm")
    mu = torch.from_numpy(synthetic.make_lifted_mu(256)).cuda()
    with online.DeviceModel(m, 0) as d1, online.DeviceModel(store.load_model(p, mmap=True), 0) as d2:
        r1, r2 = d1.solve(mu), d2.solve(mu)
        torch.cuda.synchronize()
        assert torch.equal(r1.u, r2.u) and torch.equal(r1.p, r2.p) and torch.equal(r1.iters, r2.iters)


def test_attached_pressure_modes_round_trip(tmp_path):
    """The combined scheme's attached pressure modes are stored and hashed with the model."""
    m = synthetic.make_model(8, 3, "trig3", n_p=5, attached=5)
    p = store.save_model(m, tmp_path / "att.rbm")
    back = store.load_model(p)
    assert back.n_att == 5
    np.testing.assert_array_equal(back.P_att, m.P_att)
    man = json.loads((p / "manifest.json").read_text())
    assert man["basis"]["n_attached_pressure"] == 5 and "P_att" in man["arrays"]
    raw = bytearray((p / "P_att.f64").read_bytes())
    raw[0] ^= 1
    (p / "P_att.f64").write_bytes(bytes(raw))
    with pytest.raises(store.StoreError):
        store.load_model(p)
