"""CLI end to end on the B200: sign -> verify for models and datasets, tamper detection, the
strategy table against digests printed by the reference (tests/golden/golden_bench.json).

Modelled on the reference's tests/test_cli.py (:50-82, :105-143, :160-175).
"""

import json
from pathlib import Path

import pytest

import inputs

torch = pytest.importorskip("torch")
click_testing = pytest.importorskip("click.testing")
pytestmark = pytest.mark.gpu

from paper_2510_00554_b200 import bench as sbench
from paper_2510_00554_b200 import cli
from paper_2510_00554_b200.dataset import DatasetManifest
from paper_2510_00554_b200.model import TensorMap, save_model


def run(*args):
    return click_testing.CliRunner().invoke(cli.main, [str(a) for a in args])


@pytest.fixture()
def keyfile(tmp_path):
    assert run("keygen", tmp_path / "signer").exit_code == 0
    return tmp_path / "signer.key.pem"


@pytest.fixture()
def model_manifest(tmp_path):
    tensors = inputs.model_tensors(31, [100, 8192, 5000, 0, 20000, 70001])
    path = tmp_path / "model.json"
    save_model(TensorMap([(f"t{i}", t) for i, t in enumerate(tensors)]), path)
    return path


@pytest.fixture()
def dataset_manifest(tmp_path):
    samples = inputs.dataset_samples(seed=41, n=120, n_sources=3, declared=[2, 5, 9], min_len=0, max_len=500, id_base=10)
    shard, offs, lens, _ids, _src = inputs.pack_samples(samples)
    rows = [(sid, src, label, int(offs[i]), int(lens[i])) for i, (sid, src, label, _d) in enumerate(samples)]
    path = tmp_path / "data.json"
    DatasetManifest(rows, tmp_path / "data.bin").save(path, shard)
    return path


@pytest.mark.parametrize("flags", [
    [], ["--compression", "blake2b"], ["--compression", "sha3-256", "--block-size", "1024"],
    ["--construction", "lattice"], ["--strategy", "coalesced"], ["--strategy", "per-layer"],
    ["--construction", "lattice", "--strategy", "per-layer", "--ordered"],
])
def test_sign_then_verify_model(keyfile, model_manifest, flags):
    signed = run("sign-model", model_manifest, "--key", keyfile, "--json", *flags)
    assert signed.exit_code == 0, signed.output
    info = json.loads(signed.output)
    assert info["blocks"] > 0 and Path(info["bundle"]).exists()
    # the verifier takes its configuration from the bundle, not from flags
    checked = run("verify-model", model_manifest, info["bundle"])
    assert checked.exit_code == 0 and checked.output.strip() == "OK"


def test_model_digest_matches_the_oracle(keyfile, model_manifest, porc):
    signed = run("sign-model", model_manifest, "--key", keyfile, "--json")
    tensors = inputs.model_tensors(31, [100, 8192, 5000, 0, 20000, 70001])
    assert json.loads(signed.output)["digest"] == porc.inplace_merkle("sha256", tensors, 8192).hex()


def test_tampered_model_is_rejected(keyfile, model_manifest):
    signed = json.loads(run("sign-model", model_manifest, "--key", keyfile, "--json").output)
    data = model_manifest.with_suffix(".bin")
    raw = bytearray(data.read_bytes())
    raw[12345] ^= 0x01
    data.write_bytes(bytes(raw))
    r = run("verify-model", model_manifest, signed["bundle"])
    assert r.exit_code == 1 and r.output.strip() == "DIGEST_MISMATCH"


def test_per_layer_bundle_lists_one_digest_per_tensor(keyfile, model_manifest):
    signed = json.loads(run("sign-model", model_manifest, "--key", keyfile, "--strategy", "per-layer", "--json").output)
    shown = json.loads(run("inspect", signed["bundle"]).output)
    assert sorted(shown["predicate"]["layer_digests"]) == [f"t{i}" for i in range(6)]


def test_sign_then_verify_dataset(keyfile, dataset_manifest, tmp_path):
    for extra in ([], ["--cover-labels"]):
        out = tmp_path / ("b" + "".join(extra).strip("-"))
        signed = run("sign-dataset", dataset_manifest, "--key", keyfile, "--out-dir", out, *extra)
        assert signed.exit_code == 0, signed.output
        assert signed.output.count(" samples -> ") == 3
        checked = run("verify-dataset", dataset_manifest, "--bundles", out, "--batch-size", "7", "--shuffle-seed", "99")
        assert checked.exit_code == 0, checked.output
        assert [ln.split(": ")[1] for ln in checked.output.strip().splitlines()] == ["OK"] * 3


def test_corrupted_sample_fails_only_its_source(keyfile, dataset_manifest):
    assert run("sign-dataset", dataset_manifest, "--key", keyfile).exit_code == 0
    listing = DatasetManifest.load(dataset_manifest)
    victim = next(r for r in listing.samples if r[4] > 0)
    raw = bytearray(listing.data_path.read_bytes())
    raw[victim[3]] ^= 0xFF
    listing.data_path.write_bytes(bytes(raw))
    r = run("verify-dataset", dataset_manifest)
    assert r.exit_code == 1
    verdicts = dict(ln.split(": ") for ln in r.output.strip().splitlines())
    assert verdicts.pop(f"source {victim[1]}") == "DIGEST_MISMATCH"
    assert set(verdicts.values()) == {"OK"}


def test_strategy_table_digests_equal_the_reference():
    gold = json.loads((Path(__file__).parent / "golden" / "golden_bench.json").read_text())
    cells = sbench.run_bench(shapes=("vgg19", "resnet152"), scale=0.002, worker_counts=(1,), repeats=1,
                             compressions=("sha256", "blake2b", "sha3-256"))
    got = {(c.shape, c.construction, c.compression, c.strategy): c.digest for c in cells}
    want = {(c["shape"], c["construction"], c["compression"], c["strategy"]): c["digest"] for c in gold["cells"]}
    assert got == want
    assert all(c.verified for c in cells)
    assert all(c.device_ms is not None for c in cells if c.construction != "sequential")


def test_bench_command_json():
    r = run("bench", "--sizes", "vgg19", "--scale", "0.001", "--workers", "1", "--repeats", "1", "--json")
    assert r.exit_code == 0, r.output
    cells = json.loads(r.output)
    assert {c["construction"] for c in cells} == {"sequential", "merkle", "lattice"}
    assert all(c["verified"] for c in cells)
