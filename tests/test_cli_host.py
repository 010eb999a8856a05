"""CLI behaviour that needs no GPU: key files, usage/config errors, malformed bundles, exit codes.

Modelled on the reference's tests/test_cli.py (:44-48, :84-103, :145-158, :177-184); the hashing
commands proper are exercised on the B200 in tests/test_gpu_cli.py.
"""

import json

import pytest

click_testing = pytest.importorskip("click.testing")

from paper_2510_00554_b200 import attestation as att
from paper_2510_00554_b200 import bench as sbench
from paper_2510_00554_b200 import cli
from paper_2510_00554_b200.model import TensorMap, save_model


def run(*args):
    return click_testing.CliRunner().invoke(cli.main, [str(a) for a in args])


@pytest.fixture()
def keyfile(tmp_path):
    r = run("keygen", tmp_path / "signer")
    assert r.exit_code == 0, r.output
    return tmp_path / "signer.key.pem"


@pytest.fixture()
def manifest(tmp_path):
    path = tmp_path / "m.json"
    save_model(TensorMap([("a", b"x" * 100), ("b", b"y" * 9000)]), path)
    return path


def test_command_set_matches_reference():
    assert sorted(cli.main.commands) == ["bench", "inspect", "keygen", "sign-dataset", "sign-model",
                                         "verify-dataset", "verify-model"]
    opts = {p.name for p in cli.main.commands["sign-model"].params}
    assert opts == {"manifest", "key_path", "out_path", "construction", "compression", "strategy", "block_size",
                    "ordered", "workers", "as_json"}


def test_keygen_writes_both_files_and_refuses_overwrite(tmp_path):
    assert run("keygen", tmp_path / "k").exit_code == 0
    assert (tmp_path / "k.key.pem").exists() and (tmp_path / "k.pub.pem").exists()
    again = run("keygen", tmp_path / "k")
    assert again.exit_code == 2
    assert run("keygen", tmp_path / "k", "--force").exit_code == 0


def test_unknown_strategy_is_a_usage_error(keyfile, manifest):
    assert run("sign-model", manifest, "--key", keyfile, "--strategy", "zigzag").exit_code == 2


def test_config_errors_exit_2_before_any_hashing(keyfile, manifest):
    # lattice is fixed to blake2b; block size must be a power of two >= 64; ordered needs lattice per-layer
    assert run("sign-model", manifest, "--key", keyfile, "--construction", "lattice",
               "--compression", "sha256").exit_code == 2
    assert run("sign-model", manifest, "--key", keyfile, "--block-size", "1000").exit_code == 2
    assert run("sign-model", manifest, "--key", keyfile, "--ordered").exit_code == 2


def test_verify_model_with_truncated_bundle_is_malformed(manifest, tmp_path):
    bad = tmp_path / "broken.bundle.json"
    bad.write_text('{"payloadType": "application/vnd.in-toto+json", "payl')
    r = run("verify-model", manifest, bad)
    assert r.exit_code == 1
    assert att.Verdict.MALFORMED.value in r.output


def test_verify_dataset_missing_bundles_names_every_source(tmp_path):
    doc = {"samples": [{"sample_id": 1, "source_id": 3, "label": "", "offset": 0, "length": 4},
                       {"sample_id": 2, "source_id": 8, "label": "", "offset": 4, "length": 4}],
           "data": "d.bin", "expected_digests": {}}
    (tmp_path / "d.bin").write_bytes(b"abcdefgh")
    (tmp_path / "d.json").write_text(json.dumps(doc))
    r = run("verify-dataset", tmp_path / "d.json")
    assert r.exit_code == 1
    assert "source 3: missing or unreadable bundle" in r.output
    assert "source 8: missing or unreadable bundle" in r.output


def test_verify_empty_dataset_warns_and_succeeds(tmp_path):
    (tmp_path / "e.bin").write_bytes(b"")
    (tmp_path / "e.json").write_text(json.dumps({"samples": [], "data": "e.bin"}))
    r = run("verify-dataset", tmp_path / "e.json")
    assert r.exit_code == 0
    assert "nothing to verify" in r.output


def test_bad_dataset_manifest_exits_2(tmp_path, keyfile):
    (tmp_path / "bad.json").write_text("{not json")
    assert run("sign-dataset", tmp_path / "bad.json", "--key", keyfile).exit_code == 2


def test_inspect_prints_the_statement(tmp_path):
    key = att.KeyPair.generate()
    stmt = att.Statement([att.Subject("m.json", {"sha256": "ab" * 32})], att.MODEL_PREDICATE_TYPE,
                         {"construction": "merkle"})
    path = tmp_path / "b.bundle.json"
    att.sign_bundle(stmt, key).save(path)
    r = run("inspect", path)
    assert r.exit_code == 0
    doc = json.loads(r.output)
    assert doc["subject"][0]["name"] == "m.json"
    assert doc["predicate"] == {"construction": "merkle"}


def test_bench_bad_worker_list_exits_2():
    assert run("bench", "--workers", "1,x").exit_code == 2


def test_synthetic_models_are_the_reference_bytes():
    """bench.synthetic_model reproduces the reference's seeded recipe (fingerprints from the reference)."""
    import hashlib
    from pathlib import Path

    gold = json.loads((Path(__file__).parent / "golden" / "golden_bench.json").read_text())
    for m in gold["models"]:
        got = sbench.synthetic_model(m["shape"], m["scale"], m["seed"])
        assert len(got.entries) == m["layers"] and got.total_bytes == m["total_bytes"]
        assert hashlib.sha256(b"".join(b for _, b in got.entries)).hexdigest() == m["sha256_of_bytes"]
        assert got.names()[0] == "layer_0000"


def test_format_table_has_one_row_per_cell():
    cells = [sbench.BenchCell("vgg19", "merkle", "sha256", "in-place", 1, 1.5, 3.0, "00", True, 0.25),
             sbench.BenchCell("vgg19", "sequential", "sha256", "baseline", 1, 4.5, 1.0, "11", False)]
    lines = sbench.format_table(cells).splitlines()
    assert len(lines) == 4 and lines[0].split()[:4] == ["shape", "construction", "compression", "strategy"]
    assert lines[2].split()[-1] == "y" and lines[3].split()[-1] == "N"
