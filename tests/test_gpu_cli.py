"""CLI parity: the reference's subcommands and --json documents
(/root/reference/pkg/src/neuralvol/cli.py:115-303 and schemas/{train,decode,render,bench,
metrics}.json: the required keys below are those schemas' `required` lists), exit codes, and the
repeatability contract of acceptance gate 9 (test_acceptance.py:439-473): repeating a train or
render command with the same seed reproduces the artefacts byte for byte."""
from __future__ import annotations

import json

import pytest

pytestmark = pytest.mark.gpu

TRAIN_KEYS = {"out", "history", "steps", "final_loss", "mean_ms_per_step", "model_params", "compression_ratio",
              "seed", "threads"}
DECODE_KEYS = {"out", "dims", "dtype", "model_params"}
RENDER_KEYS = {"out", "width", "height", "mode", "architecture", "macrocells", "frames", "ms", "fps",
               "field_evaluations", "majorant_violations", "seed", "threads"}
METRICS_KEYS = {"psnr_db", "mssim", "mse"}
BENCH_ENTRY_KEYS = {"architecture", "mode", "macrocells", "ms", "fps", "field_evaluations", "majorant_violations"}


def _run(capsys, *argv):
    from paper_2207_11620_b200.cli import main
    rc = main(list(argv))
    return rc, capsys.readouterr()


def test_cli_json_documents_and_gate9_repeatability(nv, tmp_path, capsys):
    models, hists = [], []
    for tag in ("a", "b"):
        out, hist = tmp_path / f"m_{tag}.vnr", tmp_path / f"h_{tag}.csv"
        rc, cap = _run(capsys, "train", "--synthetic", "gauss:16", "--steps", "30", "--batch", "1024", "--seed", "3",
                       "--out", str(out), "--history", str(hist), "--json")
        assert rc == 0, cap.err
        doc = json.loads(cap.out)
        assert set(doc) == TRAIN_KEYS and doc["steps"] == 30 and doc["final_loss"] >= 0
        models.append(out.read_bytes())
        hists.append([ln.rsplit(",", 1)[0] for ln in hist.read_text().splitlines()])
    assert models[0] == models[1] and hists[0] == hists[1]          # gate 9: train
    renders = []
    for mode, frames in (("raymarch", "1"), ("pathtrace", "2")):
        pair = []
        for tag in ("a", "b"):
            png = tmp_path / f"r_{mode}_{tag}.png"
            rc, cap = _run(capsys, "render", "--model", str(tmp_path / "m_a.vnr"), "--mode", mode, "--frames", frames,
                           "--size", "48x48", "--macrocells", "--seed", "9", "--out", str(png), "--json")
            assert rc == 0, cap.err
            doc = json.loads(cap.out)
            assert set(doc) == RENDER_KEYS and doc["field_evaluations"] > 0
            assert png.read_bytes()[:8] == b"\x89PNG\r\n\x1a\n"
            pair.append(png.read_bytes())
        renders.append(pair[0] == pair[1])
    assert all(renders)                                              # gate 9: render
    side = tmp_path / "dec.json"
    rc, cap = _run(capsys, "decode", "--model", str(tmp_path / "m_a.vnr"), "--out", str(side), "--json")
    assert rc == 0, cap.err
    doc = json.loads(cap.out)
    assert DECODE_KEYS <= set(doc) <= DECODE_KEYS | {"value_range"} and doc["dims"] == [16, 16, 16]
    raw = side.with_suffix(".raw")
    meta = json.loads(side.read_text())
    rc, cap = _run(capsys, "metrics", "--a", str(raw), "--b", str(raw), "--meta", str(side), "--json")
    assert rc == 0, cap.err
    doc = json.loads(cap.out)
    assert set(doc) == METRICS_KEYS and doc["psnr_db"] == 99.0 and meta["dims"] == [16, 16, 16]
    rc, cap = _run(capsys, "bench", "--synthetic", "gauss:16", "--size", "16x16", "--json")
    assert rc == 0, cap.err
    rep = json.loads(cap.out)
    assert len(rep["entries"]) == 12 and all(set(e) == BENCH_ENTRY_KEYS for e in rep["entries"])


def test_cli_exit_codes(nv, tmp_path, capsys):
    rc, _ = _run(capsys, "train", "--synthetic", "nosuchfield:8", "--out", str(tmp_path / "x.vnr"))
    assert rc == 1                                                   # usage problem
    rc, _ = _run(capsys, "decode", "--model", str(tmp_path / "missing.vnr"), "--out", str(tmp_path / "x.raw"))
    assert rc == 2                                                   # runtime failure
