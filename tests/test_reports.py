"""Report formats of the reference CLI against fixtures the
reference itself wrote (tests/golden/make_golden.py::report_fixtures):

* bench CSV (cli.py:71-78, 125-178): ``# config:`` line, header, config hash
  and every deterministic column (masks, tile counts, FLOPs) byte-equal;
* mask PGM (attention.py:133-138) byte-equal, selection trace JSON
  (selection.py:234-249) equal (scores to fp64 rounding) -- from the GPU
  selection through ``paper_2602_04789_b200.tools.mask_dump``.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2602_04789_b200 import reports, tools
from paper_2602_04789_b200.layout import BlockMask

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BENCH_ARGS = dict(seq=512, dim=64, block=64, kv_block=None, densities=[0.5, 0.25], repeats=3,
                  seed=5)


def _golden_bench():
    with open(os.path.join(GOLD, "report_bench.csv"), encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    return lines[0], lines[1], [ln.split(",") for ln in lines[2:]]


def test_bench_config_hash_and_static_columns():
    cfg_line, header, rows = _golden_bench()
    densities, config = tools.bench_config(BENCH_ARGS["seq"], BENCH_ARGS["dim"],
                                           BENCH_ARGS["block"], None, BENCH_ARGS["densities"],
                                           BENCH_ARGS["repeats"], BENCH_ARGS["seed"], 1)
    assert cfg_line == "# config: " + json.dumps(reports.plain(config), sort_keys=True)
    assert header == ",".join(tools.BENCH_HEADER)
    chash = reports.config_hash(config)
    n = BENCH_ARGS["seq"] // BENCH_ARGS["block"]
    for density, row in zip(densities, rows):
        m = tools.bench_mask(n, n, density, BENCH_ARGS["seed"])
        act = m.popcount()
        ours = [chash, 512, 64, 64, 64, repr(density), repr(1.0 - act / (n * n)), act, n * n,
                act * 64 * 64 * 64 * 2]
        assert [str(x) for x in ours] == row


def test_write_csv_format(tmp_path):
    cfg_line, header, rows = _golden_bench()
    config = json.loads(cfg_line[len("# config: "):])
    out = tmp_path / "b.csv"
    reports.write_csv(str(out), header.split(","), rows, config)
    raw = out.read_bytes()
    assert raw.startswith((cfg_line + "\r\n" + header + "\r\n").encode())
    assert raw.count(b"\r\n") == 2 + len(rows)


def test_pgm_writer_roundtrip(tmp_path):
    for mode in ("global", "per-frame"):
        gold = open(os.path.join(GOLD, f"report_mask_{mode}.pgm"), "rb").read()
        head, body = gold.split(b"\n255\n", 1)
        n_k, n_q = (int(x) for x in head.split(b"\n")[1].split())
        bits = np.frombuffer(body, np.uint8).reshape(n_q, n_k) == 255
        out = tmp_path / "m.pgm"
        BlockMask(bits).to_pgm(str(out))
        assert out.read_bytes() == gold


@pytest.mark.gpu
@pytest.mark.parametrize("mode,sparsity,chunk", [("global", 0.6, 7), ("per-frame", 0.7, 5)])
def test_mask_dump_matches_reference(tmp_path, mode, sparsity, chunk):
    pgm, trace = tmp_path / "m.pgm", tmp_path / "t.json"
    tools.mask_dump(frames=3, tokens=128, block=64, dim=32, chunks=7, chunk=chunk,
                    sparsity=sparsity, topk=3, mode=mode, seed=11, out=str(pgm),
                    trace=str(trace))
    assert pgm.read_bytes() == open(os.path.join(GOLD, f"report_mask_{mode}.pgm"), "rb").read()
    got = json.loads(trace.read_text())
    ref = json.load(open(os.path.join(GOLD, f"report_trace_{mode}.json")))
    assert got["config"] == ref["config"]
    assert len(got["rows"]) == len(ref["rows"])
    for a, b in zip(got["rows"], ref["rows"]):
        for key in ("query_block", "frames", "blocks", "budget_used"):
            assert a[key] == b[key], key
        for key in ("block_scores", "frame_scores"):
            np.testing.assert_allclose(a[key], b[key], rtol=1e-12, atol=1e-15)
    # canonical JSON: parse + redump is byte-identical
    assert reports.canonical_json(got) == trace.read_text()


@pytest.mark.gpu
def test_bench_sweep_csv_on_gpu(tmp_path):
    out = tmp_path / "bench.csv"
    tools.bench_sweep(out=str(out), threads=1, **BENCH_ARGS)
    cfg_line, header, rows = _golden_bench()
    with open(out, encoding="utf-8", newline="") as fh:
        lines = fh.read().split("\r\n")
    assert lines[0] == cfg_line and lines[1] == header
    body = [ln.split(",") for ln in lines[2:] if ln]
    assert [r[:10] for r in body] == rows
    for r in body:
        assert float(r[10]) > 0 and float(r[11]) > 0 and float(r[12]) > 0
        assert np.isfinite(float(r[13]))
    assert float(body[0][13]) < 1e-2  # density 1.0: the sparse path computes dense attention
