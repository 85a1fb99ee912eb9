"""The ``memsched`` CLI (paper_1801_04380_b200/cli.py + report.py) against text
the reference CLI printed for the same command lines
(tests/golden/make_cli_golden.py -> tests/golden/cli/cli_golden.json):
stdout byte-identical for table / CSV / JSON runs and sweeps and gen-resnet,
same exit codes (2 rejected, 3 does not fit) and stderr messages.  The one
intended difference: the list of bundled fixtures in the unknown-network
message (this package bundles alexnet and alex32)."""

from __future__ import annotations

import json
import re
from pathlib import Path

import pytest

GOLDEN = json.loads((Path(__file__).parent / "golden" / "cli" / "cli_golden.json").read_text())


def _bundled_free(text: str) -> str:
    return re.sub(r"\(bundled: [^)]*\)", "(bundled: ...)", text)


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_cli_matches_reference(name, capsys):
    from paper_1801_04380_b200 import cli
    case = GOLDEN[name]
    rc = cli.main(case["argv"])
    out, err = capsys.readouterr()
    assert rc == case["rc"]
    assert out == case["stdout"]
    assert _bundled_free(err) == _bundled_free(case["stderr"])


def test_report_files_and_config(tmp_path, capsys):
    """--out writes the report (no figure with --no-plot); an INI file supplies
    defaults that flags override; a bad [run] key is a ConfigError (exit 2)."""
    from paper_1801_04380_b200 import cli
    ini = tmp_path / "run.ini"
    ini.write_text("[run]\nnet = alexnet\nbatch = 200\npool = 2GiB\n"
                   "features = liveness,offload,cache,recompute=cost-aware,convselect\nreport = csv\n")
    out = tmp_path / "sub" / "r.csv"
    assert cli.main(["run", "--config", str(ini), "--out", str(out), "--no-plot"]) == 0
    assert out.read_text() == GOLDEN["run_csv_all"]["stdout"]
    assert "report written to" in capsys.readouterr().err
    assert cli.main(["run", "--config", str(ini), "--report", "table"]) == 0
    assert capsys.readouterr().out == GOLDEN["run_table_all"]["stdout"]
    bad = tmp_path / "bad.ini"
    bad.write_text("[run]\nnets = alexnet\n")
    assert cli.main(["run", "--config", str(bad)]) == 2
    assert "unknown [run] option 'nets'" in capsys.readouterr().err


def test_measured_columns_render(capsys):
    """The --execute additions render in all three formats without touching the
    reference part of the output (rendering only; execution is a GPU test)."""
    from paper_1801_04380_b200 import report as rep
    from paper_1801_04380_b200.cli import resolve_network
    from paper_1801_04380_b200 import SimConfig, CostConfig, parse_features, run_simulation
    net = resolve_network("alexnet")
    cfg = SimConfig(pool_bytes=2 << 30, features=parse_features("liveness,offload,cache,recompute=cost-aware,"
                                                                 "convselect"), cost=CostConfig(batch=200))
    r = run_simulation(net, cfg)
    m = rep.Measured(device="B200", steps=10, ms_per_step=12.5, images_per_s=16000.0, kernels_per_step=120,
                     d2h_bytes_per_step=0, h2d_bytes_per_step=0, arena_bytes=r.pool_high_water_bytes,
                     final_loss=6.9)
    table = rep.render(r, "table", m)
    assert table.replace(table.splitlines()[[i for i, l in enumerate(table.splitlines())
                                             if l.startswith("measured on")][0]] + "\n", "") == \
        GOLDEN["run_table_all"]["stdout"]
    csv = rep.render(r, "csv", m)
    assert "# measured_images_per_s=16000" in csv
    assert "\n".join(l for l in csv.splitlines() if not l.startswith("# measured_")) + "\n" == \
        GOLDEN["run_csv_all"]["stdout"]
    doc = json.loads(rep.render(r, "json", m))
    assert doc.pop("measured")["ms_per_step"] == 12.5
    assert doc == json.loads(GOLDEN["run_json_all"]["stdout"])


@pytest.mark.gpu
def test_cli_execute_on_gpu(cuda, capsys):
    """``memsched run --execute`` plans, runs the schedule on the B200 and adds
    the measured object; the plan part equals the non-executing run."""
    from paper_1801_04380_b200 import cli
    argv = ["run", "--net", "alex32", "--batch", "16", "--pool", "1GiB", "--features",
            "liveness,offload,cache,recompute=cost-aware,convselect", "--report", "json"]
    assert cli.main(argv) == 0
    plain = json.loads(capsys.readouterr().out)
    assert cli.main(argv + ["--execute", "--iters", "3"]) == 0
    doc = json.loads(capsys.readouterr().out)
    m = doc.pop("measured")
    assert doc == plain
    assert m["steps"] == 3 and m["images_per_s"] > 0 and m["kernels_per_step"] > 0
    # the arena is the whole KiB-rounded pool; the blocks kernels wrote in one
    # iteration (sentinel scan on the device) cover at least the planner's
    # peak residency
    assert m["arena_bytes"] == 1 << 30
    assert plain["summary"]["peak_bytes"] <= m["arena_written_bytes"] <= m["arena_bytes"]
    assert m["device_bytes"] > m["arena_bytes"]
    assert cli.main(["sweep", "--net", "alex32", "--pool", "1GiB", "--axis", "batch", "--values", "8,16",
                     "--execute", "--iters", "2", "--report", "csv"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0].endswith("measured_ms_per_step,measured_images_per_s") and len(lines) == 3
