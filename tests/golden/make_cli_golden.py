"""Regenerate tests/golden/cli/ from the reference CLI (needs /root/reference).

Runs ``python -m memsched.cli`` from the read-only reference tree for a fixed
list of command lines and stores stdout, stderr and the exit code of each, so
tests/test_cli.py can require byte-identical output from this package's CLI.

    python tests/golden/make_cli_golden.py
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = "/root/reference/pkg/src"

ALL = "liveness,offload,cache,recompute=cost-aware,convselect"
CASES = {
    "run_table_all": ["run", "--net", "alexnet", "--batch", "200", "--pool", "2GiB", "--features", ALL],
    "run_csv_all": ["run", "--net", "alexnet", "--batch", "200", "--pool", "2GiB", "--features", ALL,
                    "--report", "csv"],
    "run_json_all": ["run", "--net", "alexnet", "--batch", "200", "--pool", "2GiB", "--features", ALL,
                     "--report", "json"],
    "run_table_none": ["run", "--net", "alexnet", "--batch", "64", "--pool", "6GB"],
    "run_table_memory": ["run", "--net", "alexnet", "--batch", "128", "--pool", "1500MB", "--features",
                         "liveness,recompute=memory"],
    "run_csv_offload": ["run", "--net", "alexnet", "--batch", "200", "--pool", "1.5GiB", "--features",
                        "liveness,offload,cache"],
    "sweep_batch_table": ["sweep", "--net", "alexnet", "--pool", "2GiB", "--features", ALL, "--axis", "batch",
                          "--values", "32,64,128,200"],
    "sweep_pool_csv": ["sweep", "--net", "alexnet", "--batch", "200", "--features", ALL, "--axis", "pool-bytes",
                       "--values", "1GiB,1500MiB,2GiB", "--pool", "2GiB", "--report", "csv"],
    "sweep_batch_json": ["sweep", "--net", "alexnet", "--pool", "2GiB", "--axis", "batch", "--values", "16,32",
                         "--report", "json"],
    "gen_resnet": ["gen-resnet", "--blocks", "1,1,1,1", "--classes", "10"],
    "err_floor": ["run", "--net", "alexnet", "--batch", "200", "--pool", "100MiB"],
    "err_oom": ["run", "--net", "alexnet", "--batch", "200", "--pool", "1GiB"],
    "err_size": ["run", "--net", "alexnet", "--pool", "lots"],
    "err_net": ["run", "--net", "no_such_net", "--pool", "1GiB"],
    "err_features": ["run", "--net", "alexnet", "--pool", "2GiB", "--features", "liveness,teleport"],
    "err_blocks": ["gen-resnet", "--blocks", "1,2"],
}


def main() -> None:
    out = {}
    env = dict(os.environ, PYTHONPATH=REF)
    for name, argv in CASES.items():
        p = subprocess.run([sys.executable, "-m", "memsched.cli", *argv], capture_output=True, text=True, env=env,
                           cwd="/tmp")
        out[name] = {"argv": argv, "rc": p.returncode, "stdout": p.stdout, "stderr": p.stderr}
        print(name, p.returncode, len(p.stdout))
    (HERE / "cli" / "cli_golden.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
