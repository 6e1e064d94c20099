"""Regenerates tests/golden/cli/ref.out: the qforge CLI cases (tests/cli_cases.py)
through tools/qforge_cli.cpp built against the UNMODIFIED reference headers
(oracle/_ref/qforge_cli_ref; needs /root/reference)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import cli_cases  # noqa: E402

binary = os.path.join(ROOT, "oracle", "_ref", "qforge_cli_ref")
subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), binary], check=True)
text = cli_cases.transcript(binary, env=dict(os.environ, OMP_NUM_THREADS="4"))
with open(os.path.join(cli_cases.CLI_DIR, "ref.out"), "w") as f:
    f.write(text)
print("wrote tests/golden/cli/ref.out (%d cases)" % text.count("=== "))
