"""Command lines for the qforge CLI parity check (tests/test_cli_gpu.py,
tools/make_cli_golden.py).  Paths are relative to tests/golden/cli."""
import os
import subprocess

CASES = [
    ("ghz5", ["run", "ghz5.oir", "--shots", "1000", "--seed", "11"]),
    ("ghz5_default_shots", ["run", "ghz5.oir"]),
    ("midcircuit", ["run", "midcircuit.oir", "--shots", "600", "--seed", "5"]),
    ("rot10", ["run", "rot10.oir", "--shots", "4000", "--seed", "2"]),
    ("rot10_fusion", ["run", "rot10.oir", "--shots", "4000", "--seed", "2", "--opt", "fusion"]),
    ("rot10_workers", ["run", "rot10.oir", "--shots=3000", "--seed=77", "--workers", "3"]),
    ("noisy", ["run", "noisy.oir", "--backend", "noisy", "--noise", "noise.txt", "--shots", "3000", "--seed", "9"]),
    ("bench", ["bench", "--qubits", "8,11", "--layers", "3", "--seed", "4", "--opt", "none"]),
    ("bench_fusion", ["bench", "--qubits", "10", "--layers", "2", "--seed", "1", "--opt", "fusion"]),
    ("err_missing_file", ["run", "does_not_exist.oir"]),
    ("err_parse", ["run", "broken.oir"]),
    ("err_zero_shots", ["run", "ghz5.oir", "--shots", "0"]),
    ("err_unknown_backend", ["run", "ghz5.oir", "--backend", "tensor"]),
    ("err_noisy_without_config", ["run", "ghz5.oir", "--backend", "noisy"]),
    ("err_bad_opt", ["run", "ghz5.oir", "--opt", "magic"]),
    ("err_unknown_option", ["run", "ghz5.oir", "--frobnicate", "1"]),
    ("err_no_subcommand", []),
]

CLI_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


def transcript(binary, env=None):
    """'=== name rc=<exit code>' + stdout per case; bench timing columns masked."""
    out = []
    for name, args in CASES:
        r = subprocess.run([binary, *args], cwd=CLI_DIR, capture_output=True, text=True, timeout=600, env=env)
        text = r.stdout
        if args and args[0] == "bench" and r.returncode == 0:
            rows = []
            for i, line in enumerate(text.splitlines()):
                f = line.split("\t")
                if i > 0:
                    f[2] = f[3] = f[4] = "t"
                rows.append("\t".join(f))
            text = "\n".join(rows) + "\n"
        out.append("=== %s rc=%d\n%s" % (name, r.returncode, text))
    return "".join(out)
