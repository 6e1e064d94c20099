"""The qforge command line (`qforge run|bench` on the GPU
backend).  tools/qforge_cli.cpp is built against the facade + libqsb
(build/qforge) and, in this container, against the unmodified reference
headers (oracle/_ref/qforge_cli_ref -> tests/golden/cli/ref.out,
tools/make_cli_golden.py).  The same command lines must print identical
counts (same seeds -> same samples), identical bench rows up to the
checksum's last bits, and identical exit codes."""
import os

import pytest

import cli_cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "qforge")


def split(text):
    cases = {}
    for chunk in text.split("=== ")[1:]:
        head, _, body = chunk.partition("\n")
        cases[head] = body
    return cases


@pytest.mark.gpu
def test_cli_matches_reference_transcript():
    if not os.path.exists(BIN):
        pytest.fail("build/qforge missing: run `make -C paper_2212_14201_b200/csrc facadechecks` (build())")
    got = split(cli_cases.transcript(BIN))
    want = split(open(os.path.join(cli_cases.CLI_DIR, "ref.out")).read())
    assert list(got) == list(want)  # same cases, same exit codes
    for name, body in want.items():
        if name.startswith("bench"):
            g_rows = [r.split("\t") for r in got[name].splitlines()]
            w_rows = [r.split("\t") for r in body.splitlines()]
            assert g_rows[0] == w_rows[0] and len(g_rows) == len(w_rows)
            for g, w in zip(g_rows[1:], w_rows[1:]):
                assert g[:7] == w[:7], name
                assert abs(float(g[7]) - float(w[7])) <= 1e-12 * abs(float(w[7])), name
        else:
            assert got[name] == body, name
