"""Program text format (`.oir`): the facade's parse_ir /
emit_ir (paper_2212_14201_b200/include/qforge/ir.hpp) against the reference's
(ir.hpp:135-140, 319-707).

tests/ir_check.cpp is compiled against both header sets and prints a
transcript per case (the emitted text and a round-trip check, or the
ParseError kind / line / column / message).  The reference transcript of
tests/golden/ir_corpus.txt is committed (tools/make_ir_golden.sh); when the
reference is present it is also rebuilt and compared live, together with the
reference's own data/*.oir files.  CPU only (no device calls)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CORPUS = os.path.join(ROOT, "tests", "golden", "ir_corpus.txt")
GOLDEN = os.path.join(ROOT, "tests", "golden", "ir_corpus.ref.out")
OURS = os.path.join(ROOT, "build", "droptest", "ir_check")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "ir_check_ref")
REF_DATA = "/root/reference/proj/data"


@pytest.fixture(scope="module")
def ours():
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2212_14201_b200", "csrc"), OURS],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail("building the facade ir_check failed:\n" + r.stdout + r.stderr)
    return OURS


def run(binary, *args):
    return subprocess.run([binary, *args], capture_output=True, text=True, check=True, timeout=120).stdout


def test_corpus_matches_reference_golden(ours):
    got = run(ours, CORPUS)
    want = open(GOLDEN).read()
    assert got.count("=== ") == want.count("=== ") > 70
    for g, w in zip(got.split("=== ")[1:], want.split("=== ")[1:]):
        assert g == w, "case %s differs:\n--- ours\n%s--- reference\n%s" % (g.splitlines()[0], g, w)
    assert got == want


def test_corpus_round_trips(ours):
    got = run(ours, CORPUS)
    ok = got.count("\nOK ")
    assert ok >= 10 and got.count("roundtrip ok") == ok and "MISMATCH" not in got


@pytest.mark.skipif(not os.path.isdir(REF_DATA), reason="reference tree not present")
def test_live_reference_build_and_data_files(ours):
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), REF_BIN], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("reference ir_check did not build: " + r.stderr[-300:])
    assert run(REF_BIN, CORPUS) == run(ours, CORPUS)
    files = sorted(os.path.join(REF_DATA, f) for f in os.listdir(REF_DATA) if f.endswith(".oir"))
    assert files
    assert run(REF_BIN, "--files", *files) == run(ours, "--files", *files)
