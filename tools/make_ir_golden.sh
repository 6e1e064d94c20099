#!/bin/sh
# Regenerates tests/golden/ir_corpus.ref.out: the parse_ir / emit_ir transcript
# of tests/golden/ir_corpus.txt through the UNMODIFIED reference headers
# (oracle/_ref/ir_check_ref, built by oracle/Makefile from /root/reference).
set -e
cd "$(dirname "$0")/.."
make -s -C oracle "$(pwd)/oracle/_ref/ir_check_ref"
oracle/_ref/ir_check_ref tests/golden/ir_corpus.txt > tests/golden/ir_corpus.ref.out
echo "wrote tests/golden/ir_corpus.ref.out ($(grep -c '^===' tests/golden/ir_corpus.ref.out) cases)"
