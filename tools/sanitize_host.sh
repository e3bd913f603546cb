#!/bin/bash
# ASan + UBSan of the host code (SURVEY §4 "Sanitizers"): the oracle and the library's host
# C++ (encoder, split heuristic, container parse / write / combine, planner, CPU decoders) are
# rebuilt with -fsanitize=address,undefined and the CPU test suite runs against them.
# usage: tools/sanitize_host.sh [pytest args]   (no GPU needed)
cd "$(dirname "$0")/.." || exit 1
python -m paper_2306_12141_b200._build --sanitize > /dev/null || exit 1
ORACLE_SANITIZE=1 python -c "import oracle; oracle.build()" || exit 1
ASAN=$(gcc -print-file-name=libasan.so)
UBSAN=$(gcc -print-file-name=libubsan.so)
LD_PRELOAD="$ASAN:$UBSAN" ASAN_OPTIONS=detect_leaks=0:halt_on_error=1 UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1 \
  ORACLE_SANITIZE=1 RECOIL_LIB=$PWD/paper_2306_12141_b200/librecoil_san.so \
  python -m pytest tests -q -m "not gpu" -p no:cacheprovider "$@"
