#!/bin/bash
# Host-side AddressSanitizer + UndefinedBehaviorSanitizer run of the planner (libaxe's host code: layouts,
# normaliser, joint refinement, kernel selection, TMA lowering, text/JSON, redistribution planning) and of
# the oracle, under the whole CPU test suite.  Device code is unaffected (no kernel runs on a CPU box).
#   bash tools/asan_host.sh [pytest args...]      (log: profiles/r02_asan_host.log)
set -e
cd "$(dirname "$0")/.."
OUT=/tmp/axe_asan
mkdir -p "$OUT"
SAN="-fsanitize=address,undefined -fno-omit-frame-pointer -fno-sanitize-recover=undefined"
XC="-Xcompiler=-fsanitize=address -Xcompiler=-fsanitize=undefined -Xcompiler=-fno-omit-frame-pointer -Xcompiler=-fno-sanitize-recover=undefined"
AXE_BUILD_OUT=$OUT/libaxe_asan.so AXE_EXTRA_NVCC="$XC" AXE_EXTRA_LINK="-Xcompiler=-fsanitize=address -Xcompiler=-fsanitize=undefined" \
  python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'paper_2601_19092_b200/build.py')
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b); print(b.build(force=True))"
gcc -O1 -g $SAN -std=c11 -fPIC -shared -pthread -o "$OUT/liboracle_asan.so" oracle/axe_oracle.c -lm
export LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)"
export ASAN_OPTIONS=detect_leaks=0,protect_shadow_gap=0,abort_on_error=1
export UBSAN_OPTIONS=print_stacktrace=1,halt_on_error=1
AXE_LIBAXE=$OUT/libaxe_asan.so AXE_ORACLE_LIB=$OUT/liboracle_asan.so python -m pytest tests -q -m "not gpu" -p no:cacheprovider "$@"
