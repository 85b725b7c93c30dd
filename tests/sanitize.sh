#!/usr/bin/env bash
# Run the tiny-config smoke (BASELINE configs[0]: 4 virtual EP ranks on one GPU,
# every kernel of the path) under ONE compute-sanitizer tool.
#   bash tests/sanitize.sh memcheck|racecheck|synccheck|initcheck
# One tool per invocation (B200_PROFILING.md: never several tools in one call).
set -euo pipefail
tool="${1:-memcheck}"
cd "$(dirname "$0")/.."
python -m paper_2502_06643_b200.build
exec compute-sanitizer --tool "$tool" --error-exitcode 99 --target-processes all python __graft_entry__.py
