#!/bin/bash
# Build libgenred.so (and the oracle) from any working directory.
cd "$(dirname "$0")/.." && python -m paper_2004_11127_b200.build "$@" && python -c "import oracle; oracle.build()"
