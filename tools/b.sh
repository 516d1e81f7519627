#!/bin/bash
# build libamgf.so; exit non-zero (and print the first errors) on failure
cd "$(dirname "$0")/.." && python -c "
import sys; sys.path.insert(0,'.')
from paper_2505_18576_b200 import build; build.build()" > /tmp/build.log 2>&1 || { grep -iE "error" -A3 /tmp/build.log | head -20; exit 1; }
