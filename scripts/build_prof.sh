#!/bin/bash
# the cycle-counter variant of the library (KNNG_PROFILE=1 at run time prints the K1 breakdown)
cd "$(dirname "$0")/.." && KNNG_BUILD_OUT=$PWD/paper_1602_06819_b200/libknng_prof.so KNNG_BUILD_PROFILE=1 \
  python -c "from paper_1602_06819_b200 import build as B; B.build(force=True)"
