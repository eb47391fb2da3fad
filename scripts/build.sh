#!/bin/bash
# build the CUDA library; print the tail of the log and fail loudly on error
cd "$(dirname "$0")/.." && python -m paper_2001_08289_b200.build_ext > /tmp/fftc_build.log 2>&1 || { grep -m5 -B2 -A8 "error" /tmp/fftc_build.log | head -60; echo BUILD FAILED; exit 1; }
echo build ok
