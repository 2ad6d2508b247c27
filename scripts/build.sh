#!/bin/bash
# Build libappo_b200.so here (cross-compile for sm_100a); fails loudly.
cd "$(dirname "$0")/.." && python -c "
import runpy; runpy.run_path('paper_2006_11751_b200/_build.py')['build'](force=True)" && \
  python -c "import ctypes; ctypes.CDLL('paper_2006_11751_b200/libappo_b200.so')" && echo BUILD_OK
