#!/bin/bash
# Build A/B variants of the conv1 kernel: abtest/libappo_<name>.so for each
# "name:flags" argument (flags are -D defines for csrc/conv1.cu), all other
# objects shared with the in-tree build.  Run with scripts/ab_conv1_run.sh.
set -e
cd "$(dirname "$0")/.."
python -c "import sys; sys.path.insert(0,'paper_2006_11751_b200'); import _build; _build.build()"
mkdir -p abtest
B=paper_2006_11751_b200/build
OBJS=$(ls $B/*.o | grep -v conv1.cu.o)
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    --expt-relaxed-constexpr -Xcompiler -fPIC -Xcompiler -fvisibility=hidden $flags \
    -c paper_2006_11751_b200/csrc/conv1.cu -o /tmp/conv1_$name.o &
done
wait
for spec in "$@"; do
  name=${spec%%:*}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abtest/libappo_$name.so $OBJS /tmp/conv1_$name.o
  echo "built abtest/libappo_$name.so"
done
