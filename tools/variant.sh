#!/bin/bash
# Build a diagnostics variant of libdtq_b200.so with extra nvcc flags into
# variants/<name>/ (git-ignored; travels to the GPU box).  Select it at run
# time with DTQ_B200_LIB=variants/<name>/libdtq_b200.so.
# usage: tools/variant.sh <name> '<nvcc flags>'
set -e
cd "$(dirname "$0")/.."
d=variants/$1
mkdir -p "$d"
make -s -C paper_2406_02540_b200 -j8 >/dev/null
objs=""
for f in paper_2406_02540_b200/csrc/*.cu; do
  b=$(basename "$f" .cu)
  grep -q "^SRC.*$b.cu\|csrc/$b.cu" paper_2406_02540_b200/Makefile || continue
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -O3 --expt-relaxed-constexpr -Iinclude $2 -c "$f" -o "$d/$b.o" &
  objs="$objs $d/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$d/libdtq_b200.so" $objs -lcudart
rm -f $d/*.o
echo "built $d/libdtq_b200.so"
