#!/bin/bash
# Build a variant of libkpme_b200.so locally: one .cu recompiled with extra -D flags,
# linked with the default objects, into paper_2601_18838_b200/variants/libkpme_<tag>.so
# (git-ignored; it travels with gpurun). Select it at run time with KPME_LIB=<path>.
# Usage: scripts/build_variant.sh <tag> <unit: interp|sort2|...> "<flags>"
set -e
cd "$(dirname "$0")/.."
tag=$1; unit=$2; flags=$3
C=paper_2601_18838_b200/csrc
mkdir -p paper_2601_18838_b200/variants $C/build/var
NCCL_HOME=$(python3 -c "import nvidia, os; p = os.path.join(list(nvidia.__path__)[0], 'nccl'); print(p if os.path.exists(os.path.join(p, 'lib', 'libnccl.so.2')) else '')" 2>/dev/null)
NCCL_INC=""; NCCL_LINK="-lnccl"
if [ -n "$NCCL_HOME" ]; then NCCL_INC="-I$NCCL_HOME/include"; NCCL_LINK="-L$NCCL_HOME/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $NCCL_HOME/lib"; fi
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo $flags -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  -Iinclude --expt-relaxed-constexpr $NCCL_INC -Xptxas -v -c $C/$unit.cu -o $C/build/var/${unit}_$tag.o 2> $C/build/var/${unit}_$tag.ptxas.log || { grep -m5 error $C/build/var/${unit}_$tag.ptxas.log; echo "variant build FAILED"; exit 1; }
objs=""
for u in sort sort2 interp core dense dense_slab plan multi host; do
  if [ "$u" = "$unit" ]; then objs="$objs $C/build/var/${unit}_$tag.o"; else objs="$objs $C/build/$u.o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2601_18838_b200/variants/libkpme_$tag.so $objs -lcudart $NCCL_LINK
echo "built paper_2601_18838_b200/variants/libkpme_$tag.so"
