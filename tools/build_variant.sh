#!/bin/bash
# Build an A/B variant of the library into ab/<name>.so: every object from the regular build except
# <source>.cu, recompiled with the given -D flags.  usage: tools/build_variant.sh name source.cu -DFOO=1 ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; src=$2; shift 2
C=$ROOT/paper_2402_19147_b200/csrc
mkdir -p $ROOT/ab /tmp/abobj
python -m paper_2402_19147_b200.build > /dev/null
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -cudart static"
$NV $ARCH $FL "$@" -c $C/$src -o /tmp/abobj/${src%.cu}.o
objs=""
for o in $C/build/*.o; do b=$(basename $o); if [ "$b" = "${src%.cu}.o" ]; then objs="$objs /tmp/abobj/$b"; else objs="$objs $o"; fi; done
$NV $ARCH -shared -cudart static -o $ROOT/ab/$name.so $objs
echo "built ab/$name.so"
