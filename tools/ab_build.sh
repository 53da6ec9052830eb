#!/bin/bash
# A/B build of the library with extra nvcc flags: tools/ab_build.sh NAME "-DMACRO=..."
# -> paper_2307_00124_b200/_ab/NAME/libbfpmg_b200.so (load it with BFPMG_LIB=...)
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=/tmp/bfp_ab_$name
rm -rf $tmp && mkdir -p $tmp/pkg $tmp/include
cp -r $root/paper_2307_00124_b200/csrc $root/paper_2307_00124_b200/Makefile $tmp/pkg/
cp $root/include/*.h $tmp/include/
make -s -j8 -C $tmp/pkg EXTRA="$*" > $tmp/build.log 2>&1 || { tail -20 $tmp/build.log; exit 1; }
mkdir -p $root/paper_2307_00124_b200/_ab/$name
cp $tmp/pkg/_lib/libbfpmg_b200.so $root/paper_2307_00124_b200/_ab/$name/
echo "built _ab/$name"
