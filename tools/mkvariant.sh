#!/bin/bash
# Build an experiment variant of libigalr.so: tools/mkvariant.sh <tag> "<extra nvcc defines>" [p3|p4|p3p4]
# Recompiles the canonical-kernel units with the defines, links them with the product's other objects and
# lays out exp/<tag>/ as an importable package root (tools/ab_time.py: IGALR_PKG_ROOT=exp/<tag>).
set -e
tag=$1; defs=$2; units=${3:-p3}
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/exp/$tag; bdir=$root/build/exp_$tag
mkdir -p $out/paper_1811_06797_b200 $bdir
cp $root/paper_1811_06797_b200/__init__.py $root/paper_1811_06797_b200/workloads.py $out/paper_1811_06797_b200/
rm -rf $out/synth && cp -r $root/synth $out/synth
objs=""
for s in abi factors apply_unfused apply_fused apply_fused2 canon_p3 canon_p4 kkt minres prec weights tt; do
  o=$root/build/igalr/$s.cu.o
  if [[ "$units" == *p3* && $s == canon_p3 ]] || [[ "$units" == *p4* && $s == canon_p4 ]]; then
    o=$bdir/$s.cu.o
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr -Xptxas -warn-spills $defs -I$root/include -I$root/paper_1811_06797_b200/csrc \
      -c $root/paper_1811_06797_b200/csrc/$s.cu -o $o 2>&1 | grep -i "spill.*ELb1ELb1ELb0ELb0\|error" || true &
  fi
  objs="$objs $o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/paper_1811_06797_b200/libigalr.so $objs -cudart=static
echo built $out
