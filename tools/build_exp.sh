# build an experiment variant of libigalr into exp/<tag>/ : build_exp.sh <tag> <extra nvcc flags...>
tag=$1; shift
IGALR_BUILD_DIR=$PWD/exp/$tag IGALR_LIB_OUT=$PWD/exp/libigalr_$tag.so IGALR_NVCC_EXTRA="$*" python -c "
import importlib.util,sys
spec=importlib.util.spec_from_file_location('b','paper_1811_06797_b200/_build.py'); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build()" 2>&1 | grep -i "error\|spill" | cut -c1-160
ls -la exp/libigalr_$tag.so
