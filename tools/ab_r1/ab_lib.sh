# Dev A/B: build an alternative libpgcn.so with one translation unit replaced or recompiled.
#   bash tools/ab_lib.sh <name> <source .cu> <replaced TU, e.g. kernels.cu> [extra nvcc flags...]
#   -> tools/ab/libpgcn_<name>.so ; use with PGCN_LIB=tools/ab/libpgcn_<name>.so python bench.py ...
set -e
N=$1; SRC=$2; TU=$3; shift 3
R=$(cd "$(dirname "$0")/.." && pwd)
O=$R/paper_2203_10428_b200/build
mkdir -p $R/tools/ab
NI=$(python -c "import nvidia.nccl as m,os;print(os.path.dirname(m.__file__) if getattr(m,'__file__',None) else list(m.__path__)[0])")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I$R/include \
  -I$R/paper_2203_10428_b200/csrc -DPGCN_WITH_NCCL=1 -I$NI/include "$@" -c $SRC -o $R/tools/ab/$N.o
OBJS=$(ls $O/*.o | grep -v "/$TU.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/ab/libpgcn_$N.so $OBJS $R/tools/ab/$N.o \
  -L$NI/lib -l:libnccl.so.2 -Xlinker -rpath=$NI/lib
echo built tools/ab/libpgcn_$N.so
