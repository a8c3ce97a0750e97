# build a variant of libbnreg.so with extra -D flags: tools/buildvar.sh NAME [-DX=Y ...]
name=$1; shift
S=paper_1901_07643_b200/csrc
SRCS=$(python -c "import sys; sys.path.insert(0, 'paper_1901_07643_b200'); import build; print(' '.join('$S/' + s for s in build.SOURCES))")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o tmpvar/lib$name.so $SRCS 2>&1 | grep -i "error" || true
