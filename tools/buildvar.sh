# build a variant of libbnreg.so with extra -D flags: tools/buildvar.sh NAME [-DX=Y ...]
name=$1; shift
S=paper_1901_07643_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o tmpvar/lib$name.so $S/bnreg_api.cu $S/bnreg_kernels.cu $S/walk_kernel.cu $S/seed_kernel.cu 2>&1 | grep -i "error" || true
