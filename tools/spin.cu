// spin.cu -- a kernel that spins for a given time (tools/coresid_probe.py: does a small
// kernel on another stream run beside the walk?).  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -o tools/spin.so tools/spin.cu
#include <cuda_runtime.h>
__global__ void spin_k(long long ns, int pad)
{
    extern __shared__ unsigned char sm[];
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    long long t = t0;
    while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (pad < 0) sm[threadIdx.x] = 1;
}
extern "C" int spin_launch(void* st, long long ns, int ctas, int threads, int smem)
{
    if (smem > 48000) cudaFuncSetAttribute(spin_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    spin_k<<<ctas, threads, smem, (cudaStream_t)st>>>(ns, 0);
    return (int)cudaGetLastError();
}
