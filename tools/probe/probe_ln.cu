// ptxas probe: instantiate one LayerNorm warp-tier kernel and read the
// register / spill report in seconds instead of building the whole library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v \
//     -DPT=__nv_bfloat16 -DPVB=16 -DPG=32 -DPNV=4 -DPMINB=2 -DPPF=1 -DPEX=1 \
//     -c tools/probe/probe_ln.cu -o /tmp/probe.o
#include "../../paper_2010_05680_b200/csrc/layernorm_kernels.cuh"

namespace tt {
bool pdl_enabled() { return true; }
cudaError_t smem_optin(const void*, size_t) { return cudaSuccess; }
template __global__ void ln_warp_kernel<PT, PVB, PG, PNV, 256, PMINB, (bool)PPF, (bool)PEX>(
    PT*, const PT*, const PT*, const PT*, const PT*, const PT*, uint32_t, int, float);
}  // namespace tt
