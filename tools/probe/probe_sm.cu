// ptxas probe: instantiate one softmax warp-tier kernel (see probe_ln.cu).
//   -DPT=__half -DPVB=32 -DPG=16 -DPNV=1 -DPMINB=6 -DPAL=0
#include "../../paper_2010_05680_b200/csrc/softmax_row.cuh"
#include "../../paper_2010_05680_b200/csrc/softmax_kernels.cuh"

namespace tt {
bool pdl_enabled() { return true; }
cudaError_t smem_optin(const void*, size_t) { return cudaSuccess; }
template __global__ void softmax_warp_kernel<PT, PVB, PG, PNV, 256, PMINB, (bool)PAL, false, false>(
    PT*, const int32_t*, FastDivU32, uint32_t, int, float, int);
}  // namespace tt
