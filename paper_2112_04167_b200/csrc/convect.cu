// convect.cu -- instantiations of the LLF convection kernel (see convect.cuh).
#include "dev_common.cuh"
namespace dg {
DG_DEFINE_CONV_TABLES(upload_tables_convect)
}
#include "convect.cuh"
namespace dg {
cudaError_t launch_convect_k(const ConvParams &a, cudaStream_t st)
{
    return a.g.dim == 3 ? ConvDispatch<3>::run(a, st) : ConvDispatch<2>::run(a, st);
}
}  // namespace dg
