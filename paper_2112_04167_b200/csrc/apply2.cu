// apply2.cu -- 2-D instantiations of the SIP apply / diagonal kernels (see apply.cuh).
#include "dev_common.cuh"
namespace dg {
DG_DEFINE_CONST_TABLES(upload_tables_apply2)
}
#include "apply.cuh"
namespace dg {
cudaError_t launch_apply2(const ApplyParams &a, bool varnu, int mode, int *grid, int smem, cudaStream_t st)
{
    return ApplyDispatch<2>::apply(a, varnu, mode, grid, smem, st);
}
cudaError_t launch_diag2(const Geom &g, double lam, const double *nu, double nuc, const Halo &h, double *d,
                         cudaStream_t st, int invert)
{
    return ApplyDispatch<2>::diag(g, lam, nu, nuc, h, d, invert, st);
}
}  // namespace dg
