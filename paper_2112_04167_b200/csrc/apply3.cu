// apply3.cu -- 3-D instantiations of the SIP apply / diagonal kernels (see apply.cuh).
#include "dev_common.cuh"
namespace dg {
DG_DEFINE_CONST_TABLES(upload_tables_apply3)
}
#include "apply.cuh"
namespace dg {
cudaError_t launch_apply3(const ApplyParams &a, bool varnu, bool pcg, int *grid, int smem, cudaStream_t st)
{
    return ApplyDispatch<3>::apply(a, varnu, pcg, grid, smem, st);
}
cudaError_t launch_diag3(const Geom &g, double lam, const double *nu, double nuc, const Halo &h, double *d,
                         cudaStream_t st)
{
    return ApplyDispatch<3>::diag(g, lam, nu, nuc, h, d, st);
}
}  // namespace dg
