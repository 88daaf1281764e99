// apply3.cu -- 3-D instantiations of the SIP apply / diagonal kernels (see apply.cuh).
#include "dev_common.cuh"
namespace dg {
DG_DEFINE_CONST_TABLES(upload_tables_apply3)
}
#include "apply.cuh"
namespace dg {
cudaError_t launch_apply3(const ApplyParams &a, bool varnu, int mode, int *grid, int smem, cudaStream_t st)
{
    return ApplyDispatch<3>::apply(a, varnu, mode, grid, smem, st);
}
bool apply3_ranges_ok(const Geom &g) { return ApplyDispatch<3>::ranges_ok(g); }
bool apply3_split_pcg_ok(const Geom &g, const double *nu) { return ApplyDispatch<3>::split_pcg_ok(g, nu); }
cudaError_t launch_diag3(const Geom &g, double lam, const double *nu, double nuc, const Halo &h, double *d,
                         cudaStream_t st, int invert)
{
    return ApplyDispatch<3>::diag(g, lam, nu, nuc, h, d, invert, st);
}
}  // namespace dg

#ifdef DG_V5_DEBUG
extern "C" int dg_debug_counters(unsigned long long *out, int reset)
{
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out, dg::v5::g_dbg, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(dg::v5::g_dbg, z, sizeof(z));
    }
    return 0;
}
#endif
