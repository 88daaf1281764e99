"""B200-native SIP-DG implicit-stage solver for arXiv 2112.04167 (Guesmi, Grotteschi, Stiller).

Thin Python binding over the C-ABI library ``libdgsip.so`` (``include/dg.h``): argument
marshalling only -- every step of the hot path runs in the hand-written sm_100a kernels.
There is no CPU fallback: importing this package fails loudly when the library is
missing, and every call raises :class:`DGError` on a non-zero status.

PyTorch is used only for device memory, streams and process groups.
"""
from ._capi import (  # noqa: F401
    DG_EBREAKDOWN,
    DG_ECUDA,
    DG_EINVAL,
    DG_ENCCL,
    DG_ENOMEM,
    DG_ENOTCONV,
    DG_EUNSUPPORTED,
    DG_OK,
    DG_PC_JACOBI,
    DG_PC_SCHWARZ2,
    DGError,
    Mesh,
    SolveInfo,
    StageInfo,
    StepInfo,
    Tableau,
    dg_check_field,
    dg_convect_rhs,
    ViscModel,
    dg_derivative,
    dg_div_stab_apply,
    dg_div_stab_solve,
    dg_divergence,
    dg_gradient,
    dg_gll_tables,
    dg_helmholtz_apply,
    dg_helmholtz_apply_host,
    dg_helmholtz_diag,
    dg_imex_rk_step,
    dg_imex_rk_step_vv,
    dg_imex_stage,
    dg_last_apply_kernel,
    dg_last_error,
    dg_mesh_create,
    dg_mesh_destroy,
    dg_mesh_set_div_stab,
    dg_mesh_element_offset,
    dg_mesh_launch_count,
    dg_mesh_local_elements,
    dg_mesh_local_ndof,
    dg_mesh_mass,
    dg_mesh_node_coords,
    dg_mesh_get_precond,
    dg_mesh_set_precond,
    dg_mesh_set_stream,
    dg_schwarz_apply,
    dg_nccl_unique_id,
    dg_pcg_solve,
    dg_pcg_solve_host,
    dg_version,
    library_path,
)
from .tableaux import TABLEAUX  # noqa: F401,E402
