"""Butcher tableaux of the paper's IMEX Runge-Kutta methods (Appendix).

Each entry: (implicit DIRK tableau A_im, explicit tableau A_ex, b_im, b_ex, c) in the paper's
layout (a_im[0][0] = 0, equal nodes c for both parts).  Used to fill the C struct
``dg_tableau`` of ``dg_imex_rk_step``; method data only (no arithmetic).
"""
from fractions import Fraction as F

TABLEAUX = {
    # RK-TR
    "RK-TR": dict(
        c=[0, 1, 1],
        a_im=[[0, 0, 0], [0, 1, 0], [F(1, 2), 0, F(1, 2)]],
        a_ex=[[0, 0, 0], [1, 0, 0], [F(1, 2), F(1, 2), 0]],
        b_im=[F(1, 2), 0, F(1, 2)],
        b_ex=[F(1, 2), F(1, 2), 0],
    ),
    # RK-CB2
    "RK-CB2": dict(
        c=[0, F(2, 5), 1],
        a_im=[[0, 0, 0], [0, F(2, 5), 0], [0, F(5, 6), F(1, 6)]],
        a_ex=[[0, 0, 0], [F(2, 5), 0, 0], [0, 1, 0]],
        b_im=[0, F(5, 6), F(1, 6)],
        b_ex=[0, F(5, 6), F(1, 6)],
    ),
    # RK-CB3e
    "RK-CB3e": dict(
        c=[0, F(1, 3), 1, 1],
        a_im=[[0, 0, 0, 0], [0, F(1, 3), 0, 0], [0, F(1, 2), F(1, 2), 0], [0, F(3, 4), F(-1, 4), F(1, 2)]],
        a_ex=[[0, 0, 0, 0], [F(1, 3), 0, 0, 0], [0, 1, 0, 0], [0, F(3, 4), F(1, 4), 0]],
        b_im=[0, F(3, 4), F(-1, 4), F(1, 2)],
        b_ex=[0, F(3, 4), F(-1, 4), F(1, 2)],
    ),
    # RK-ARS3
    "RK-ARS3": dict(
        c=[0, F(1, 2), F(2, 3), F(1, 2), 1],
        a_im=[[0, 0, 0, 0, 0], [0, F(1, 2), 0, 0, 0], [0, F(1, 6), F(1, 2), 0, 0],
              [0, F(-1, 2), F(1, 2), F(1, 2), 0], [0, F(3, 2), F(-3, 2), F(1, 2), F(1, 2)]],
        a_ex=[[0, 0, 0, 0, 0], [F(1, 2), 0, 0, 0, 0], [F(11, 18), F(1, 18), 0, 0, 0],
              [F(5, 6), F(-5, 6), F(1, 2), 0, 0], [F(1, 4), F(7, 4), F(3, 4), F(-7, 4), 0]],
        b_im=[0, F(3, 2), F(-3, 2), F(1, 2), F(1, 2)],
        b_ex=[F(1, 4), F(7, 4), F(3, 4), F(-7, 4), 0],
    ),
}
