"""TGP at the paper's degree P = 10 on 8 x 8 elements: RK-CB2 / RK-CB3e
temporal convergence from dt = 2^-5, without and with the divergence / mass-flux stabilisation."""
import sys
sys.path.insert(0, '.')
from tools.tg_eoc import run

for stab in (None, (1.0, 1.0)):
    for name in ("RK-CB3e", "RK-CB2", "RK-ARS3"):
        try:
            errs, eoc = run(name, N=8, P=10, stab=stab, ks=(5, 6, 7, 8))
            print(name, "P=10", "stab" if stab else "nostab", ["%.3e" % e for e in errs], ["%.2f" % x for x in eoc], flush=True)
        except Exception as e:
            print(name, "P=10", "stab" if stab else "nostab", "failed", str(e)[:80], flush=True)
