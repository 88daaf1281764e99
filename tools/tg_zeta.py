import sys; sys.path.insert(0,'.')
from tools.tg_eoc import run
for z in (10.0, 100.0):
    for name in ("RK-CB3e","RK-CB2"):
        try:
            errs,eoc=run(name, stab=(z,z), ks=(5,6,7))
            print(name,z,["%.3e"%e for e in errs],["%.2f"%x for x in eoc],flush=True)
        except Exception as e:
            print(name,z,"failed",str(e)[:80],flush=True)
