"""Set up one config and launch ONE sub-kernel of the step a few times (sc_profile), for ncu
captures of that kernel (diagnostics).  usage: python scripts/prof_kernel.py CONFIG WHICH [N]
(WHICH: 0 explicit, 1 c-element products, 2 solve)"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import sc_inputs  # noqa: E402
import paper_2310_14712_b200 as pkg  # noqa: E402

cid, which = int(sys.argv[1]), int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = sc_inputs.get_config(cid)
s = pkg.from_config(cfg)
s.profile(which, n)
s.sync()
s.close()
print("ok")
