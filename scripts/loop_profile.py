"""Phase times of the device closed loop (RG_LOOP_PROFILE build via RG_LIB_PATH): per step,
block 0's passes, the grid barrier and the between-step work (us), for 1k and 10k."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop
PLANT = rg.make_plant("surrogate-fc")
BOX = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
DESK = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
lib = _capi.context(0).lib
for n in (1000, 10_000):
    cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=n)
    run_closed_loop(PLANT, BOX, rg.DisturbanceModel.scaled(0.001, 3), cfg, DESK, 300, 2024)
    buf = np.zeros((4096, 6), dtype=np.uint64)
    assert lib.rg_loop_profile(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    b = buf[20:280].astype(float) / 1000
    passes, bar, tot = b[:, 0], b[:, 1] - b[:, 0], b[:, 2] - b[:, 1]
    print(f"n={n}: block 0: passes {np.median(passes):.2f} us, barrier {np.median(bar):.2f} us, "
          f"between {np.median(tot):.2f} us; last block: passes {np.median(b[:, 3]):.2f}, "
          f"barrier {np.median(b[:, 4] - b[:, 3]):.2f}, between {np.median(b[:, 5] - b[:, 4]):.2f} "
          f"(medians over steps 20-279)", flush=True)
