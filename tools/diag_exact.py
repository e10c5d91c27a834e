"""Reference-exact (fixed) mode vs the engine oracle after one step on the
perturbed 6x6 KAT scene: which nodes differ and how (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2507_11794_b200 as P
from conftest import load_golden
from oracle import oracle as O

k = load_golden("kats.npz")
mesh = P.generate_cloth_grid(6, 6)
mesh.positions = k["pert_positions"]
params = P.SimParams(gravity=(0.0, 0.0, 0.0), stiffness=30.0, damping=0.4)
for kern in ("pair", "strip"):
    eng = P.Engine(mesh, params=params, precision="fixed", kernel=kern)
    eng.buffers.vel[...] = k["pert_vel"]
    eo = O.EngineOracle(mesh, params)
    eo.vel[...] = k["pert_vel"]
    eng.step()
    eo.step()
    pos, vel = eng.read_positions(), eng.read_velocities()
    dp = np.argwhere(pos != eo.pos)
    dv = np.argwhere(vel != eo.vel)
    print(kern, "pos diff", len(dp), "vel diff", len(dv))
    for n, c in dv[:10]:
        print("  node", n, "comp", c, "vel", vel[n, c], eo.vel[n, c], "forces oracle", eo.forces[n])
    print("  pos==golden", np.array_equal(pos, k["pert_eng_pos1"]), "oracle==golden", np.array_equal(eo.pos, k["pert_eng_pos1"]))
