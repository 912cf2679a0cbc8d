"""Print a hash of every synthetic input table, to compare machines."""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as O
from paper_2312_08715_b200 import configs, synth
import math
tr = configs.cfg4(lambda k, v, t, p: O.render(k, [(v, t, p)]), O.voxel_to_mesh, seed=0, n_frames=5)
for s in tr["stages"]:
    print("cfg4 rot", hashlib.md5(s["rotations"].tobytes()).hexdigest())
    print("  ", [x.hex() for x in s["rotations"][26]])
print("cos", math.cos(0.06046212).hex(), math.sin(0.06046212).hex(), math.log(0.3).hex())
a = 2.0 * math.pi / 180 * math.sqrt(3.0)
print("cos a/2", math.cos(a / 2).hex(), math.sin(a / 2).hex())
print("gt", hashlib.md5(np.array(tr["gt"]).tobytes()).hexdigest())
