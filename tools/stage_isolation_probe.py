import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1910_01031_b200 import Config, Ensemble
s = torch.cuda.Stream()
ens = Ensemble(Config(), 100, stream=s.cuda_stream)
ens.init_double_jet()
for _ in range(3): ens.model_step(1)
ens.sync()
iso = [ens.time_stages(1) for _ in range(3)]
r = []
for _ in range(20):
    time.sleep(0.005)
    r.append(ens.time_stages(1))
print("isolated (1 substep, 5 ms idle before):", np.median(np.array(r), axis=0))
r = [ens.time_stages(7) for _ in range(5)]
print("back to back (7 substeps):", np.median(np.array(r), axis=0))
