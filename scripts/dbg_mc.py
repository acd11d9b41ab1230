import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, oracle
import paper_1201_2025_b200 as hs
cube = oracle.port.random_cube(12, 600, 4, 6012)
reqs = [hs.DetectRequest("lrx", hs.WindowConfig.single(11))]
os.environ.pop("HSAD_NO_STAGE", None)
a = hs.detect_multi(torch.as_tensor(cube).cuda(), reqs)[0][0].cpu().numpy()
os.environ["HSAD_NO_STAGE"] = "1"
b = hs.detect_multi(torch.as_tensor(cube).cuda(), reqs)[0][0].cpu().numpy()
tag = os.path.basename(os.environ.get("HSAD_B200_LIB", "cur"))
np.save(f"gpurun_out/mc_{tag}_staged.npy", a); np.save(f"gpurun_out/mc_{tag}_plain.npy", b)
print(tag, "differ", int((a != b).sum()))
