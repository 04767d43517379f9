import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
os.environ.setdefault("HSRQ_TIMELINE", "84")
import subprocess
exec(open("tools/profile_solve.py").read().split("import ctypes")[0])
from paper_2101_05063_b200 import _lib
L = _lib.load()
gs.launch(start, True)  # one solve with the timeline armed (HSRQ_TIMELINE = tile column)
L.hsrq_debug_timeline.restype = ctypes.c_int64
buf = np.zeros(8192 * 8, dtype=np.uint64)
print("rc", L.hsrq_debug_timeline(ctypes.c_void_p(buf.ctypes.data)))
tl = buf.reshape(8192, 8)[:, :8].astype(np.int64)
tl = tl[tl[:, 1] > 0]
t0 = tl[:, 1].min()
np.save("gpurun_out/timeline.npy", tl)
pro = tl[:, 2] - tl[:, 1]; mma = tl[:, 3] - tl[:, 2]; epi = tl[:, 4] - tl[:, 3]
print("n", len(tl), "prologue us", np.median(pro)/1e3, "mma us", np.median(mma)/1e3, "epi us", np.median(epi)/1e3)
print("epi parts (us): stage+loads", np.median(tl[:,5]-tl[:,3])/1e3, "pass1", np.median(tl[:,6]-tl[:,5])/1e3, "step3", np.median(tl[:,7]-tl[:,6])/1e3, "pass2+tail", np.median(tl[:,4]-tl[:,7])/1e3)
sm = tl[:, 0]
for s in (0, 1, 77):
    rows = tl[sm == s]
    rows = rows[np.argsort(rows[:, 1])][:8]
    for r in rows:
        print(s, [(int(x - t0) // 100) / 10 for x in r[1:5]])
