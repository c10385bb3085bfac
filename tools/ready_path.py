"""Critical path of a factor_kernel per-block profile (diagnostic build) through the recorded
releasers: for every block the profile holds the time it became ready (slot 18) and the block
whose release made it ready (slot 26); walking back from the last block to finish gives the
chain that actually gated the run.  usage: python tools/ready_path.py blkprof.npy"""
import sys
import numpy as np
a = np.load(sys.argv[1])
t0 = a[:, 0].min()
st = (a[:, 0] - t0) / 1e3; en = (a[:, 10] - t0) / 1e3
rd = np.where(a[:, 18] > 0, (a[:, 18] - t0) / 1e3, np.nan)
rel = a[:, 26].astype(np.int64)
ph = a[:, 2:10] / 1965.
names = ["contrib", "Lprep", "Uprep", "upd", "pivot", "drop", "reg", "release"]
K = int(np.argmax(en)); path = [K]
while not np.isnan(rd[K]) and len(path) < 100000:
    K = int(rel[K]); path.append(K)
path = np.array(path[::-1])
rel_lat = np.array([rd[path[i + 1]] - st[path[i]] for i in range(len(path) - 1)])
wait = np.array([st[path[i + 1]] - rd[path[i + 1]] for i in range(len(path) - 1)])
print("ready path: %d blocks, %.2f ms -> %.2f ms" % (len(path), st[path[0]] / 1e3, en[path[-1]] / 1e3))
print("  releaser start -> ready: sum %.2f ms, mean %.1f us, median %.1f" % (rel_lat.sum() / 1e3, rel_lat.mean(), np.median(rel_lat)))
print("  ready -> start (queue):  sum %.2f ms, mean %.1f us, median %.1f" % (wait.sum() / 1e3, wait.mean(), np.median(wait)))
print("  path block phases us:", {k: round(float(ph[path, i].mean()), 1) for i, k in enumerate(names)})
print("  nR %.0f nC %.0f" % (a[path, 13].mean(), a[path, 14].mean()))
q = np.percentile(rel_lat, [10, 50, 90, 99])
print("  releaser latency percentiles", np.round(q, 1))
