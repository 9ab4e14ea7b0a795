"""Phase timeline of the decode-step kernel (debug build: KVRING_NVCC_DEFS=-DKV_TIMELINE).

Builds libkvring with per-CTA %globaltimer stamps (the last 4 launches are kept), runs
tools/step_probe.py decode steps through the one-launch loop without events (launches
overlap: programmatic dependent launch) and prints, per launch, when its CTAs pass each
phase boundary, relative to the first shown launch's first CTA:
  start | blob (descriptor in shared memory) | wait (work list + wait for the previous
  grid) | copies | tables | done.   Rebuild without the define afterwards.
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    env = dict(os.environ, KVRING_NVCC_DEFS="-DKV_TIMELINE")
    subprocess.run([sys.executable, "-m", "paper_2601_22438_b200.build", "--force"], env=env,
                   check=True, cwd=ROOT, stdout=subprocess.DEVNULL)
    os.environ["STEP_PROBE_NOFLUSH"] = "1"
    os.environ["STEP_PROBE_NOEVENTS"] = "1"
    import numpy as np
    argv = list(sys.argv)
    sys.argv = ["step_probe", "decode", argv[1] if len(argv) > 1 else "12"]
    import step_probe
    step_probe.main()
    from paper_2601_22438_b200 import kvring as K
    f = K.lib().kv_debug_timeline
    f.restype = ctypes.c_int
    NL = 32
    buf = np.zeros(NL * 1024 * 8, dtype=np.uint64)
    f(buf.ctypes.data, buf.size)
    t = buf.reshape(NL, 1024, 8)
    launches = []
    for k in range(NL):
        nz = t[k][:, 7] != 0
        if nz.any():
            launches.append((int(t[k][nz][0, 7]), t[k][nz].astype(np.float64)))
    launches.sort()
    names = ["start", "blob", "wait", "copies", "tables", "done"]
    t0 = min(x[:, 0].min() for _, x in launches[-4:])
    for nonce, x in launches[-4:]:     # the last 4 in full
        print("launch %d (%d CTAs):" % (nonce, len(x)))
        for k, name in enumerate(names):
            col = (x[:, k] - t0) / 1e3
            print("   %-7s min %8.2f  median %8.2f  max %8.2f us" % (name, col.min(),
                                                                     np.median(col), col.max()))
    # every kept launch, relative to its own first CTA start (copies = warp 0 of each CTA)
    print("\nlaunch  CTAs  period | blob.med wait.med wait.max | copies.med copies.max | "
          "done.med done.max | prev.done.max->wait.min")
    prev = None
    for nonce, x in launches:
        s0 = x[:, 0].min()
        r = lambda k, fn: (fn(x[:, k]) - s0) / 1e3
        period = (s0 - prev[:, 0].min()) / 1e3 if prev is not None else float("nan")
        gap = (x[:, 2].min() - prev[:, 5].max()) / 1e3 if prev is not None else float("nan")
        print("%6d %5d %7.2f | %8.2f %8.2f %8.2f | %10.2f %10.2f | %8.2f %8.2f | %6.2f" % (
            nonce, len(x), period, r(1, np.median), r(2, np.median), r(2, np.max),
            r(3, np.median), r(3, np.max), r(5, np.median), r(5, np.max), gap))
        prev = x


if __name__ == "__main__":
    try:
        main()
    finally:  # back to the product build
        subprocess.run([sys.executable, "-m", "paper_2601_22438_b200.build", "--force"],
                       cwd=ROOT, stdout=subprocess.DEVNULL)
