"""Where a single C1 image's latency goes (stage CUDA events vs wall clock)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17869_b200 as ds
from oracle.oracle import Oracle
img = Oracle("port").value_noise(640, 480, 0x5EED0000, 5, 32)
with ds.Extractor() as ex:
    ex.set_profiling(True)
    for _ in range(3):
        ex.extract(img)
    ts = []
    st = {}
    for _ in range(20):
        t0 = time.perf_counter()
        fs = ex.extract(img)
        ts.append(time.perf_counter() - t0)
        for k, v in ex.stage_times().items():
            st[k] = st.get(k, 0) + v / 20
    print("wall ms median", 1e3 * float(np.median(ts)), "stages", {k: round(v, 3) for k, v in st.items()},
          "sum", round(sum(st.values()), 3), "kps", len(fs), "launches", ex.kernel_launches())
