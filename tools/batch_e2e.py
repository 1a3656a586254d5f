"""Where the cfg3 batch (4096 x n=16) end-to-end time goes: Python marshalling, the C ABI call
(host prep + device), device time, result conversion (development aid)."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import api  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402

ms = W.load_cfg3_batch(4096)
for prec in sys.argv[1:] or ["fp64", "128"]:
    T.torontonian_batch(ms[:64], prec)
    for rep in range(2):
        t0 = time.perf_counter()
        ins = [api._In(m) for m in ms]
        arr = (api.TorInput * len(ins))(*[i.s for i in ins])
        res = (api.TorResult * len(ins))()
        err = api.TorError()
        t1 = time.perf_counter()
        api._check(api.lib().tor_torontonian_batch(arr, len(ins), api._prec(prec), 0, res, C.byref(err)), err)
        t2 = time.perf_counter()
        out = [api._result_dict(res[i], 1) for i in range(len(ins))]
        t3 = time.perf_counter()
        print(f"{prec}: marshal {1e3 * (t1 - t0):.1f} ms, C call {1e3 * (t2 - t1):.1f} ms "
              f"(device {out[0]['device_ms']:.2f} ms), results {1e3 * (t3 - t2):.1f} ms, "
              f"total {1e3 * (t3 - t0):.1f} ms", flush=True)
