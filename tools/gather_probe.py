"""Achievable HBM bandwidth of random whole-row gathers (K1's access pattern)
for the row sizes of the bench shapes, against the measured copy peak.

    python tools/gather_probe.py
"""
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2507_17094_b200 import _abi  # noqa: E402

lib = _abi.load()
dev = torch.device("cuda", 0)
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
peak = float(peaks.get("hbm_gbs", 6650.0))
sms = torch.cuda.get_device_properties(dev).multi_processor_count
sink = torch.zeros(1, dtype=torch.int32, device=dev)
g = torch.Generator(device=dev)
g.manual_seed(5)
for row_bytes, label in ((128, "C3 u8 d=128"), (384, "C2 f32 d=96"), (512, "f32 d=128"), (800, "C5 f32 d=200"),
                         (3840, "C4 f32 d=960")):
    n_rows = (8 << 30) // row_bytes  # an 8 GB table (>> L2)
    table = torch.empty(n_rows * row_bytes // 4, dtype=torch.int32, device=dev).random_(generator=g)
    n_ids = min(n_rows, (2 << 30) // row_bytes)  # ~2 GB gathered per launch
    ids = torch.randint(0, n_rows, (n_ids,), device=dev, dtype=torch.int32, generator=g)
    st = torch.cuda.current_stream(dev).cuda_stream
    for blocks in (sms, 2 * sms):
        for _ in range(2):
            _abi.check(lib.pw_gather_probe(table.data_ptr(), row_bytes, ids.data_ptr(), n_ids, sink.data_ptr(),
                                           blocks, C.c_void_p(st)))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            _abi.check(lib.pw_gather_probe(table.data_ptr(), row_bytes, ids.data_ptr(), n_ids, sink.data_ptr(),
                                           blocks, C.c_void_p(st)))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = n_ids * row_bytes / (ms / 1e3) / 1e9
        print(json.dumps({"row_bytes": row_bytes, "shape": label, "blocks": blocks, "rows": n_ids,
                          "ms": round(ms, 3), "gather_gbs": round(gbs, 1), "frac_of_copy_peak": round(gbs / peak, 3),
                          "copy_peak_gbs": peak}), flush=True)
    del table, ids
    torch.cuda.empty_cache()
