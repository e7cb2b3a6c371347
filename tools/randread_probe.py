"""How fast can a B200 serve RANDOM reads of one 128-byte line (or a 32-byte sector) out of a table far larger
than L2?  The deep-node arena reads of K1 (BASELINE configs 4 and 5) are exactly that, so this number is their
roofline, not the streaming copy bandwidth.  Uses torch's row gather (library kernel: measurement aid only).

    python tools/randread_probe.py [--gb 16]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=16.0)
    ap.add_argument("--reads", type=int, default=200_000_000)
    args = ap.parse_args()
    out = {}
    for row_bytes in (128, 32, 8):
        words = row_bytes // 8
        rows = int(args.gb * 1e9) // row_bytes
        table = torch.zeros((rows, words), dtype=torch.int64, device="cuda")
        idx = torch.randint(0, rows, (args.reads,), device="cuda")
        dst = torch.empty((args.reads, words), dtype=torch.int64, device="cuda")
        for _ in range(2):
            torch.index_select(table, 0, idx, out=dst)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            torch.index_select(table, 0, idx, out=dst)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        out[f"row_{row_bytes}B"] = {"table_gb": args.gb, "reads": args.reads, "ms": ms,
                                    "greads_per_s": args.reads / ms / 1e6, "useful_GBps": args.reads * row_bytes / ms / 1e6,
                                    "note": "time also covers reading the 8-byte index and writing the row"}
        print(row_bytes, out[f"row_{row_bytes}B"], flush=True)
        del table, idx, dst
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "randread_probe.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
