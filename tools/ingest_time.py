"""Container ingest throughput: record payloads (records.py:126-183) of
C3-size structures (100 atoms, ~29 record edges per atom) decoded on the
device (decode_payloads: CRC32 + scatter) vs the host codec
(decode_record per payload), bytes per second.

    python tools/ingest_time.py [n_records]"""

import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_12909_b200.records import GraphRecord, decode_record, encode_record  # noqa: E402
from paper_2406_12909_b200.store import decode_payloads  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 20000
rng = np.random.default_rng(0)
proto = []
for k in range(16):  # 16 distinct payloads, repeated
    n, deg = 100, 29
    src = rng.integers(0, n, n * deg)
    dst = np.repeat(np.arange(n), deg)
    proto.append(encode_record(GraphRecord(rng.integers(1, 9, n), rng.uniform(0, 12, (n, 3)),
                                           np.stack([src, dst], 1), float(k),
                                           rng.normal(size=(n, 3)), f"s{k}")))
payloads = [proto[k % 16] for k in range(S)]
lens = np.array([len(p) for p in payloads], np.int64)
offs = np.concatenate([[0], np.cumsum(lens)])[:-1].astype(np.int64)
blob_np = np.frombuffer(b"".join(payloads), np.uint8)
pin = "--pageable" not in sys.argv
blob = torch.empty(blob_np.shape[0], dtype=torch.uint8, pin_memory=pin).numpy()  # as read_range_raw
blob[:] = blob_np
decode_payloads(blob[:int(offs[64])], offs[:64], lens[:64])  # warm up
torch.cuda.synchronize()
t0 = time.perf_counter()
d = decode_payloads(blob, offs, lens)
torch.cuda.synchronize()
t_dev = time.perf_counter() - t0
k_host = min(S, 2000)
t0 = time.perf_counter()
for p in payloads[:k_host]:
    decode_record(p)
t_host = (time.perf_counter() - t0) * S / k_host
print(f"{S} records, {blob.nbytes / 1e6:.0f} MB: device decode (H2D + CRC + scatter) "
      f"{t_dev * 1e3:.1f} ms = {blob.nbytes / t_dev / 1e9:.2f} GB/s; host decode_record "
      f"{t_host * 1e3:.0f} ms = {blob.nbytes / t_host / 1e9:.3f} GB/s (1 core, sampled on "
      f"{k_host})")

# kernel-only: blob already in HBM, CUDA events around scan and decode
from paper_2406_12909_b200._lib import call, ptr, stream_handle  # noqa: E402
dev = torch.device("cuda")
bd = torch.as_tensor(blob, device=dev)
od, ld = torch.as_tensor(offs, device=dev), torch.as_tensor(lens, device=dev)
nm = torch.empty(3, S, dtype=torch.int32, device=dev)
s = stream_handle()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
N = int(d["n"].sum())
E = int(d["m"].sum())
z = torch.empty(N, dtype=torch.int32, device=dev)
pos = torch.empty(N, 3, dtype=torch.float64, device=dev)
frc = torch.empty(N, 3, dtype=torch.float64, device=dev)
en = torch.empty(S, dtype=torch.float64, device=dev)
ed = torch.empty(E, 2, dtype=torch.int32, device=dev)
for _ in range(2):
    ev[0].record()
    call("gfm_record_scan", ptr(bd), ptr(od), ptr(ld), S, ptr(nm[0]), ptr(nm[1]), ptr(nm[2]), s)
    ev[1].record()
    call("gfm_record_decode", ptr(bd), ptr(od), S, ptr(d["noff"]), ptr(d["eoff"]), ptr(z),
         ptr(pos), ptr(frc), ptr(en), ptr(ed), None, None, s)
    ev[2].record()
    torch.cuda.synchronize()
ts, tdd = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
print(f"  kernels only: scan (length + CRC32) {ts:.2f} ms = {blob.nbytes / ts / 1e6:.1f} GB/s, "
      f"decode (scatter) {tdd:.2f} ms = {blob.nbytes / tdd / 1e6:.1f} GB/s")
