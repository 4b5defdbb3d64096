"""TMEM vs shared-memory operand feeds for the config-5 phase B
(tools/csrc/tmem_probe.cu, built to tools/libtmem_probe.so):

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -shared \\
         -Xcompiler -fPIC tools/csrc/tmem_probe.cu -o tools/libtmem_probe.so
    python tools/tmem_probe.py > profiles/r02/tmem_probe.json

Prints raw tcgen05.ld bandwidth (bytes / clk / SM at the SM clock sampled
during the run) and, for the phase-B loop on 128 points per CTA, point-terms
per clock per SM, with the outputs checked bit for bit against numpy's
((c * v_p) * v_q) summed left to right.
"""
import ctypes as C
import json
import statistics
from pathlib import Path

import numpy as np
import torch

lib = C.CDLL(str(Path(__file__).resolve().parent / "libtmem_probe.so"))
lib.ldtm_launch.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
lib.phaseb_launch.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream().cuda_stream


def clock_mhz():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:  # noqa: BLE001
        return 1965


def timed(fn, reps=7):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    mhz = []
    for i in range(reps):
        fn()
        ev[i + 1].record()
    mhz.append(clock_mhz())
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps)) * 1e-3, statistics.median(mhz)


res = {"sm_count": sms}
out = torch.zeros(1 << 12, dtype=torch.int64, device="cuda")
for n, k in ((2, 4), (2, 8), (2, 16), (4, 4), (4, 8), (8, 4), (8, 8)):
    for warps in (4, 8, 16):
        iters = 4096
        s, mhz = timed(lambda: lib.ldtm_launch(n, k, out.data_ptr(), sms, warps * 32, iters, st))
        assert torch.cuda.synchronize() is None
        by = sms * warps * iters * k * n * 4 * 32
        res[f"ldtm_x{n}_k{k}_w{warps}_B_per_clk_sm"] = by / s / sms / (mhz * 1e6)
        res[f"ldtm_x{n}_k{k}_w{warps}_instr_per_clk_sm"] = sms * warps * iters * k / s / sms / (mhz * 1e6)

# LDTM.x2 vs LDS.64: separate or shared data path?  (8 LDS.64 and/or K LDTM per step)
lib.mix_launch.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
for k, wl in ((0, 1), (8, 0), (8, 1), (4, 1)):
    for warps in (8, 16):
        iters = 4096
        s, mhz = timed(lambda: lib.mix_launch(k, wl, out.data_ptr(), sms, warps * 32, iters, st))
        per = sms * warps * iters / s / sms / (mhz * 1e6)
        res[f"mix_lds{8 * wl}_ldtm{k}_w{warps}"] = {"ms": s * 1e3, "lds_wavefronts_per_clk_sm": per * 8 * wl * 2,
                                                     "ldtm_instr_per_clk_sm": per * k}

# phase B
NOPS, NOUT, NTERM, NPTS, NSM = 240, 24, 64, 128, 112
rng = np.random.default_rng(7)
ops = rng.uniform(0.9, 1.1, (NOPS, NPTS))
tdt = np.dtype([("c", "<f8"), ("p", "<u4"), ("q", "<u4")])
tab = np.zeros((NOUT, NTERM), dtype=tdt)
tab["c"] = rng.standard_normal((NOUT, NTERM))
tab["p"] = rng.integers(0, NOPS, (NOUT, NTERM))
tab["q"] = rng.integers(0, NSM, (NOUT, NTERM))
tab_smem = tab.copy()
tab_smem["p"] = rng.integers(0, NSM, (NOUT, NTERM))
tab_tm = tab.copy()
tab_tm["p"] = rng.integers(0, 128, (NOUT, NTERM))


def want_of(t):
    w = np.empty((NOUT, NPTS))
    for o in range(NOUT):
        acc = None
        for k in range(NTERM):
            term = (t["c"][o, k] * ops[t["p"][o, k]]) * ops[t["q"][o, k]]
            acc = term if acc is None else acc + term
        w[o] = acc
    return w


d_ops = torch.from_numpy(ops).cuda()
for src, t in ((0, tab), (1, tab), (2, tab_smem), (3, tab_tm), (4, tab_smem)):
    want = want_of(t)
    d_tab = torch.from_numpy(t.view(np.uint8).copy()).cuda()
    for nw in (4, 8, 12, 16, 24):
        d_out = torch.zeros((NOUT, NPTS), dtype=torch.float64, device="cuda")
        reps = 64
        rc = lib.phaseb_launch(src, nw, d_ops.data_ptr(), d_tab.data_ptr(), d_out.data_ptr(), sms, reps, st)
        if rc == -1:
            continue
        torch.cuda.synchronize()
        ok = d_out.cpu().numpy().tobytes() == want.tobytes()
        s, mhz = timed(lambda: lib.phaseb_launch(src, nw, d_ops.data_ptr(), d_tab.data_ptr(), d_out.data_ptr(), sms,
                                                 reps, st))
        pt_terms = sms * reps * NOUT * NTERM * NPTS
        res[f"phaseb_src{src}_w{nw}"] = {"point_terms_per_clk_sm": pt_terms / s / sms / (mhz * 1e6), "ms": s * 1e3,
                                         "bits_ok": ok, "mhz": mhz}
# SRC 5: 64 points, packed production table, TMEM (ops < 128) / shared (>= 128) by operand
NPT5 = 64
ops5 = rng.uniform(0.9, 1.1, (NOPS, NPT5))
c5 = rng.standard_normal((NOUT, NTERM))
p5 = rng.integers(0, NOPS, (NOUT, NTERM))
q5 = rng.integers(0, NOPS, (NOUT, NTERM))
packed = np.zeros((NOUT, 40, 16), dtype=np.uint8)
for o in range(NOUT):
    for g in range(8):
        packed[o, 5 * g:5 * g + 4] = c5[o, 8 * g:8 * g + 8].astype("<f8").view(np.uint8).reshape(4, 16)
        pq = (p5[o, 8 * g:8 * g + 8] | (q5[o, 8 * g:8 * g + 8] << 8)).astype("<u2")
        packed[o, 5 * g + 4] = pq.view(np.uint8)
want5 = np.empty((NOUT, NPT5))
for o in range(NOUT):
    acc = None
    for k in range(NTERM):
        t = (c5[o, k] * ops5[p5[o, k]]) * ops5[q5[o, k]]
        acc = t if acc is None else acc + t
    want5[o] = acc
d_ops5 = torch.from_numpy(ops5).cuda()
d_tab5 = torch.from_numpy(packed.reshape(-1).copy()).cuda()
for nw in (8, 12, 16, 24):
    d_out = torch.zeros((NOUT, NPT5), dtype=torch.float64, device="cuda")
    reps = 64
    rc = lib.phaseb_launch(5, nw, d_ops5.data_ptr(), d_tab5.data_ptr(), d_out.data_ptr(), sms, reps, st)
    torch.cuda.synchronize()
    ok = d_out.cpu().numpy().tobytes() == want5.tobytes()
    s5, mhz = timed(lambda: lib.phaseb_launch(5, nw, d_ops5.data_ptr(), d_tab5.data_ptr(), d_out.data_ptr(), sms,
                                              reps, st))
    res[f"phaseb_src5_w{nw}"] = {"point_terms_per_clk_sm": sms * reps * NOUT * NTERM * NPT5 / s5 / sms / (mhz * 1e6),
                                 "ms": s5 * 1e3, "bits_ok": ok, "mhz": mhz, "rc": rc}
print(json.dumps(res, indent=1))
