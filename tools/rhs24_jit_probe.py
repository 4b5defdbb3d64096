"""Probe: can a table-specialised (generated, straight-line) phase B of
config 5 with ALL 24 outputs per thread (lane = point, one code block shared
by every warp) run near the FP64 pipe ceiling?

Round-2's codegen probe (tools/rhs24_codegen_probe.py) gave each warp its own
outputs, i.e. 12 distinct code blocks per SM, and was instruction-cache
bound.  Here every warp runs the SAME block — the 1536 terms of all 24
outputs, interleaved, with at most R operands cached in registers (Belady
eviction over the interleaved order) — on its own 32 points.  Operands come
from shared memory (SRC S, all warps read one [240][32] array: the bank
pattern of per-warp arrays) or from Tensor Memory (SRC T, TMEM lane =
point, 240 operands in 480 columns, loads issued one segment ahead and
waited for at the segment end).

    python tools/rhs24_jit_probe.py gen     # here: writes + compiles the variants
    python tools/rhs24_jit_probe.py run     # GPU box
"""
from __future__ import annotations

import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1308_1343_b200 import inputs  # noqa: E402

CSRC = ROOT / "tools" / "csrc"
OUT = ROOT / "tools"

NT, NO, NIN = 64, 24, 240


CHAINS = list(range(24))


def interleave(P, Q, R):
    """Order the 1536 terms: at each step the chain head with the most
    operands in an LRU model cache of R values (ties: the chain that is
    furthest behind, which keeps chains level and the code ILP-rich)."""
    pos = [0] * NO
    cache: dict[int, int] = {}
    order = []
    clock = 0
    while len(order) < len(CHAINS) * NT:
        best = None
        for o in CHAINS:
            t = pos[o]
            if t >= NT:
                continue
            key = ((P[o, t] in cache) + (Q[o, t] in cache), -t, -o)
            if best is None or key > best[0]:
                best = (key, o)
        o = best[1]
        t = pos[o]
        for v in (int(P[o, t]), int(Q[o, t])):
            clock += 1
            if v not in cache and len(cache) >= R:
                del cache[min(cache, key=cache.get)]
            cache[v] = clock
        order.append((o, t))
        pos[o] += 1
    return order


def belady(P, Q, order, R):
    """Given the term order, the load events with Belady eviction: returns
    a list of ('load', name, op) / ('term', o, t, name_p, name_q) and the
    load count."""
    uses = []
    for o, t in order:
        uses.append(int(P[o, t]))
        uses.append(int(Q[o, t]))
    nxt = [0] * len(uses)
    last: dict[int, int] = {}
    for i in range(len(uses) - 1, -1, -1):
        nxt[i] = last.get(uses[i], 1 << 30)
        last[uses[i]] = i
    cache: dict[int, tuple[str, int]] = {}   # op -> (name, next use)
    ev, nvar, loads = [], 0, 0
    for k, (o, t) in enumerate(order):
        names = []
        for j in (0, 1):
            i = 2 * k + j
            v = uses[i]
            if v not in cache:
                if len(cache) >= R:
                    protect = uses[2 * k] if j == 1 else None
                    victim = max((x for x in cache if x != protect), key=lambda x: cache[x][1])
                    del cache[victim]
                name = f"v{nvar}"
                nvar += 1
                loads += 1
                ev.append(("load", name, v))
                cache[v] = (name, nxt[i])
            else:
                cache[v] = (cache[v][0], nxt[i])
            names.append(cache[v][0])
        ev.append(("term", o, t, names[0], names[1]))
    return ev, loads


def lit(x: float) -> str:
    return f"__longlong_as_double({int(np.float64(x).view(np.int64))}ll)"


CONST_CF = False


def term_lines(ev, Cf, started):
    out = []
    for e in ev:
        if e[0] != "term":
            continue
        _, o, t, a, b = e
        c = f"CF[cz + {o * NT + t}]" if CONST_CF else lit(Cf[o, t])
        tm = f"__dmul_rn(__dmul_rn({c}, {a}), {b})"
        if o in started:
            out.append(f"  a{o} = __dadd_rn(a{o}, {tm});")
        else:
            out.append(f"  a{o} = {tm};")
            started.add(o)
    return out


def gen_body_S(ev, Cf, sync_every):
    L = ["__device__ __forceinline__ void body_S(uint32_t vb, double (&a)[NCH], int nw) {", "  const int cz = (int)opaque(0u);"]
    L += [f"  double a{o};" for o in range(NO)]
    started: set = set()
    nterm = 0
    for e in ev:
        if e[0] == "load":
            L.append(f"  const double {e[1]} = lds64(vb + {e[2] * 256});")
        else:
            L += term_lines([e], Cf, started)
            nterm += 1
            if sync_every and nterm % sync_every == 0:
                L.append("  named_bar(1, nw * 32);" if sync_every > 0 else "  __syncwarp();")
            if sync_every < 0 and nterm % (-sync_every) == 0:
                L.append("  __syncwarp();")
    L += [f"  a[{o - CHAINS[0]}] = a{o};" for o in CHAINS]
    L.append("}")
    return L


def gen_body_T(ev, Cf, seg, fname="body_T"):
    """Segments of `seg` terms; the loads a segment needs are issued during
    the previous segment and waited for (wait::ld + pin) at its end."""
    segs = []          # list of (loads, terms)
    cur_loads, cur_terms = [], []
    for e in ev:
        if e[0] == "load":
            cur_loads.append(e)
        else:
            cur_terms.append(e)
            if len(cur_terms) == seg:
                segs.append((cur_loads, cur_terms))
                cur_loads, cur_terms = [], []
    if cur_terms or cur_loads:
        segs.append((cur_loads, cur_terms))
    L = [f"__device__ __forceinline__ void {fname}(uint32_t tb, double (&a)[NCH]) {{", "  const int cz = (int)opaque(0u);"]
    L += [f"  double a{o};" for o in range(NO)]

    def issue(loads):
        r = []
        for _, name, op in loads:
            r.append(f"  uint32_t {name}l, {name}h; ld_x2(tb + {2 * op}, {name}l, {name}h);")
        return r

    def land(loads):
        r = ["  tmem_wait_ld();"]
        for _, name, op in loads:
            r.append(f"  pin({name}l); pin({name}h); const double {name} = __hiloint2double((int){name}h, (int){name}l);")
        return r

    started: set = set()
    L += issue(segs[0][0])
    L += land(segs[0][0])
    for k, (loads, terms) in enumerate(segs):
        if k + 1 < len(segs):
            L += issue(segs[k + 1][0])
        L += term_lines(terms, Cf, started)
        if k + 1 < len(segs):
            L += land(segs[k + 1][0])
    L += [f"  a[{o - CHAINS[0]}] = a{o};" for o in CHAINS]
    L.append("}")
    return L


HEADER = r"""
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double lds64(uint32_t a) {
    double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a)); return v; }
__shared__ uint32_t g_zero;
// a value ptxas cannot see through: every call re-reads a shared word that holds 0
__device__ __forceinline__ uint32_t opaque(uint32_t a) {
    uint32_t z; asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(z) : "r"(smem_u32(&g_zero)) : "memory"); return a + z; }
__device__ __forceinline__ void stg(double *p, double v) { asm volatile("st.global.f64 [%0], %1;" :: "l"(p), "d"(v) : "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tmem_alloc(uint32_t *slot, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st_x2(uint32_t taddr, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory"); }
__device__ __forceinline__ void ld_x2(uint32_t taddr, uint32_t &a, uint32_t &b) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr) : "memory"); }
__device__ __forceinline__ void pin(uint32_t &r) { asm volatile("" : "+r"(r)); }
"""

KERNEL_S = r"""
extern "C" __global__ void __launch_bounds__(384, 1) probe_S(const double *ops, double *out, int reps) {
    extern __shared__ double vals[];
    for (int e = threadIdx.x; e < 240 * 32; e += blockDim.x) vals[e] = ops[e];
    if (threadIdx.x == 0) g_zero = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t vb = smem_u32(vals + lane);
    double *o = out + ((size_t)(blockIdx.x * nw + warp) * 24) * 32 + lane;
    for (int r = 0; r < reps; ++r) {
        double a[NCH] = {0};
        _Pragma("unroll 1") for (int b = 0; b < NBLK; ++b) body_S(opaque(vb), a, nw);
#pragma unroll
        for (int k = 0; k < NCH; ++k) stg(o + 32 * k, a[k]);
    }
}
extern "C" int launch_S(const double *ops, double *out, int blocks, int threads, int reps) {
    cudaFuncSetAttribute(probe_S, cudaFuncAttributeMaxDynamicSharedMemorySize, 240 * 32 * 8);
    probe_S<<<blocks, threads, 240 * 32 * 8>>>(ops, out, reps);
    return (int)cudaGetLastError();
}
"""

KERNEL_T = r"""
extern "C" __global__ void __launch_bounds__(128 * WQ, 1) probe_T(const double *ops, double *out, int reps) {
    __shared__ uint32_t slot;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&slot, 512);
    if (threadIdx.x == 0) g_zero = 0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = slot + ((uint32_t)(32 * (warp & 3)) << 16);
    if (warp < 4) {
        for (int op = 0; op < 240; ++op) {
            const double v = ops[op * 32 + lane];
            st_x2(tb + 2 * op, (uint32_t)__double2loint(v), (uint32_t)__double2hiint(v));
        }
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    double *o = out + ((size_t)(blockIdx.x * 4 * WQ + warp) * 24) * 32 + lane;
    for (int r = 0; r < reps; ++r) {
        double a[NCH] = {0};
        if (warp < 4) { _Pragma("unroll 1") for (int b = 0; b < NBLK; ++b) { body_T(tb, a); st_x2(tb + 500, 0u, 0u); } }
#if WQ > 1
        else if (warp < 8) { _Pragma("unroll 1") for (int b = 0; b < NBLK; ++b) { body_T1(tb, a); st_x2(tb + 500, 0u, 0u); } }
#endif
#if WQ > 2
        else { _Pragma("unroll 1") for (int b = 0; b < NBLK; ++b) { body_T2(tb, a); st_x2(tb + 500, 0u, 0u); } }
#endif
#pragma unroll
        for (int k = 0; k < NCH; ++k) stg(o + 32 * k, a[k]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(slot, 512);
}
extern "C" int launch_T(const double *ops, double *out, int blocks, int threads, int reps) {
    probe_T<<<blocks, 128 * WQ>>>(ops, out, reps);
    return (int)cudaGetLastError();
}
"""

# name -> (src, R, sync_every / seg)
VARIANTS = {
    "T_r56_seg32_cb": ("T", 56, 32),
    "T_g2_r40_seg16_cb": ("T", 40, 16),
    "T_g2_r32_seg16": ("T", 32, 16),
    "T_g2_r32_seg16_wq2": ("T", 32, 16),
    "T_g2_r32_seg16_wq3": ("T", 32, 16),
    "T_g1_r24_seg16_wq2": ("T", 24, 16),
    "T_g4_r40_seg16_wq2": ("T", 40, 16),
    "T_g4_r48_seg16": ("T", 48, 16),
    "S_g2_r32_warp16": ("S", 32, -16),
}


def gen():
    global CONST_CF
    poly = inputs.c5_poly()
    P, Q, Cf = poly.p, poly.q, poly.coef
    info = {}
    for name, (src, R, x) in VARIANTS.items():
        global CHAINS
        CONST_CF = name.endswith("_cb")
        G = int(name.split("_g")[1].split("_")[0]) if "_g" in name else 24
        WQ = int(name.split("_wq")[1].split("_")[0]) if "_wq" in name else 1
        body = []
        for b in range(WQ):
            CHAINS = list(range(b * G, (b + 1) * G))
            order = interleave(P, Q, R)
            ev, loads = belady(P, Q, order, R)
            body += gen_body_S(ev, Cf, x) if src == "S" else gen_body_T(ev, Cf, x, "body_T" + (str(b) if b else ""))
        cb = "__constant__ double CF[1536] = {" + ", ".join(repr(float(v)) for v in Cf.reshape(-1)) + "};\n"
        text = HEADER + f"#define NBLK {24 // (G * WQ)}\n#define NCH {G}\n#define WQ {WQ}\n" + cb + "\n".join(body) + "\n" + (KERNEL_S if src == "S" else KERNEL_T)
        cu = CSRC / f"jitprobe_{name}.cu"
        cu.write_text(text)
        so = OUT / f"libjitprobe_{name}.so"
        r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false", "-Xptxas", "-v",
                            "-shared", "-Xcompiler", "-fPIC", str(cu), "-o", str(so)], capture_output=True, text=True)
        regs = [l.strip() for l in r.stderr.splitlines() if "registers" in l or "spill" in l]
        info[name] = {"rc": r.returncode, "loads_per_point": loads, "ptxas": regs}
        print(name, info[name], flush=True)
        if r.returncode:
            print(r.stderr[-3000:])
    (OUT / "jitprobe_gen.json").write_text(json.dumps(info, indent=1))


def run():
    import torch
    poly = inputs.c5_poly()
    rng = np.random.default_rng(3)
    ops = rng.uniform(0.9, 1.1, (NIN, 32))
    want = np.empty((NO, 32))
    for o in range(NO):
        acc = (poly.coef[o, 0] * ops[poly.p[o, 0]]) * ops[poly.q[o, 0]]
        for t in range(1, NT):
            acc = acc + (poly.coef[o, t] * ops[poly.p[o, t]]) * ops[poly.q[o, t]]
        want[o] = acc
    d_ops = torch.from_numpy(ops).cuda()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    gen_info = json.loads((OUT / "jitprobe_gen.json").read_text())
    res = {"sm_count": sms, "fp64_ceiling_pt_terms_per_clk_sm": 18.44e12 / 3 / sms / 1.965e9}
    for name, (src, R, x) in VARIANTS.items():
        lib = C.CDLL(str(OUT / f"libjitprobe_{name}.so"))
        fn = getattr(lib, f"launch_{src}")
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int]
        WQ = int(name.split("_wq")[1].split("_")[0]) if "_wq" in name else 1
        for nw in ((4, 8, 12) if src == "S" else (4 * WQ,)):
            out = torch.zeros((sms * nw, NO, 32), dtype=torch.float64, device="cuda")
            reps = 16
            assert fn(d_ops.data_ptr(), out.data_ptr(), sms, nw * 32, reps) == 0
            torch.cuda.synchronize()
            got = out.cpu().numpy()
            G = int(name.split("_g")[1].split("_")[0]) if "_g" in name else 24
            ok = all(got[w][:G].tobytes() == want[:G].tobytes() for w in (0, nw - 1, sms * nw - 1))
            for _ in range(2):
                fn(d_ops.data_ptr(), out.data_ptr(), sms, nw * 32, reps)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            n = 5
            for _ in range(n):
                fn(d_ops.data_ptr(), out.data_ptr(), sms, nw * 32, reps)
            ev[1].record()
            torch.cuda.synchronize()
            s = ev[0].elapsed_time(ev[1]) / n * 1e-3
            pt_terms = sms * nw * 32 * reps * NO * NT
            res[f"{name}_w{nw}"] = {"bits_ok": ok, "ms": s * 1e3,
                                    "pt_terms_per_clk_sm_at_1965": pt_terms / s / sms / 1.965e9,
                                    "loads_per_point": gen_info[name]["loads_per_point"],
                                    "ptxas": gen_info[name]["ptxas"]}
            print(name, nw, res[f"{name}_w{nw}"], flush=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    gen() if sys.argv[1] == "gen" else run()
