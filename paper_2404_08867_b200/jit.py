"""Expression -> CUDA source for NVRTC (the lowering step before the path,
SURVEY.md §8(f) item 1).

An integrand outside the closed families becomes straight-line device code in
the reference's evaluation order (sums ``v = const; v = v + c*t``, products
``v = coeff; v = v*f``, /root/reference/pkg/src/latquad/exprcore.py:442-480),
with every constant as an exact hex literal and every coordinate formed once
per point -- for expressions of at most STEP_MAX_VARS coordinates by stepping
its residue from the thread's previous point (r + z_j mod n) instead of a
modular product, the same integer either way.  liblq compiles it for sm_100a
(``lq_jit_create``) and launches it over a resident grid with the same tiles
and fixed reduction tree as the bytecode interpreter it replaces, so the two
agree to rounding and the JIT is purely a speed-up.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import _native as N
from .expr import topo

__all__ = ["source_for", "compile_expr", "jit_wanted", "JIT_THRESHOLD"]

_PRELUDE = r"""
typedef unsigned int u32;
typedef unsigned long long u64;
typedef long long i64;
struct LqZZ { u32 z, zs; };

__device__ __forceinline__ double lq_exact_div(double a, double b, double inv) {
    double q = a * inv;
    double e = fma(-q, b, a);
    return fma(e, inv, q);
}
__device__ __forceinline__ u32 lq_shoup(u32 x, u32 z, u32 zs, u32 n) {
    u32 q = __umulhi(x, zs);
    u32 r = x * z - q * n;
    u32 t = r - n;
    return t < r ? t : r;
}
__device__ __forceinline__ u64 lq_mulmod64(u64 a, u64 b, u64 n, double ninv) {
    u64 lo = a * b;
    double qd = (double)a * (double)b * ninv;
    u64 q = qd <= 0.0 ? 0ull : (u64)qd;
    i64 r = (i64)(lo - q * n);
    while (r < 0) r += (i64)n;
    while (r >= (i64)n) r -= (i64)n;
    return (u64)r;
}
__device__ __forceinline__ double lq_block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < 8 ? sh[lane] : 0.0;
        for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}
__device__ __forceinline__ double lq_ipow(double b, int k) { return k == 2 ? b * b : pow(b, (double)k); }

struct LqLat32 {
    u32 i, n; double nd, inv; const LqZZ* zz;
    __device__ __forceinline__ double operator()(int j) const {
        const LqZZ t = zz[j];
        return lq_exact_div((double)lq_shoup(i, t.z, t.zs, n), nd, inv);
    }
};
struct LqLat64 {
    u64 i, n; double nd, inv; const u64* z;
    __device__ __forceinline__ double operator()(int j) const {
        return lq_exact_div((double)lq_mulmod64(i, __ldg(z + j), n, inv), nd, inv);
    }
};
struct LqArr {
    const double* v;
    __device__ __forceinline__ double operator()(int k) const { return v[k]; }
};
struct LqTen {
    const double* nodes; const i64* off; const u32* digit;
    __device__ __forceinline__ double operator()(int j) const { return __ldg(nodes + off[j] + digit[j]); }
};
"""

_KERNELS = r"""
// (r + b) mod n for an integer r in [0, n) and bm = b - n with b in [0, n),
// n < 2^53, all exact doubles: r + bm is exact and lies in [-n, n); the sign
// bit (high word) says whether n goes back on.  r + bm == 0 rounds to +0.0.
__device__ __forceinline__ double lq_addmod_d(double r, double bm, double nd) {
    const double t = r + bm;
    return __double2hiint(t) < 0 ? t + nd : t;
}

// plain lattice sum: 256 threads x 16 consecutive points per tile (the
// interpreter's tiling, so the tile partials line up with k_prog_lattice);
// CTAs stride over the tiles
extern "C" __global__ void __launch_bounds__(256) lq_jit_lattice(const void* zt, u64 n, double nd, double inv,
                                                                u64 base, u64 end, int wide, double* tile_out,
                                                                i64 ntiles) {
    __shared__ double sh[8];
#ifdef LQ_STEP
    // the coordinates a point uses are stepped from point to point of the
    // thread's run, r_k(i + 1) = r_k(i) + z_k mod n, and from one tile of the
    // CTA to its next by jump_k = (G 4096 - 16) z_k mod n, each fed to the same
    // exactly rounded division -- the coordinates, and so the sums, are those
    // of the per-point products.  The residues are integers below n < 2^53 and
    // are carried as exact doubles: one add of z_k - n, a sign test on the
    // high word and a conditional add of n per coordinate, with no integer
    // carry chain and no int -> double conversion (issue-bound before:
    // profiles/r02_jit_lattice_step.md)
    __shared__ double jmn[LQ_NU];
    const u64 gap = (u64)gridDim.x * 4096ull - 16ull;
    if (threadIdx.x < LQ_NU) {
        const int j = lq_use[threadIdx.x];
        const u64 jump = wide ? lq_mulmod64(gap % n, ((const u64*)zt)[j], n, inv)
                              : (gap % n) * (u64)((const LqZZ*)zt)[j].z % n;
        jmn[threadIdx.x] = (double)jump - nd;
    }
    __syncthreads();
    const u64 i00 = base + (u64)blockIdx.x * 4096ull + (u64)threadIdx.x * 16ull;
    double r[LQ_NU], zmn[LQ_NU];
    if (wide) {
        const u64* z = (const u64*)zt;
        const u64 im = i00 < n ? i00 : i00 % n;
#pragma unroll
        for (int k = 0; k < LQ_NU; ++k) {
            const u64 zk = __ldg(z + lq_use[k]);
            r[k] = (double)lq_mulmod64(im, zk, n, inv);
            zmn[k] = (double)zk - nd;
        }
    } else {
        const LqZZ* zz = (const LqZZ*)zt;
#pragma unroll
        for (int k = 0; k < LQ_NU; ++k) {
            const LqZZ t = zz[lq_use[k]];
            r[k] = (double)lq_shoup((u32)i00, t.z, t.zs, (u32)n);
            zmn[k] = (double)t.z - nd;
        }
    }
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const u64 i0 = base + (u64)tile * 4096ull + (u64)threadIdx.x * 16ull;
        double s = 0.0;
        for (int p = 0; p < 16; ++p) {
            if (i0 + p < end) {
                double xv[LQ_NU];
#pragma unroll
                for (int k = 0; k < LQ_NU; ++k) xv[k] = lq_exact_div(r[k], nd, inv);
                s += lq_fc(LqArr{xv});
            }
#pragma unroll
            for (int k = 0; k < LQ_NU; ++k) r[k] = lq_addmod_d(r[k], zmn[k], nd);
        }
        s = lq_block_sum(s, sh);
        if (threadIdx.x == 0) tile_out[tile] = s;
#pragma unroll
        for (int k = 0; k < LQ_NU; ++k) r[k] = lq_addmod_d(r[k], jmn[k], nd);
    }
#else
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const u64 i0 = base + (u64)tile * 4096ull + (u64)threadIdx.x * 16ull;
        double s = 0.0;
        for (int p = 0; p < 16; ++p) {
            const u64 i = i0 + p;
            if (i < end) {
                if (wide) {
                    LqLat64 x{i < n ? i : i % n, n, nd, inv, (const u64*)zt};
                    s += lq_f(x);
                } else {
                    LqLat32 x{(u32)i, (u32)n, nd, inv, (const LqZZ*)zt};
                    s += lq_f(x);
                }
            }
        }
        s = lq_block_sum(s, sh);
        if (threadIdx.x == 0) tile_out[tile] = s;
    }
#endif
}

// direct tensor-grid sum, flat index first axis fastest: an odometer per
// thread, set up once by division and carried from one tile of the CTA to its
// next by adding the mixed-radix digits of G 4096 - 16
extern "C" __global__ void __launch_bounds__(256) lq_jit_tensor(int d, const i64* counts, const i64* off,
                                                               const double* nodes, u64 base, u64 end,
                                                               double* tile_out, i64 ntiles) {
    __shared__ double sh[8];
    __shared__ u32 gapd[LQ_AXES];
    if (threadIdx.x == 0) {
        u64 rem = (u64)gridDim.x * 4096ull - 16ull;
        for (int k = 0; k < d; ++k) {
            const u64 c = (u64)counts[k];
            gapd[k] = (u32)(rem % c);
            rem /= c;
        }
    }
    __syncthreads();
    u32 digit[LQ_AXES];
    {
        u64 rem = base + (u64)blockIdx.x * 4096ull + (u64)threadIdx.x * 16ull;
        for (int k = 0; k < d; ++k) {
            const u64 c = (u64)counts[k];
            digit[k] = (u32)(rem % c);
            rem /= c;
        }
    }
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const u64 s0 = base + (u64)tile * 4096ull + (u64)threadIdx.x * 16ull;
        double s = 0.0;
#ifdef LQ_STEP
        // the used axes' node values stay in registers: a step of the first
        // axis re-reads one node, a carry re-reads them all -- same nodes
        double xv[LQ_NU];
#pragma unroll
        for (int k = 0; k < LQ_NU; ++k) xv[k] = __ldg(nodes + off[lq_use[k]] + digit[lq_use[k]]);
        const u32 c0 = (u32)counts[0];
        const double* node0 = nodes + off[0];
        for (int p = 0; p < 16; ++p) {
            if (s0 + p < end) s += lq_fc(LqArr{xv});
            if (++digit[0] < c0) {
                if (lq_use[0] == 0) xv[0] = __ldg(node0 + digit[0]);
            } else {
                digit[0] = 0;
                for (int k = 1; k < d; ++k) {
                    if (++digit[k] < (u64)counts[k]) break;
                    digit[k] = 0;
                }
#pragma unroll
                for (int k = 0; k < LQ_NU; ++k) xv[k] = __ldg(nodes + off[lq_use[k]] + digit[lq_use[k]]);
            }
        }
#else
        LqTen x{nodes, off, digit};
        for (int p = 0; p < 16; ++p) {
            if (s0 + p < end) s += lq_f(x);
            for (int k = 0; k < d; ++k) {
                if (++digit[k] < (u64)counts[k]) break;
                digit[k] = 0;
            }
        }
#endif
        s = lq_block_sum(s, sh);
        if (threadIdx.x == 0) tile_out[tile] = s;
        u32 carry = 0;
        for (int k = 0; k < d; ++k) {
            const u64 c = (u64)counts[k];
            u64 t = (u64)digit[k] + gapd[k] + carry;
            carry = t >= c;
            digit[k] = (u32)(carry ? t - c : t);
        }
    }
}
"""


def _lit(v):
    v = float(v)
    if v != v or v in (float("inf"), float("-inf")):
        return {"inf": "(1.0/0.0)", "-inf": "(-1.0/0.0)"}.get(repr(v), "(0.0/0.0)")
    return v.hex()


# stepped coordinates in the lattice kernel for expressions of at most this
# many distinct coordinates (their residues live in registers)
STEP_MAX_VARS = 24


def source_for(e, var_map=None, n_axes=1):
    """CUDA source of an expression: ``lq_f(x)`` (coordinates by index),
    ``lq_fc(x)`` (coordinates by their rank among the used ones, for the
    stepped lattice kernel) plus both kernel bodies."""
    vm = var_map if var_map is not None else (lambda j: j - 1)
    order = list(topo(e))
    uses = sorted({vm(node.idx) for node in order if node.op == "var"})
    body = _body(order, e, vm)
    src = _PRELUDE + (f"template <class X> __device__ __forceinline__ double lq_f(const X& x) {{\n{body}\n}}\n")
    if 0 < len(uses) <= STEP_MAX_VARS:
        rank = {j: k for k, j in enumerate(uses)}
        bodyc = _body(order, e, lambda j: rank[vm(j)])
        src += (f"template <class X> __device__ __forceinline__ double lq_fc(const X& x) {{\n{bodyc}\n}}\n"
                f"#define LQ_STEP 1\n#define LQ_NU {len(uses)}\n"
                f"__constant__ int lq_use[LQ_NU] = {{{', '.join(str(j) for j in uses)}}};\n")
    return src + f"#define LQ_AXES {max(1, int(n_axes))}\n" + _KERNELS


def _body(order, e, vm):
    names = {}
    lines = []
    for k, node in enumerate(order):
        t = f"t{k}"
        names[node] = t
        op = node.op
        if op == "const":
            lines.append(f"    const double {t} = {_lit(node.val)};")
        elif op == "var":
            lines.append(f"    const double {t} = x({vm(node.idx)});")
        elif op == "add":
            lines.append(f"    double {t} = {_lit(node.val)};")
            for c, ch in node.terms:
                lines.append(f"    {t} = {t} + {_lit(c)} * {names[ch]};")
        elif op == "mul":
            lines.append(f"    double {t} = {_lit(node.val)};")
            for ch in node.args:
                lines.append(f"    {t} = {t} * {names[ch]};")
        elif op == "pow":
            b = names[node.args[0]]
            if node.idx >= 2:
                lines.append(f"    const double {t} = lq_ipow({b}, {node.idx});")
            else:
                k_ = -node.idx
                inner = b if k_ == 1 else f"lq_ipow({b}, {k_})"
                lines.append(f"    const double {t} = 1.0 / ({inner});")
        else:
            fn = {"exp": "exp", "sin": "sin", "cos": "cos", "abs": "fabs"}[op]
            lines.append(f"    const double {t} = {fn}({names[node.args[0]]});")
    lines.append(f"    return {names[e]};")
    return "\n".join(lines)


class _Module:
    def __init__(self, src):
        log = C.create_string_buffer(4096)
        h = C.c_void_p()
        N.check(N.lib().lq_jit_create(src.encode(), b"lq_jit.cu", C.byref(h), log, len(log)))
        self.handle = h

    def __del__(self):
        try:
            if self.handle:
                N.lib().lq_jit_destroy(self.handle)
        except Exception:
            pass


_cache = {}
_lock = threading.Lock()


# interpreter instruction-points above which compiling pays for itself
# (NVRTC takes ~0.3 s for a small expression; the interpreter runs ~2e9
# insn-points/s)
JIT_THRESHOLD = 1e9
# NVRTC time grows faster than quadratically with the straight-line body
# (tools/jit_compile_probe.py on the B200 box: 37/69/133/261 bytecode
# instructions -> 0.36/0.82/2.6/11.6 s; ~3000 -> 620 s), while the
# interpreter is only ~4x slower than the compiled kernel: past this size the
# interpreter always wins
JIT_MAX_INSN = 160


def jit_wanted(work, n_insn=1):
    """LQ_JIT=0 never, =always for any size; default: programs of at most
    JIT_MAX_INSN instructions whose work pays for the compile (the threshold
    grows with the square of the program length, as the compile time does)."""
    mode = os.environ.get("LQ_JIT", "auto")
    if mode == "0":
        return False
    if mode == "always":
        return True
    if n_insn > JIT_MAX_INSN:
        return False
    return work >= JIT_THRESHOLD * max(1.0, (n_insn / 32.0) ** 2)


def compile_expr(e, n_axes=1):
    """Compiled module handle (int) for e, cached per process, or None if NVRTC
    is unavailable (the bytecode interpreter then runs -- still on the GPU)."""
    key = (e, int(n_axes))
    with _lock:
        mod = _cache.get(key)
        if mod is None:
            try:
                mod = _Module(source_for(e, n_axes=n_axes))
            except N.NativeUnavailable:
                mod = False
            except NotImplementedError:
                mod = False
            _cache[key] = mod
    return mod.handle.value if mod else None
