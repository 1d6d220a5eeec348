#!/usr/bin/env python
"""Generate paper_2401_16543_b200/csrc/kfvm_gen.cuh — fully unrolled sparse
stencil contractions of the KFVM-WENO reconstruction for (dim, R) in
{(2,2), (2,3), (3,2)}.

The generated code is the device form of the oracle's weno_field
(oracle/kfvm_oracle.cpp): for every (sub)stencil q it evaluates the n_alpha
derivative dot products (beta_q), the nonlinear weights
and, for every face point s, the WENO-AO combination of the per-stencil point
values, each dot product accumulated in stencil order from 0.0 with
explicit fma — the pinned FP contract.  Because the gather pattern is known at
compile time, the stencil values live in registers and every weight is a
__constant__ operand with a literal offset (DFMA R, R, c[bank][imm], R): the
inner loop issues nothing but DFMAs.

Only the sparsity structure is generated (it follows from the stencil
geometry, proj/core/src/geometry.cpp:10-34 and PAPER.md §3.1); the weight
values are uploaded at run time from the binary128 table, and
kfvm_gpu_create checks the table's gather/offset arrays against the
structure compiled in here.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2401_16543_b200", "csrc", "kfvm_gen.cuh")

CASES = [(2, 2), (2, 3), (3, 2), (3, 3)]
# (3,3): structure only — its 198 KB of weights exceed __constant__ and its
# unrolled contractions (25k fma per variable) would not fit the I-cache
UNROLLED = {(2, 2), (2, 3), (3, 2)}


def full_stencil(dim, R):
    kr = R if dim == 3 else 0
    out = []
    for k in range(-kr, kr + 1):
        for j in range(-R, R + 1):
            for i in range(-R, R + 1):
                if i * i + j * j + k * k <= R * R:
                    out.append((i, j, k))
    return out


def in_sub(dim, R, q, o):
    if q == 1:
        return sum(c * c for c in o) <= (R - 1) ** 2
    axis = (q - 2) // 2
    sgn = -1 if (q - 2) % 2 else 1
    a = sgn * o[axis]
    return all(abs(o[t]) <= a for t in range(dim) if t != axis)


def graded(dim, lo, hi):
    out = []
    for n in range(lo, hi + 1):
        if dim == 2:
            out += [(n - k, k, 0) for k in range(n + 1)]
        else:
            for a in range(n, -1, -1):
                for b in range(n - a, -1, -1):
                    out.append((a, b, n - a - b))
    return out


def gen_case(dim, R):
    full = full_stencil(dim, R)
    ns = 2 * dim + 2
    members = [list(range(len(full)))]
    for q in range(1, ns):
        members.append([h for h, o in enumerate(full) if in_sub(dim, R, q, o)])
    sizes = [len(m) for m in members]
    offs, acc = [], 0
    for n in sizes:
        offs.append(acc)
        acc += n
    total = acc
    na = len(graded(dim, 1, R))
    npnt = 2 * dim * R ** (dim - 1)
    tag = f"{dim}{R}"
    L = []
    L.append(f"// ---- dim={dim} R={R}: N0={len(full)} sizes={sizes} n_alpha={na} n_points={npnt}")
    unrolled = (dim, R) in UNROLLED
    if unrolled:
        L.append(f"__constant__ __align__(16) double c_f{tag}[{total * npnt}];  // table.face transposed, [q][h][s]")
        L.append(f"__constant__ __align__(16) double c_d{tag}[{total * na}];  // table.deriv, [q][a][h]")
    L.append(f"template <> struct Gen<{dim}, {R}> {{")
    L.append(f"  static constexpr int N0 = {len(full)}, NP = {npnt}, NA = {na}, NS = {ns}, NTOT = {total};")
    L.append(f"  static constexpr int OFF[{len(full)}][3] = {{" +
             ", ".join("{%d, %d, %d}" % o for o in full) + "};")
    L.append("  __host__ __device__ static constexpr int off(int h, int a) {")
    L.append(f"    constexpr int T[{len(full)}][3] = {{" + ", ".join("{%d, %d, %d}" % o for o in full) + "};")
    L.append("    return T[h][a];")
    L.append("  }")
    flat = [h for m in members for h in m]
    L.append(f"  static constexpr int GATHER[{total}] = {{" + ", ".join(map(str, flat)) + "};")
    # sizes as constexpr functions (usable in device code after unrolling)
    L.append("  __host__ __device__ static constexpr int qsize(int q) {")
    L.append("    return " + " : ".join(f"q == {q} ? {sizes[q]}" for q in range(ns - 1)) + f" : {sizes[-1]};")
    L.append("  }")
    L.append("  __host__ __device__ static constexpr int kc(int q) { return (qsize(q) + 3) / 4; }")
    L.append("  __host__ __device__ static constexpr int cbase(int q) { return q == 0 ? 0 : cbase(q - 1) + kc(q - 1); }")
    L.append(f"  static constexpr int NCHUNK = {sum((n + 3) // 4 for n in sizes)};")
    L.append(f"  static constexpr bool UNROLLED = {'true' if unrolled else 'false'};")
    if not unrolled:
        L.append("};")
        return "\n".join(L)
    L.append("  static const void* face_symbol() { return (const void*)&c_f%s; }" % tag)
    L.append("  static const void* deriv_symbol() { return (const void*)&c_d%s; }" % tag)
    # WENO body, fully unrolled: stencil values in registers, every weight a
    # __constant__ operand with a literal offset (table layouts [q][a][h] and
    # [q][s][h]); each dot product is the stencil-order fma chain from 0.0.
    L.append("  // beta_q, omega_q, WENO-AO values of one scalar field g on S0")
    L.append("  static __device__ __forceinline__ void weno(const double (&g)[%d], double (&w)[%d],"
             % (len(full), npnt))
    L.append("                                              const double* __restrict__ sc,")
    L.append("                                              const double* __restrict__ gam, double eps,")
    L.append("                                              double inv_g0) {")
    for q in range(ns):
        m, N, o = members[q], sizes[q], offs[q]
        # beta: four interleaved partials, alpha = 8n + 2j + e -> partial j,
        # combined as (b0 + b1) + (b2 + b3) (oracle weno_field)
        L.append(f"    double wt{q};")
        L.append("    {")
        L.append("      double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;")
        # 3-D tail alphas (>= 8 floor(na/8)): four slot chains, entry hh in
        # slot (hh + pad) % 4, combined (s0 + s1) + (s2 + s3) (oracle weno_field)
        a_tail = 8 * (na // 8) if dim == 3 else na
        pad = (4 - N % 4) % 4
        for a in range(na):
            base = o * na + a * N
            L.append("      {")
            if a < a_tail:
                L.append("        double d = 0.0;")
                for hh, h in enumerate(m):
                    L.append(f"        d = fma(c_d{tag}[{base + hh}], g[{h}], d);")
            else:
                L.append("        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;")
                for hh, h in enumerate(m):
                    L.append(f"        s{(hh + pad) % 4} = fma(c_d{tag}[{base + hh}], g[{h}], s{(hh + pad) % 4});")
                L.append("        const double d = (s0 + s1) + (s2 + s3);")
            j = (a & 7) >> 1
            L.append(f"        b{j} = fma(sc[{a}], d * d, b{j});")
            L.append("      }")
        L.append("      const double b = (b0 + b1) + (b2 + b3);")
        L.append(f"      wt{q} = gam[{q}] * (1.0 / fma(b, b, eps));")
        L.append("    }")
    L.append("    double sum = wt0;")
    for q in range(1, ns):
        L.append(f"    sum = sum + wt{q};")
    L.append("    const double inv_sum = 1.0 / sum;")
    for q in range(ns):
        L.append(f"    const double om{q} = wt{q} * inv_sum;")
    L.append("    const double c0 = om0 * inv_g0;")
    for q in range(1, ns):
        L.append(f"    const double c{q} = fma(-c0, gam[{q}], om{q});")
    # face points: one chain per point over every stencil entry, the entry
    # scaled by its stencil's coefficient (oracle weno_field); c_f is the
    # face table transposed to [q][h][s] so the point weights of one entry
    # are adjacent (paired uniform loads)
    for s_ in range(npnt):
        L.append(f"    w[{s_}] = 0.0;")
    for q in range(ns):
        m, N, o = members[q], sizes[q], offs[q]
        for hh, h in enumerate(m):
            L.append("    {")
            L.append(f"      const double cg = c{q} * g[{h}];")
            for s_ in range(npnt):
                L.append(f"      w[{s_}] = fma(c_f{tag}[{(o + hh) * npnt + s_}], cg, w[{s_}]);")
            L.append("    }")
    L.append("  }")
    # KXRCF pass 1: unlimited full-stencil r_0 values (stencil 0 = the first
    # block of the transposed face table), stencil-order chains per point
    L.append("  // KXRCF pass 1 (S:565): r_0(s) . u over S_0 for one scalar field")
    L.append("  static __device__ __forceinline__ void pass1(const double (&u)[%d], double (&w)[%d]) {"
             % (len(full), npnt))
    for s_ in range(npnt):
        L.append(f"    w[{s_}] = 0.0;")
    for h in range(len(full)):
        for s_ in range(npnt):
            L.append(f"    w[{s_}] = fma(c_f{tag}[{h * npnt + s_}], u[{h}], w[{s_}]);")
    L.append("  }")
    L.append("};")
    return "\n".join(L)


def main():
    parts = [
        "// AUTO-GENERATED by tools/gen_kernels.py — do not edit by hand.",
        "// Unrolled sparse stencil contractions (see the generator's docstring).",
        "#ifndef KFVM_GEN_CUH_",
        "#define KFVM_GEN_CUH_",
        "namespace kfvm_b200 {",
        "template <int D, int R> struct Gen;",
    ]
    for d, r in CASES:
        parts.append(gen_case(d, r))
    parts += ["}  // namespace kfvm_b200", "#endif", ""]
    src = "\n".join(parts)
    if os.path.exists(OUT) and open(OUT).read() == src:
        return
    with open(OUT, "w") as f:
        f.write(src)


if __name__ == "__main__":
    main()
