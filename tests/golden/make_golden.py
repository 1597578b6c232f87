"""Regenerate tests/golden/golden.json from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libgapref.so, compiled from
/root/reference/proj/include by oracle/Makefile):

    python tests/golden/make_golden.py

Everything recorded comes from the reference's own code paths --
GenerateKronecker/GenerateUniform, BuildCsr, PickSources, detail::BfsDepths,
Bfs/VerifyBfs and its detail:: step functions (via gkr_bfs_schedule) --
except the two NEW generators the BASELINE configs require and the reference
lacks (the seeded ID permutation and the road-like grid), whose edge lists
come from the C restatement in oracle/gk_oracle.c; their CSR is still built
by the reference BuildCsr.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

SEED = 24601


def fnv(a) -> str:
    return f"{O.fnv1a(np.ascontiguousarray(a)):016x}"


def small(pairs, n):
    e = np.array([x for p in pairs for x in p], np.uint32)
    return n, e


def cases(R: O.RefLib):
    out = {}
    out["path8"] = ("edges", *small([(v, v + 1) for v in range(7)], 8), False)
    out["star9"] = ("edges", *small([(4, v) for v in range(9) if v != 4], 9), False)
    out["ring16"] = ("edges", *small([(v, (v + 1) % 16) for v in range(16)], 16), False)
    out["k5"] = ("edges", *small([(u, v) for u in range(5) for v in range(u + 1, 5)], 5), False)
    out["kron10"] = ("kron", 1 << 10, R.gen("kron", 10, 16, SEED), False)
    out["urand10"] = ("urand", 1 << 10, R.gen("urand", 10, 16, SEED), False)
    out["kron12_s7"] = ("kron", 1 << 12, R.gen("kron", 12, 16, 7), False)
    out["urand14"] = ("urand", 1 << 14, R.gen("urand", 14, 16, SEED), False)
    # config 1: Kronecker scale 16, edge factor 16, permuted IDs
    out["kron16p"] = ("kronp", 1 << 16, O.permute_edges(R.gen("kron", 16, 16, SEED), 16, SEED), False)
    out["grid60x70"] = ("grid", 60 * 70, O.gen_grid(60, 70, 0.15, 0.02, SEED), False)
    # bfs.hpp bottom-up on in-edges of a directed graph (test_kernels_source.cc:55-67)
    out["dkron10_s11"] = ("kron", 1 << 10, R.gen("kron", 10, 16, 11), True)
    return out


def main():
    R = O.RefLib()
    gold = {"seed": SEED, "graphs": {}, "kat": {}}
    for name, (kind, n, edges, directed) in cases(R).items():
        g = R.build(n, edges, directed=directed, symmetrize=not directed)
        csr = g.csr()
        ent = {"kind": kind, "n": int(n), "m": int(g.m), "directed": bool(directed),
               "edges_fnv": fnv(edges), "off_fnv": fnv(csr.off), "nb_fnv": fnv(csr.nb)}
        if directed:
            ent["in_off_fnv"] = fnv(csr.in_off)
            ent["in_nb_fnv"] = fnv(csr.in_nb)
        srcs = g.pick_sources(64, SEED)
        ent["sources"] = [int(s) for s in srcs]
        runs = []
        ab = [(1, 1)] if directed else [(15, 18)]
        for s in srcs[:8]:
            d = g.depths(int(s))
            for alpha, beta in ab:
                for strat in (0, 1, 2):
                    sch = g.schedule(int(s), alpha, beta, strat)
                    ok, msg = g.verify(int(s), sch.parent)
                    assert ok, (name, s, msg)
                    p = g.bfs(int(s), alpha, beta, strat)
                    ok, msg = g.verify(int(s), p)
                    assert ok, (name, s, msg)
                    runs.append({"source": int(s), "alpha": alpha, "beta": beta, "strategy": strat,
                                 "depth_fnv": fnv(d), "reached": int((d >= 0).sum()), "max_depth": int(d.max()),
                                 "dirs": sch.dirs, "frontier": sch.frontier, "result": sch.result,
                                 "edges_to_check": sch.edges_to_check})
        ent["runs"] = runs
        gold["graphs"][name] = ent
        print(name, n, g.m, len(runs), runs[0]["dirs"] if runs else "")
    # known answers (test_kernels_source.cc:13-23)
    g = R.build(3, np.array([0, 1, 1, 2], np.uint32))
    gold["kat"]["path3_parent"] = [int(x) for x in g.bfs(0)]
    g = R.build(4, np.array([0, 1, 1, 2], np.uint32))
    gold["kat"]["isolated_parent"] = [int(x) for x in g.bfs(0)]
    gold["kat"]["perm_scale16_first8"] = [O.permute(v, 16, SEED) for v in range(8)]
    gold["kat"]["perm_keys_s16"] = [f"{int(k):016x}" for k in O.perm_keys(SEED, 16)]
    # Brandes betweenness (betweenness.hpp:84-145) from the reference; the
    # graphs of test_kernels_source.cc:136-180 plus kron10/urand10
    gold["bc"] = {}
    bc_cases = {
        "star5": (R.build(5, np.array([x for v in range(4) for x in (4, v)], np.uint32)), [0, 1, 2, 3, 4]),
        "path2": (R.build(2, np.array([0, 1], np.uint32)), [0]),
    }
    for nm, kind, scale, seed, directed in (("kron10", "kron", 10, SEED, False), ("urand10", "urand", 10, SEED, False),
                                            ("dkron9_s13", "kron", 9, 13, True)):
        g = R.build(1 << scale, R.gen(kind, scale, 16, seed), directed=directed, symmetrize=not directed)
        bc_cases[nm] = (g, [int(x) for x in g.pick_sources(4, SEED)])
    for nm, (g, srcs) in bc_cases.items():
        sc = g.brandes(srcs)
        ok, msg = g.verify_bc(srcs, sc)
        assert ok, (nm, msg)
        gold["bc"][nm] = {"sources": [int(x) for x in srcs], "scores": [float(x) for x in sc],
                          "directed": bool(g.directed)}
    # .sg fixtures written by the reference's WriteSerialized (io.hpp:364-389)
    gdir = os.path.dirname(os.path.abspath(__file__))
    R.build(2, np.array([0, 1], np.uint32), directed=True, symmetrize=False).write_sg(
        os.path.join(gdir, "directed_1edge.sg"))  # test_io.cc:174-203's golden graph
    kg = R.build(1 << 10, R.gen("kron", 10, 16, SEED))
    kg.write_sg(os.path.join(gdir, "kron10.sg"))
    kg.write_sg(os.path.join(gdir, "kron10.wsg"), SEED)
    R.build(1 << 9, R.gen("kron", 9, 8, 5), directed=True, symmetrize=False).write_sg(
        os.path.join(gdir, "dkron9.sg"))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
