"""TEST INFRASTRUCTURE — a numpy executor for the engine's host plan.

Runs the matvec exactly as the GPU kernels do (phase-1 items -> spos/partials
-> reduce -> proxy solves -> phase-2 leaf tiles), but in numpy, from a
`paper_2307_16303_b200.h3d.Plan` and factors derived from the oracle's ACA
(pivots + packed LU, the reference's representation). This verifies the
planner's shard ownership, pair selection, layout, spos mapping, partial
reductions, proxy segments and solve directions on CPU.
"""
import numpy as np


def kernel_matrix(kind, A, B):
    d = A[:, None, :] - B[None, :, :]
    r2 = np.einsum("ijk,ijk->ij", d, d)
    with np.errstate(divide="ignore", over="ignore", invalid="ignore"):
        if kind == "laplace3d":
            return 1.0 / np.sqrt(r2)
        if kind == "r4":
            return 1.0 / (r2 * r2)
        r = np.sqrt(r2)
        return np.cos(r) / r


def oracle_inputs(oracle, n, seed, n_max, eps, kind, variant="hodlr3d"):
    pts = oracle.generate_points(n, seed)
    orep = oracle.initialize(pts, kind, n_max=n_max, eps=eps, variant=variant)
    L = orep.depth
    offsets = [orep.offsets(l) for l in range(L + 1)]
    lists = [None] + [[orep.list(l, k) for k in range(4)] for l in range(1, L + 1)]
    pairs = {}
    for l in range(1, L + 1):
        t, s, r = orep.lr_blocks(l)
        for k in range(len(t)):
            if t[k] < s[k]:
                pairs[(l, int(t[k]), int(s[k]))] = orep.lr_block_detail(l, k, int(r[k]))
    perm = orep.perm()
    return dict(pts=pts, orep=orep, L=L, offsets=offsets, lists=lists, pairs=pairs, perm=perm,
                ppts=pts[perm])


TILE_R, TILE_C = 16, 64  # csrc/planner.h kTileRows / kTileCols


def tile_index(i, c, nct):
    """Offset of element (row i, column c) in a tile-major stream-level pool."""
    return ((i // TILE_R) * nct + c // TILE_C) * (TILE_R * TILE_C) + (i % TILE_R) * TILE_C + c % TILE_C


def node_matrix(W, woff, g, rows, R):
    """Row-major (rows x R) view of node g's tile-major factor pool."""
    nrp = -(-rows // TILE_R) * TILE_R
    t = W[woff: woff + nrp * R].reshape(nrp // TILE_R, R // TILE_C, TILE_R, TILE_C)
    return t.transpose(0, 2, 1, 3).reshape(nrp, R)[:rows]


def simulate(plan, inp, xp, kind, diag=0.0, modes=None):
    """Returns b in Morton order for the plan's owned rows (others zero)."""
    L, off, ppts, pd = inp["L"], inp["offsets"], inp["ppts"], inp["pairs"]
    # ranks, optional mode switches, layout
    for l in range(1, L + 1):
        X, Y = plan.pairs(l)
        plan.set_ranks(l, [len(pd[(l, int(a), int(b))][0]) for a, b in zip(X, Y)])
    if modes is not None:
        for l in range(1, L + 1):
            if modes[l] != 2 and plan.array("modes")[l] != 2:
                plan.set_mode(l, modes[l])
    plan.layout()
    md = plan.array("modes")
    sizes = plan.array("sizes")
    W = np.zeros(max(sizes[0], 1))
    S = np.zeros(max(sizes[1], 1))
    P = np.zeros(max(sizes[2], 1))
    piv = np.zeros(max(sizes[3], 1), np.int64)
    lu = np.zeros(max(sizes[4], 1))
    woff, soff, rowbeg = plan.array("woff"), plan.array("soff"), plan.array("rowbeg")
    rpad, spos, nb = plan.array("rpad"), plan.array("spos"), plan.array("node_base")
    rows = plan.array("rows")

    def pts_of(l, z):
        return ppts[off[l][z]:off[l][z + 1]]

    for l in range(1, L + 1):
        X, Y = plan.pairs(l)
        if md[l] in (0, 3, 5):
            wx, wy = plan.array("pair_wx", l), plan.array("pair_wy", l)
            rx, ry = plan.array("pair_rx", l), plan.array("pair_ry", l)
            cx, cy = plan.array("pair_cx", l), plan.array("pair_cy", l)
        if md[l] in (1, 4, 5, 6):
            po, lo = plan.array("pair_piv", l), plan.array("pair_lu", l)
        for p, (a, b) in enumerate(zip(X, Y)):
            rp, cp, LU = pd[(l, int(a), int(b))]
            r = len(rp)
            if r == 0:
                continue
            Lm = np.tril(LU, -1) + np.eye(r)
            Um = np.triu(LU)
            Xp, Yp = pts_of(l, a), pts_of(l, b)
            if md[l] in (0, 3):
                FX = np.linalg.solve(Um.T, kernel_matrix(kind, Xp, Yp[cp]).T).T  # K(X,tau) R^-1
                FY = np.linalg.solve(Lm, kernel_matrix(kind, Yp, Xp[rp]).T).T    # K(Y,sigma) L^-T
                I, Q = np.meshgrid(np.arange(len(Xp)), np.arange(r), indexing="ij")
                J, Qy = np.meshgrid(np.arange(len(Yp)), np.arange(r), indexing="ij")
                if md[l] == 0:
                    W[wx[p] + tile_index(I, cx[p] + Q, rx[p])] = FX
                    W[wy[p] + tile_index(J, cy[p] + Qy, ry[p])] = FY
                else:  # pair-major: U then V, row-major with stride rp
                    W[wx[p] + I * rx[p] + Q] = FX
                    W[wy[p] + J * ry[p] + Qy] = FY
            if md[l] == 5:
                # half level: U' = K(X, tau) (L R)^-1 explicit on X's stream
                # group; the Y side regenerated from the row pivots
                FX = np.linalg.solve((Lm @ Um).T, kernel_matrix(kind, Xp, Yp[cp]).T).T
                I, Q = np.meshgrid(np.arange(len(Xp)), np.arange(r), indexing="ij")
                W[wx[p] + tile_index(I, cx[p] + Q, rx[p])] = FX
            if md[l] in (1, 4, 5, 6):
                piv[po[p]: po[p] + r] = rp
                piv[po[p] + r: po[p] + 2 * r] = cp
            if md[l] in (1, 4, 6):  # half levels keep the pivots only
                lu[lo[p]: lo[p] + r * r] = LU.reshape(-1)
    # proxy coordinates (padding far away, weight 0)
    Q = np.full((max(sizes[1], 1), 3), 1e100)
    for sg in plan.array("proxy_segs"):
        r = int(sg["r"])
        loc = piv[sg["piv_off"] + (r if sg["side"] == 0 else 0): sg["piv_off"] + (r if sg["side"] == 0 else 0) + r]
        Q[sg["so"]: sg["so"] + r] = ppts[sg["base"] + loc]

    # ---- phase 1
    for it in plan.array("items"):
        g = int(it["node"])
        rb = rowbeg[g] + it["row0"]
        c0, nc = int(it["col0"]), int(it["ncols"])
        xs = xp[rb: rb + it["nrows"]]
        if it["kind"] == 0:
            assert it["row0"] % TILE_R == 0 and c0 % TILE_C == 0
            Wn = node_matrix(W, woff[g], g, int(rows[g]), int(rpad[g]))
            v = Wn[it["row0"]: it["row0"] + it["nrows"], c0: c0 + nc].T @ xs
        else:
            v = kernel_matrix(kind, Q[soff[g] + c0: soff[g] + c0 + nc], ppts[rb: rb + it["nrows"]]) @ xs
        if it["pslot"] < 0:
            dst = spos[soff[g] + c0: soff[g] + c0 + nc]
            ok = dst >= 0
            S[dst[ok]] = v[ok]
        else:
            P[it["pslot"]: it["pslot"] + nc] = v
    def reduce(rd):
        g, nc, k = int(rd["node"]), int(rd["ncols"]), int(rd["nchunks"])
        v = P[rd["pbase"]: rd["pbase"] + k * nc].reshape(k, nc).sum(axis=0)
        dst = spos[soff[g]: soff[g] + nc]
        ok = dst >= 0
        S[dst[ok]] = v[ok]
    reds = plan.array("reds")
    for rd in reds:
        if rd["kind"] != 5:
            reduce(rd)

    def solve_segs(which):
        for sg in plan.array("proxy_segs"):
            if sg["solve"] != which:
                continue
            r, so = int(sg["r"]), int(sg["so"])
            LU = lu[sg["lu_off"]: sg["lu_off"] + r * r].reshape(r, r)
            Lm = np.tril(LU, -1) + np.eye(r)
            Um = np.triu(LU)
            v = S[so: so + r]
            if sg["side"] == 0:
                S[so: so + r] = np.linalg.solve(Um, np.linalg.solve(Lm, v))
            else:
                S[so: so + r] = np.linalg.solve(Lm.T, np.linalg.solve(Um.T, v))
    # split levels: the Y-role weights are solved before the two-use pass
    solve_segs(2)
    # half levels, the regenerated side: both uses per entry (planner.h H2Item);
    # its t (the partners' streamed phase 1) is in S, its v feeds their phase 2
    h2 = plan.array("h2_items")
    h2b = []
    for it in h2:
        g = int(it["node"])
        R, so = int(rpad[g]), int(soff[g])
        r0 = rowbeg[g] + it["row0"]
        E = kernel_matrix(kind, ppts[r0: r0 + it["nrows"]], Q[so: so + R])
        h2b.append((int(it["slot"]), r0, int(it["nrows"]), E @ S[so: so + R], g))
        v = E.T @ xp[r0: r0 + it["nrows"]]
        if it["pslot"] >= 0:
            P[it["pslot"]: it["pslot"] + R] = v
        else:
            dst = spos[so: so + R]
            ok = dst >= 0
            S[dst[ok]] = v[ok]
    for rd in reds:
        if rd["kind"] == 5:
            reduce(rd)
    # ---- proxy solves (and the split levels' X-role ones, after the two-use pass)
    solve_segs(1)
    # ---- phase 2: near field + direct leaf blocks per owned leaf (cpart),
    # proxy / stream levels per node row chunk into one partial per level
    leaf0, leaf1, row0, row1 = plan.array("ranges")
    noff, nids = plan.array("near_off"), plan.array("near_ids")
    n = len(ppts)
    cpart = np.zeros(n)
    for X in range(leaf0, leaf1):
        xb, xe = off[L][X], off[L][X + 1]
        if xe == xb:
            continue
        T = ppts[xb:xe]
        for Y in nids[noff[X]: noff[X + 1]]:
            yb, ye = off[L][Y], off[L][Y + 1]
            K = kernel_matrix(kind, T, ppts[yb:ye])
            if Y == X:
                np.fill_diagonal(K, diag)
            cpart[xb:xe] += K @ xp[yb:ye]
    # the symmetric matrix-free lists must give the same near field: each
    # owned pair once, the partner's part through the pair buffer
    y_off, y_ids, y_cnt = plan.array("sym_off"), plan.array("sym_ids"), plan.array("sym_cnt")
    ooff, ioff, ipos = plan.array("out_off"), plan.array("in_off"), plan.array("in_pos")
    pairbuf = np.zeros(max(int(ooff[-1]), 1))
    csym = np.zeros(n)
    for X in range(leaf0, leaf1):
        xb, xe = off[L][X], off[L][X + 1]
        if xe == xb:
            continue
        ids = [int(v) for v in y_ids[y_off[X]: y_off[X + 1]]]
        assert ids[0] == X
        nsym_from = 1 + int(y_cnt[4 * X]) + int(y_cnt[4 * X + 1])
        T = ppts[xb:xe]
        pos = int(ooff[X])
        for e, Y in enumerate(ids):
            yb, ye = off[L][Y], off[L][Y + 1]
            K = kernel_matrix(kind, T, ppts[yb:ye])
            if Y == X:
                np.fill_diagonal(K, diag)
            csym[xb:xe] += K @ xp[yb:ye]
            if e >= nsym_from:
                assert row0 <= yb < row1 and Y > X
                pairbuf[pos: pos + ye - yb] = K.T @ xp[xb:xe]
                pos += ye - yb
    for Y in range(leaf0, leaf1):
        yb, ye = off[L][Y], off[L][Y + 1]
        for q in ipos[ioff[Y]: ioff[Y + 1]]:
            csym[yb:ye] += pairbuf[int(q): int(q) + ye - yb]
    np.testing.assert_allclose(csym[row0:row1], cpart[row0:row1], rtol=1e-12,
                               atol=1e-12 * (np.abs(cpart).max() + 1))
    items2 = plan.array("p2_items")
    items2s = plan.array("p2s_items")
    pgit = plan.array("pg_items")
    nslots = 1 + max([int(v) for v in items2["slot"]] + [int(v) for v in items2s["slot"]] +
                     [int(v) for v in pgit["slot"]] + [int(v) for v in h2["slot"]] + [-1])
    lvl = np.zeros((nslots, n))
    hits = np.zeros((L + 1, n), np.int64)
    shits = np.zeros((nslots, n), np.int64)
    vb = plan.array("vbase")

    def level_of(g):
        if g >= nb[-1]:  # half levels' regenerated groups (virtual node ids)
            return max(l for l in range(L + 1) if 0 <= vb[l] <= g)
        return int(np.searchsorted(nb, g, side="right")) - 1
    for it in items2:
        g = int(it["node"])
        R, so = int(rpad[g]), int(soff[g])
        assert it["nrows"] <= 256
        r0 = rowbeg[g] + it["row0"]
        lvl[it["slot"], r0: r0 + it["nrows"]] = kernel_matrix(kind, ppts[r0: r0 + it["nrows"]],
                                                              Q[so: so + R]) @ S[so: so + R]
        shits[it["slot"], r0: r0 + it["nrows"]] += 1
        if g < nb[-1]:
            hits[level_of(g), r0: r0 + it["nrows"]] += 1
    for it in items2s:
        g = int(it["node"])
        R, so = int(rpad[g]), int(soff[g])
        assert it["nrows"] <= TILE_R and it["row0"] % TILE_R == 0
        Wn = node_matrix(W, woff[g], g, int(rows[g]), R)
        r0 = rowbeg[g] + it["row0"]
        lvl[it["slot"], r0: r0 + it["nrows"]] = Wn[it["row0"]: it["row0"] + it["nrows"]] @ S[so: so + R]
        shits[it["slot"], r0: r0 + it["nrows"]] += 1
        hits[level_of(g), r0: r0 + it["nrows"]] += 1
    # pair levels: one fused pass per pair descriptor, gathered per node
    pdesc = plan.array("pair_descs")
    fdesc = plan.array("fused_descs")
    pout = np.zeros(max(int(sum(int(d["m"]) + int(d["n"]) for d in pdesc) +
                            sum(int(d["m"]) + int(d["n"]) for d in fdesc)), 1))
    for d in pdesc:
        m_, n_, rp_ = int(d["m"]), int(d["n"]), int(d["rp"])
        F = W[d["woff"]: d["woff"] + (m_ + n_) * rp_].reshape(m_ + n_, rp_)
        tu = F[:m_].T @ xp[d["xrow"]: d["xrow"] + m_]
        tv = F[m_:].T @ xp[d["yrow"]: d["yrow"] + n_]
        pout[d["out"]: d["out"] + m_] = F[:m_] @ tv
        pout[d["out"] + m_: d["out"] + m_ + n_] = F[m_:] @ tu
    # fused levels: per pair, E = K(partner pivots, own points) once for both
    # orientations (fused.cu): b_X += K(X,tau) R^-1 L^-1 K(sigma,Y) x_Y and
    # b_Y += K(Y,sigma) L^-T R^-T K(tau,X) x_X
    for d in plan.array("fused_descs"):
        m_, n_, r = int(d["m"]), int(d["n"]), int(d["r"])
        if r == 0:
            continue
        Xp = ppts[d["xrow"]: d["xrow"] + m_]
        Yp = ppts[d["yrow"]: d["yrow"] + n_]
        sig = piv[d["piv_off"]: d["piv_off"] + r]
        tau = piv[d["piv_off"] + r: d["piv_off"] + 2 * r]
        LU = lu[d["lu_off"]: d["lu_off"] + r * r].reshape(r, r)
        Lm = np.tril(LU, -1) + np.eye(r)
        Um = np.triu(LU)
        EX = kernel_matrix(kind, Yp[tau], Xp)  # r x m: K(tau, X)
        EY = kernel_matrix(kind, Xp[sig], Yp)  # r x n: K(sigma, Y)
        sX = np.linalg.solve(Um, np.linalg.solve(Lm, EY @ xp[d["yrow"]: d["yrow"] + n_]))
        sY = np.linalg.solve(Lm.T, np.linalg.solve(Um.T, EX @ xp[d["xrow"]: d["xrow"] + m_]))
        pout[d["out"]: d["out"] + m_] = EX.T @ sX
        pout[d["out"] + m_: d["out"] + m_ + n_] = EY.T @ sY
    for slot, r0, nr, bv, g in h2b:
        if slot >= 0:
            lvl[slot, r0: r0 + nr] = bv
            shits[slot, r0: r0 + nr] += 1
    pcoff, pcpos = plan.array("pc_off"), plan.array("pc_pos")
    for it in pgit:
        g = int(it["node"])
        r0 = rowbeg[g] + it["row0"]
        v = np.zeros(it["nrows"])
        for q in pcpos[pcoff[g]: pcoff[g + 1]]:
            v += pout[int(q) + it["row0"]: int(q) + it["row0"] + it["nrows"]]
        lvl[it["slot"], r0: r0 + it["nrows"]] = v
        shits[it["slot"], r0: r0 + it["nrows"]] += 1
        hits[level_of(g), r0: r0 + it["nrows"]] += 1
    assert hits.max(initial=0) <= 1, "a row written twice at one level"
    assert shits.max(initial=0) <= 1, "a row written twice into one partial"
    # every owned row of a node with partners is covered once at its level
    for l in range(1, L + 1):
        if md[l] == 2:
            continue
        for z in range(1 << (3 * l)):
            g = nb[l] + z
            b0, b1 = off[l][z], off[l][z + 1]
            if rpad[g] == 0 or b1 == b0 or not (row0 <= b0 < row1):
                continue
            assert hits[l, b0:b1].sum() == b1 - b0, (l, z)
    b = np.zeros(n)
    b[row0:row1] = cpart[row0:row1] + lvl[:, row0:row1].sum(axis=0)
    return b, (int(row0), int(row1))


def symmetric_reference(inp, x, kind, direct_leaf=False, diag=0.0):
    """Dense numpy evaluation of the representation the engine applies: the
    reference's dense leaf blocks (exact), one pivot/LU factorization per
    unordered pair applied to both block orientations, optionally the leaf
    level's admissible blocks exact. Morton order in, original order out."""
    L, off, ppts, pd, perm = inp["L"], inp["offsets"], inp["ppts"], inp["pairs"], inp["perm"]
    xp = x[perm]
    b = np.zeros(len(xp))
    lists = inp["lists"]
    for X in range(1 << (3 * L)):
        xb, xe = off[L][X], off[L][X + 1]
        if xe == xb:
            continue
        nbrs = [X]
        if L > 0:
            for k in (1, 2, 3):
                o, ids = lists[L][k]
                nbrs += [int(v) for v in ids[o[X]:o[X + 1]]]
        for Y in nbrs:
            yb, ye = off[L][Y], off[L][Y + 1]
            K = kernel_matrix(kind, ppts[xb:xe], ppts[yb:ye])
            if Y == X:
                np.fill_diagonal(K, diag)
            b[xb:xe] += K @ xp[yb:ye]
    for (l, a, c), (rp, cp, LU) in pd.items():
        xa, xe = off[l][a], off[l][a + 1]
        ya, ye = off[l][c], off[l][c + 1]
        Xp, Yp = ppts[xa:xe], ppts[ya:ye]
        if direct_leaf and l == L:
            K = kernel_matrix(kind, Xp, Yp)
            b[xa:xe] += K @ xp[ya:ye]
            b[ya:ye] += K.T @ xp[xa:xe]
            continue
        r = len(rp)
        if r == 0:
            continue
        Lm = np.tril(LU, -1) + np.eye(r)
        Um = np.triu(LU)
        t = np.linalg.solve(Um, np.linalg.solve(Lm, kernel_matrix(kind, Xp[rp], Yp) @ xp[ya:ye]))
        b[xa:xe] += kernel_matrix(kind, Xp, Yp[cp]) @ t
        t2 = np.linalg.solve(Lm.T, np.linalg.solve(Um.T, kernel_matrix(kind, Yp[cp], Xp) @ xp[xa:xe]))
        b[ya:ye] += kernel_matrix(kind, Yp, Xp[rp]) @ t2
    out = np.empty_like(b)
    out[perm] = b
    return out
