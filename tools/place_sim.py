"""Bank-conflict simulation of record / Phi placements on a C1 partition layout (dev tool, CPU):
the library's permutation-in-group greedy (place_kernels.cuh) against a global 8-colouring with
capacity; wavefronts per quarter-warp 128-bit load / per-warp 32-bit load.

    python tools/place_sim.py [partitions]
"""
import os, sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O, synth as S

M = S.config_mesh('c1')
P = 1024
k = O.num_parts(M.m, P)
part, rank = O.partition(M.edges, M.n, P, method=2, ranked=True)
L = O.remap(M.edges, M.n, part, k, key=rank)
NP = int(sys.argv[1]) if len(sys.argv) > 1 else 60

def parts():
    for p in range(0, min(k, NP)):
        e0, e1 = L.part_edge_begin[p], L.part_edge_begin[p + 1]
        sl = L.slots[e0:e1].astype(np.int64)
        yield sl[:, 0], sl[:, 1]

def incidence(a, b, nv):
    inc = [[] for _ in range(nv)]
    for i in range(len(a)):
        inc[a[i]].append(2 * i); inc[b[i]].append(2 * i + 1)
    return inc

def wf_octets(ids, pos):           # 128-bit loads per quarter: max multiplicity of bank group among distinct ids
    tot = 0
    for g in range(0, len(ids), 8):
        sub = ids[g:g + 8]; sub = [x for x in sub if x >= 0]
        if not sub: continue
        cnt = {}
        for x in set(sub): cnt[pos[x] % 8] = cnt.get(pos[x] % 8, 0) + 1
        tot += max(cnt.values())
    return tot

def wf_warp32(ids, pos):            # 32-bit loads per warp: max multiplicity of bank among distinct words
    tot = 0
    for g in range(0, len(ids), 32):
        sub = [x for x in ids[g:g + 32] if x >= 0]
        if not sub: continue
        cnt = {}
        for x in set(sub): cnt[pos[x] % 32] = cnt.get(pos[x] % 32, 0) + 1
        tot += max(cnt.values())
    return tot

def measure(a, b, inc, vpos, epos, W=4):
    s, nv = len(a), len(inc)
    edge = 0
    for side in (a, b):
        edge += wf_octets(list(side), vpos)
    red4 = red1 = 0
    for q in range(W):
        ent = [inc[j][q] >> 1 if q < len(inc[j]) else -1 for j in range(nv)]
        red4 += wf_octets(ent, epos)
        red1 += wf_warp32(ent, epos)
    ideal_edge = 2 * ((s + 7) // 8)
    return edge, red4, red1, ideal_edge

def greedy_perm(count, partners, sweeps=2):
    """current library scheme: permutation in aligned groups of 8, most constrained first"""
    col = [-1] * count
    for _ in range(sweeps):
        for g0 in range(0, count, 8):
            nm = min(8, count - g0)
            for x in range(nm): col[g0 + x] = -1
            pen = np.zeros((nm, 8), int)
            for x in range(nm):
                for o in partners[g0 + x]:
                    if o != g0 + x and col[o] >= 0: pen[x, col[o]] += 1
            spread = [pen[x, :nm].max() - pen[x, :nm].min() for x in range(nm)]
            order = sorted(range(nm), key=lambda x: -spread[x])
            used = set()
            for x in order:
                best = min((c for c in range(nm) if c not in used), key=lambda c: pen[x, c])
                used.add(best); col[g0 + x] = best
    return [((j & ~7) | col[j]) for j in range(count)]

def greedy_global(count, partners, sweeps=3):
    """8 colours with capacity ceil(count/8) each (any slot of the colour class), most constrained first"""
    cap = [(count + 7 - c) // 8 for c in range(8)]   # slots of colour c in [0, up8(count))
    col = [-1] * count
    for sw in range(sweeps):
        used = [0] * 8
        if sw > 0:
            for j in range(count): used[col[j]] += 1
        order = sorted(range(count), key=lambda j: -len(partners[j]))
        for j in order:
            if sw > 0: used[col[j]] -= 1
            pen = [0] * 8
            for o in partners[j]:
                if o != j and col[o] >= 0: pen[col[o]] += 1
            cands = [c for c in range(8) if used[c] < cap[c]]
            best = min(cands, key=lambda c: (pen[c], used[c]))
            col[j] = best; used[best] += 1
    # positions: rank within colour class
    rk = [0] * 8; pos = [0] * count
    for j in range(count):
        pos[j] = 8 * rk[col[j]] + col[j]; rk[col[j]] += 1
    return pos

tot = {}
for a, b in parts():
    nv = int(max(a.max(), b.max())) + 1
    inc = incidence(a, b, nv)
    s = len(a)
    # record partners: same side, same edge octet
    vp = [set() for _ in range(nv)]
    for side in (a, b):
        for g in range(0, s, 8):
            mem = set(side[g:g + 8].tolist())
            for x in mem: vp[x] |= mem
    vp = [list(x) for x in vp]
    # phi partners: edges read in the same vertex octet and entry q
    ep = [set() for _ in range(s)]
    for q in range(4):
        for g in range(0, nv, 8):
            mem = set(inc[j][q] >> 1 for j in range(g, min(g + 8, nv)) if q < len(inc[j]))
            for x in mem: ep[x] |= mem
    ep = [list(x) for x in ep]
    variants = {
        'identity': (list(range(nv)), list(range(s))),
        'perm': (greedy_perm(nv, vp), greedy_perm(s, ep)),
        'global': (greedy_global(nv, vp), greedy_perm(s, ep)),
    }
    for name, (vpos, epos) in variants.items():
        r = measure(a, b, inc, vpos, epos)
        t = tot.setdefault(name, np.zeros(4)); t += r
for name, t in tot.items():
    print(f"{name:9s} edge {t[0]/t[3]:.3f}x ideal   phi4 octets {t[1]:.0f}  phi1 warp {t[2]:.0f}")

print("--- phi variants")
tot = {}
for a, b in parts():
    nv = int(max(a.max(), b.max())) + 1
    inc = incidence(a, b, nv); s = len(a)
    ep = [set() for _ in range(s)]
    for q in range(4):
        for g in range(0, nv, 8):
            mem = set(inc[j][q] >> 1 for j in range(g, min(g + 8, nv)) if q < len(inc[j]))
            for x in mem: ep[x] |= mem
    ep_st = [set(x) for x in ep]
    for g in range(0, s, 8):
        mem = set(range(g, min(g + 8, s)))
        for x in mem: ep_st[x] |= mem
    ep = [list(x) for x in ep]; ep_st = [list(x) for x in ep_st]
    ideal4 = sum(1 for q in range(4) for g in range(0, nv, 8) if any(q < len(inc[j]) for j in range(g, min(g + 8, nv))))
    for name, epos in {'perm': greedy_perm(s, ep), 'global+store': greedy_global(s, ep_st), 'global(nostore)': greedy_global(s, ep)}.items():
        r4 = r1 = 0
        for q in range(4):
            ent = [inc[j][q] >> 1 if q < len(inc[j]) else -1 for j in range(nv)]
            r4 += wf_octets(ent, epos); r1 += wf_warp32(ent, epos)
        st = wf_octets(list(range(s)), epos)
        t = tot.setdefault(name, np.zeros(5)); t += (r4, r1, st, ideal4, (s + 7) // 8)
for name, t in tot.items():
    print(f"{name:16s} phi4 {t[0]/t[3]:.3f}x  phi1 {t[1]:.0f}  store {t[2]/t[4]:.3f}x")

print("--- record variants incl. derive stores (weight w of the derive-octet partners)")
tot = {}
for a, b in parts():
    nv = int(max(a.max(), b.max())) + 1
    s = len(a)
    vp = [set() for _ in range(nv)]
    for side in (a, b):
        for g in range(0, s, 8):
            mem = set(side[g:g + 8].tolist())
            for x in mem: vp[x] |= mem
    vpl = [list(x) for x in vp]
    vd = [set(x) for x in vp]
    for g in range(0, nv, 8):
        mem = set(range(g, min(g + 8, nv)))
        for x in mem: vd[x] |= mem
    vd = [list(x) for x in vd]
    vdd = [vpl[j] + [o for o in range((j & ~7), min((j & ~7) + 8, nv))] * 3 for j in range(nv)]  # weight 4 on derive mates
    for name, vpos in {'perm': greedy_perm(nv, vpl), 'global': greedy_global(nv, vpl), 'global+derive': greedy_global(nv, vd), 'global+derive4': greedy_global(nv, vdd)}.items():
        e = wf_octets(list(a), vpos) + wf_octets(list(b), vpos)
        dst = wf_octets(list(range(nv)), vpos)
        t = tot.setdefault(name, np.zeros(4)); t += (e, 2 * ((s + 7) // 8), dst, (nv + 7) // 8)
for name, t in tot.items():
    print(f"{name:16s} edge {t[0]/t[1]:.3f}x  derive-store {t[2]/t[3]:.3f}x   (edge wf {t[0]:.0f}, derive wf x2 halves {2*t[2]:.0f})")
