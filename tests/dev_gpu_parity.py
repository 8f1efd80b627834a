"""Dev harness: GPU vs oracle, printing the first mismatch (run on the box)."""
import sys, time, numpy as np
sys.path.insert(0, ".")
import oracle as O
from paper_2402_16801_b200 import GridrogueBatch

def shapes(tier, n):
    return {k: (dt, shp) for k, (dt, shp) in O.field_shapes(tier, n).items()}

def cmp_state(gb, ob, tier, n, tag):
    ex = gb.export_state(shapes(tier, n))
    ox = ob.state.export_fields()
    bad = [f for f in O.FIELD_NAMES if not np.array_equal(ex[f], ox[f])]
    if bad:
        print(tag, "STATE MISMATCH", bad[:8])
        for f in bad[:4]:
            idx = np.argwhere(ex[f] != ox[f])
            print("   ", f, len(idx), idx[:4].tolist(), ex[f][tuple(idx[0])], ox[f][tuple(idx[0])])
        return False
    return True

def run(tier, n, steps, seed, obs_mode="symbolic", maxlen=None, every=10):
    t0 = time.time()
    gb = GridrogueBatch(n, tier, seed, obs_mode, maxlen)
    obs = gb.reset().cpu().numpy()
    ob = O.OracleBatch(tier, n, seed, max_episode_length=maxlen, threads=8)
    ok = cmp_state(gb, ob, tier, n, f"{tier} reset")
    if obs_mode == "symbolic":
        o2 = ob.state.encode_symbolic()
        if not np.array_equal(obs, o2):
            idx = np.argwhere(obs != o2); print("reset obs mismatch", len(idx), idx[:4].tolist()); ok = False
    if not ok: return False
    na = O.TIERS[tier]["NA"]
    for k in range(steps):
        a = O.random_actions(seed, k, n, na)
        import torch
        obs, rew, done, newly, tm, fl = gb.step(torch.from_numpy(a).cuda())
        r2, d2, nw2, info = ob.step(a)
        obs = obs.cpu().numpy(); rew = rew.cpu().numpy(); done = done.cpu().numpy().astype(bool)
        if not np.array_equal(rew, r2.astype(np.float32)) or not np.array_equal(done, d2) or \
           not np.array_equal(newly.cpu().numpy().astype(bool), nw2) or \
           not np.array_equal(tm.cpu().numpy().view(np.uint32), info["time"]) or not np.array_equal(fl.cpu().numpy(), info["floor"]):
            print(tier, "step", k, "OUTPUT MISMATCH", np.nonzero(rew != r2.astype(np.float32))[0][:5], np.nonzero(done != d2)[0][:5])
            cmp_state(gb, ob, tier, n, "   state"); return False
        if obs_mode == "symbolic":
            o2 = ob.state.encode_symbolic()
            if not np.array_equal(obs, o2):
                idx = np.argwhere(obs != o2); print(tier, "step", k, "OBS mismatch", len(idx), idx[:4].tolist(), obs[tuple(idx[0])], o2[tuple(idx[0])])
                cmp_state(gb, ob, tier, n, "   state"); return False
        elif obs_mode == "pixels":
            px = 7 if tier == "classic" else 10
            o2 = ob.state.render_pixels(px)
            if not np.array_equal(obs, o2):
                idx = np.argwhere(obs != o2); print(tier, "step", k, "PIX mismatch", len(idx), idx[:4].tolist(), obs[tuple(idx[0])], o2[tuple(idx[0])])
                return False
        if k % every == 0 or k == steps - 1:
            if not cmp_state(gb, ob, tier, n, f"{tier} step {k}"): return False
    print("OK", tier, obs_mode, n, steps, "episodes", gb.stats()["episodes"], ob.stats()["episodes"], "%.1fs" % (time.time() - t0), gb.worldgen_counters())
    return True

def observe_check(tier, n, seed):
    """gr_observe after importing a foreign (oracle) state."""
    import torch
    gb = GridrogueBatch(n, tier, seed, "symbolic")
    gb.reset()
    ob = O.OracleBatch(tier, n, seed + 1)
    for k in range(30):
        ob.step(O.random_actions(seed, k, n, O.TIERS[tier]["NA"]))
    gb.import_state(ob.state.export_fields())
    o1 = gb.observe().cpu().numpy()
    o2 = ob.state.encode_symbolic()
    ok = np.array_equal(o1, o2)
    print("observe-after-import", tier, "OK" if ok else "MISMATCH")
    return ok

if __name__ == "__main__":
    r = True
    r &= run("classic", 256, 200, 0)
    r &= run("extended", 256, 200, 0)
    r &= run("extended", 128, 100, 3, maxlen=16)
    r &= run("classic", 64, 60, 1, obs_mode="pixels")
    r &= run("extended", 64, 60, 2, obs_mode="pixels")
    r &= observe_check("extended", 64, 5)
    r &= observe_check("classic", 64, 6)
    r &= observe_check("extended", 64, 5)
    r &= observe_check("classic", 64, 6)
    print("ALL OK" if r else "FAILURES")

