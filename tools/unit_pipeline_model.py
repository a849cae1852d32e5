"""Model of k_umma's unit pipeline for c5 (diagnostics): MMA passes of a unit alternate between
two TMEM accumulator buffers; the 8 epilogue warps drain one pass at a time; the MMA issuer
may start pass i only when the epilogue has drained pass i - 2 (same buffer), and a unit only
when its window is converted (one window buffer: after the previous unit's last MMA).  Prints
the modelled cycles per unit for epilogue times / buffer counts -- the accumulator buffers, not
the window, are the main stall (measured: MMA waits 10 % on acc_empty, 6 % on win_full)."""
tiles = [84, 25, 8, 4, 2]  # K-step tiles per pass of c5 (heavy pass first)


def run(busy=49.7, e=7.4, conv=4.0, order=(0, 1, 2, 3, 4), nbuf=2, units=40):
    m = [busy * t / sum(tiles) for t in tiles]
    t_mma = t_epi = last = 0.0
    buf_free = [0.0] * nbuf
    k = 0
    starts = []
    for u in range(units):
        t_mma = max(t_mma, last + conv if u else conv)
        starts.append(t_mma)
        for p in order:
            b = k % nbuf
            t_mma = max(t_mma, buf_free[b]) + m[p]
            t_epi = max(t_epi, t_mma) + e
            buf_free[b] = t_epi
            k += 1
        last = t_mma
    return (starts[-1] - starts[10]) / (units - 11)


if __name__ == "__main__":
    print("k cycles per unit (MMA busy 49.7 k):")
    for label, kw in (("epilogue 7.4 k per pass (measured r02j)", {}), ("epilogue 6.5 k", {"e": 6.5}),
                      ("epilogue 5 k", {"e": 5.0}), ("epilogue 3 k", {"e": 3.0}),
                      ("no window wait", {"conv": 0.0}), ("three buffers", {"nbuf": 3}),
                      ("four buffers", {"nbuf": 4}), ("light passes first", {"order": (4, 3, 2, 1, 0)})):
        print(f"  {label:42s} {run(**kw):6.1f}")
