"""Per-P exchange volumes and bounds of the sharded programs, from the
synthetic inputs and the hash partition owner(key) = splitmix64(key ^ seed) % P (numpy here,
the same function as rnn_hash_partition).  Host-only; prints a markdown table."""
import sys
import numpy as np
sys.path.insert(0, ".")
import synth

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    with np.errstate(over="ignore"):
        z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def owner(keys, P, seed=0x5EED):
    return (splitmix64(np.asarray(keys, np.int64).view(np.uint64) ^ np.uint64(seed)) % np.uint64(P)).astype(np.int64)


HBM, LINK = 6551.4e9, 900e9   # B/s: measured HBM copy (MEASURED_PEAKS.json), NVLink 5 per direction


def gcn(g, P, d=128, layers=3, bytes_step=4.69e9):
    keys, src, dst = g["nodes"]["key"], g["edges"]["src"], g["edges"]["dst"]
    o = owner(keys, P)
    kpos = np.argsort(keys)
    own_of = lambda k: o[kpos[np.searchsorted(keys[kpos], k)]]
    od, os_ = own_of(dst), own_of(src)
    n_pad = np.bincount(o, minlength=P).max()
    allg = (P - 1) * n_pad
    halo = max(len(np.unique(src[(od == r) & (os_ != r)])) for r in range(P))
    per_layer = lambda rows: 2 * rows * d * 4            # fwd rows + bwd gradient rows
    return allg, halo, [layers * per_layer(allg) / LINK, layers * per_layer(halo) / LINK,
                        bytes_step / P / HBM]


def main():
    g = synth.arxiv_like(42)
    print("| config | P | all-gather rows / rank | halo rows / rank | ratio | link bound all-gather (ms) | link bound halo (ms) | HBM bound (ms) |")
    print("|---|---|---|---|---|---|---|---|")
    for P in (2, 4, 8):
        a, h, (la, lh, hb) = gcn(g, P)
        print(f"| arxiv GCN | {P} | {a:,} | {h:,} | {h / a:.2f} | {la * 1e3:.3f} | {lh * 1e3:.3f} | {hb * 1e3:.3f} |")
    mag = synth.mag_like(42)
    d = 128
    blocks = {"paper": 4, "author": 4}          # K'/M' blocks per source type
    for P in (2, 4, 8):
        own = {t: owner(k, P) for t, k in mag["key"].items()}
        n_pad = {t: np.bincount(o, minlength=P).max() for t, o in own.items()}
        allg = sum(2 * (P - 1) * n_pad[t] * nb * d * 4 for t, nb in blocks.items())
        halo = 0
        for t, nb in blocks.items():
            keys = mag["key"][t]
            kp = np.argsort(keys)
            worst = 0
            for r in range(P):
                srcs = []
                for x in mag["rels"].values():
                    if x["src_type"] != t:
                        continue
                    tk = mag["key"][x["dst_type"]]
                    tp = np.argsort(tk)
                    od = own[x["dst_type"]][tp[np.searchsorted(tk[tp], x["dst"])]]
                    srcs.append(x["src"][od == r])
                ref = np.unique(np.concatenate(srcs))
                osrc = own[t][kp[np.searchsorted(keys[kp], ref)]]
                worst = max(worst, int((osrc != r).sum()))
            halo += 2 * worst * nb * d * 4
        print(f"| MAG HGT (K'/M' rows) | {P} | {allg // (2 * d * 4 * 8):,} | {halo // (2 * d * 4 * 8):,} | {halo / allg:.2f} | {allg / LINK * 1e3:.3f} | {halo / LINK * 1e3:.3f} | {75.9e9 / P / HBM * 1e3:.3f} |")


if __name__ == "__main__":
    main()
