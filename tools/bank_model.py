"""Half-warp shared-memory bank model of the 3-D R=2 tensor engines' A-operand
loads (profiles/r02/README.md).

A 64-bit shared load is processed per half-warp: 16 lanes = 4 cells (r8) x 4
chunk slots (k4) over 16 banks of 8 bytes; the wavefronts of a half are the
largest number of DISTINCT words that fall on one bank.  The four slots of a
chunk sit at the stencil offsets of the (host-built) chunk tables.  Prints the
wavefronts per LDS.64 for the ring loads under several (row stride, cell
mapping) choices and for the W cache under several layouts; the ncu counts
(L1 Wavefronts Shared / instruction, profiles/r02/prof_c4_states*.ncu-rep)
are 4.0-4.57 for (36, stride 4) and 3.4-4.0 for (36, contiguous)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_16543_b200 as K  # noqa: E402

R = 2
rs = K.precompute(R, dim=3)
off = rs.offsets
ch1, flat = [], []
for st in rs.st:  # pass 1: front-padded chunks per stencil; pass 2: packed
    g = list(st.gather)
    kc = (len(g) + 3) // 4
    sl = [g[0]] * (4 * kc - len(g)) + g
    ch1 += [sl[4 * j:4 * j + 4] for j in range(kc)]
    flat += g
while len(flat) % 4:
    flat.append(flat[-1])
ch2 = [flat[i:i + 4] for i in range(0, len(flat), 4)]
K0 = (len(rs.st[0].gather) + 3) // 4


def wavefronts(chunks, addr):
    tot = 0
    for c in chunks:
        for half in (0, 1):
            words = {}
            for k4, e in enumerate(c):
                for r8 in range(4 * half, 4 * half + 4):
                    a = addr(k4, e, r8)
                    words.setdefault(a % 16, set()).add(a)
            tot += max(len(v) for v in words.values())
    return tot / len(chunks)


def ring(rx, cell):
    return lambda k4, e, r8: (off[e][1] + R) * rx + off[e][0] + R + cell(r8)


def main():
    print("ring loads (wavefronts per LDS.64: pass 1, pass 2)")
    for name, cm in (("cells w + 4 r8", lambda r: 4 * r), ("cells 8 w + r8", lambda r: r)):
        for rx in (36, 38, 40, 42, 44):
            print(f"  {name}  row stride {rx}: {wavefronts(ch1, ring(rx, cm)):.2f} "
                  f"{wavefronts(ch2, ring(rx, cm)):.2f}")
    print("W cache rows of 8 cells, S words apart (address S e + r8)")
    for S in (8, 12, 20):
        f = lambda k4, e, r8, S=S: S * e + r8  # noqa: E731
        print(f"  S = {S}: {wavefronts(ch1[K0:], f):.2f} {wavefronts(ch2, f):.2f}")
    print("W cache split by half-warp, position mod 4 = a 4-colouring of S0: the host's search "
          "(kfvm_gpu.cu upload_gen) reaches ~1.2 wavefronts per half = 2.4 per load")


if __name__ == "__main__":
    main()
