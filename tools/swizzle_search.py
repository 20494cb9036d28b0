"""Search / verify the XOR swizzle of the training kernel's 64-float shared
tiles (pg_train_mma.cu swz): every warp-wide access pattern the kernel uses
must touch 32 distinct banks (one wavefront).  Prints the linear masks that
work and the wavefront count of each pattern under the chosen one."""
import itertools

KS = 64


def make(v):
    def f(r):
        x = 0
        for i in range(3):
            if (r >> i) & 1:
                x ^= v[i]
        return x
    return f


def patterns(f):
    """Yield (name, [32 word addresses]) for every warp access pattern."""
    lanes = [(ln >> 2, ln & 3) for ln in range(32)]
    idx = lambda r, c: r * KS + (c ^ f(r))
    for r0 in range(0, 64, 8):
        for c0 in range(0, 64, 8):
            for h in (0, 4):
                # fragment, rows indexed by k (lane%4), columns m/n (lane/4)
                yield "rowk", [idx(c0 + c + h if c0 + c + h < 64 else c + h, r0 + g) for g, c in lanes]
                # fragment, rows indexed by m/n (lane/4), columns k (lane%4)
                yield "rowmn", [idx(r0 + g, c0 + c + h) for g, c in lanes]
            for e in (0, 1):
                # C-fragment stores: rows n0 + 2c + e, columns m0 + g
                yield "store", [idx(r0 + 2 * c + e, c0 + g) for g, c in lanes]
    for r0 in range(0, 64, 8):
        for i in range(16):
            # bias row sums: rows r0 + lane/4, columns lane%4 + 4i
            yield "rowsum", [idx(r0 + g, c + 4 * i) for g, c in lanes]
    for r in range(64):
        for q0 in (0, 32):
            yield "row", [idx(r, q0 + ln) for ln in range(32)]


def wavefronts(addrs):
    banks = {}
    for a in set(addrs):
        banks.setdefault(a % 32, set()).add(a)
    return max(len(s) for s in banks.values())


def ok(f):
    return all(wavefronts(a) == 1 for _, a in patterns(f))


if __name__ == "__main__":
    sols = [v for v in itertools.product(range(32), repeat=3) if ok(make(v))]
    print(f"{len(sols)} conflict-free linear masks, e.g. {sols[:4]}")
    f = make((8, 16, 12))
    worst = {}
    for name, a in patterns(f):
        worst[name] = max(worst.get(name, 0), wavefronts(a))
    print("swz(r) = ((r&3)<<3) ^ (((r>>2)&1)*12): worst wavefronts per pattern", worst)
    f72 = lambda r: 0
    worst72 = {}
    for name, a in patterns(f72):
        a72 = [(x // KS) * 72 + x % KS for x in a]
        worst72[name] = max(worst72.get(name, 0), wavefronts(a72))
    print("stride 72, no swizzle: worst wavefronts per pattern", worst72)
