"""Regenerate paper_2206_14735_b200/csrc/gsb_pcg_tables.cuh (PCG64 jump-ahead constants)."""
M = (0x2360ED051FC65DA4 << 64) | 0x4385DF649FCCF645  # numpy PCG64 multiplier
MASK = (1 << 128) - 1


def tables():
    mult, plus, cur, p = [], [], M, 1
    for _ in range(64):
        mult.append(cur)
        plus.append(p)
        p = (p * (cur + 1)) & MASK
        cur = (cur * cur) & MASK
    return mult, plus


if __name__ == "__main__":
    m, p = tables()
    print(len(m), hex(m[1]), hex(p[1]))
