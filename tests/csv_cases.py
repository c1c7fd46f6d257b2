"""CSV inputs for the load_csv parity tests (proj/src/csv.cpp:63-115).

Seeded generators of cell texts (printf-style, shortest round-trip, hex floats, long digit
strings, exact binary64 midpoints for round-half-even, subnormals and overflow edges,
inf/nan spellings, whitespace and quoting variants) and of whole files (quoted separators,
CRLF, blank lines, label columns, ragged rows), plus byte-level mutations. The expected
result is always the oracle's (oracle/renyi_oracle.cpp: read_record / parse_cell with glibc
std::strtod), never a value written here."""
from __future__ import annotations

import math
import random
import struct
from decimal import Decimal, getcontext

getcontext().prec = 1200


def _next_up(x: float) -> float:
    return math.nextafter(x, math.inf)


def _random_double(rng: random.Random) -> float:
    kind = rng.random()
    if kind < 0.5:
        return rng.gauss(0.0, 1.0) * 10.0 ** rng.randint(-5, 5)
    if kind < 0.8:
        bits = rng.getrandbits(64)
        x = struct.unpack("<d", struct.pack("<Q", bits))[0]
        return x if math.isfinite(x) else 1.0
    if kind < 0.9:  # subnormal
        return struct.unpack("<d", struct.pack("<Q", rng.randint(1, (1 << 52) - 1)))[0]
    return rng.choice([0.0, -0.0, 1.0, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 0.1, 1e22, 1e23])


def _midpoint_text(rng: random.Random) -> str:
    """Exact decimal expansion of the midpoint of two adjacent doubles (a tie), optionally nudged."""
    a = abs(_random_double(rng))
    if a == 0.0 or not math.isfinite(_next_up(a)):
        a = 1.0
    b = _next_up(a)
    mid = (Decimal(a) + Decimal(b)) / 2  # exact: Decimal(float) is the binary value
    s = format(mid, "E")
    nudge = rng.random()
    if nudge < 0.3:  # just above the tie: an extra nonzero digit far out
        mant, exp = s.split("E")
        if "." not in mant:
            mant += "."
        s = mant + "0" * rng.randint(0, 40) + "1" + "E" + exp
    elif nudge < 0.4:  # just below: truncate the expansion
        mant, exp = s.split("E")
        if len(mant) > 4:
            s = mant[:-1] + "E" + exp
    return s


def _long_digits(rng: random.Random) -> str:
    nd = rng.choice([16, 17, 18, 19, 20, 25, 40, 120, 900])
    digits = "".join(rng.choice("0123456789") for _ in range(nd)).lstrip("0") or "0"
    if rng.random() < 0.5:
        p = rng.randint(0, len(digits))
        digits = digits[:p] + "." + digits[p:]
    return digits + (f"e{rng.randint(-340, 320)}" if rng.random() < 0.7 else "")


def number_text(rng: random.Random) -> str:
    x = _random_double(rng)
    k = rng.random()
    if k < 0.2:
        s = repr(x)
    elif k < 0.35:
        s = "%.*g" % (rng.randint(1, 17), x)
    elif k < 0.45:
        s = "%g" % x  # std::ostream default (make_labeled_csv, test_cli.cpp:60-77)
    elif k < 0.55:
        s = "%.*e" % (rng.randint(0, 20), x)
    elif k < 0.62:
        s = x.hex() if rng.random() < 0.7 else x.hex().upper().replace("0X", "0x")
    elif k < 0.75:
        s = _midpoint_text(rng)
    elif k < 0.85:
        s = _long_digits(rng)
    elif k < 0.9:
        s = str(rng.randint(-10 ** 18, 10 ** 18))
    else:
        s = rng.choice(["inf", "-inf", "INF", "Infinity", "+infinity", "nan", "-NaN", "nan()", "nan(123)",
                        "nan(0x7fff)", "NAN(abc_1)", "nan(017)", "nan(0x)", "nan(99999999999999999999999)",
                        "1e400", "-1e400", "1e-400", "2.4703282292062327e-324", "2.4703282292062328e-324",
                        "1.7976931348623158e308", "1.7976931348623159e308", "4.9406564584124654e-324",
                        "0x1p-1074", "0x1p-1075", "0x1.8p-1074", "0x1.fffffffffffff8p1023", "0x1p1024",
                        "0x.8p1", "0x10", "1.", ".5", "+.5e1", "-0", "0e0", "00012.50", "0.000"])
    # decorations strtod accepts
    d = rng.random()
    if d < 0.1:
        s = rng.choice([" ", "\t", "  ", "\v", "\f"]) + s
    elif d < 0.2:
        s = s + " " * rng.randint(1, 3)
    elif d < 0.25:
        s = '"' + s + '"'
    return s


BAD_CELLS = ["", "abc", "1e", "1e+", "--1", "1.2.3", "0x", "0xg", "0x.p1", "inf1", "infinit", "nan(", "nan(a b)",
             "1 2", "1\t", ".", "+", "e5", "1,5", "0x1p", "nanx", "in", "1e5x", "\"\"", "  ", "1.5\"x\""]


def field_text(cell: str) -> str:
    """Quote a cell when it holds separators or quotes (RFC 4180 style)."""
    if any(c in cell for c in ',\n"') and not (cell.startswith('"') and cell.endswith('"') and len(cell) > 1):
        return '"' + cell.replace('"', '""') + '"'
    return cell


def make_csv(rng: random.Random, n: int, d: int, label_at: int | None = None, crlf: bool = False,
             blank_lines: bool = False, bad: str | None = None, bad_at: tuple[int, int] | None = None) -> str:
    cols = d + (1 if label_at is not None else 0)
    header = [f"f{j}" for j in range(d)]
    if label_at is not None:
        header.insert(label_at, "class")
    nl = "\r\n" if crlf else "\n"
    lines = [",".join(field_text(h) for h in header)]
    for i in range(n):
        cells = [number_text(rng) for _ in range(d)]
        if label_at is not None:
            cells.insert(label_at, rng.choice(["pos", "neg", "a,b", 'q"t', "multi\nline", ""]))
        if bad_at is not None and bad_at[0] == i:
            cells[bad_at[1] % cols] = bad
        lines.append(",".join(field_text(c) for c in cells))
        if blank_lines and rng.random() < 0.1:
            lines.append(rng.choice(["", '""', "\r"]))
    text = nl.join(lines)
    if rng.random() < 0.7:
        text += nl
    return text


def mutate(rng: random.Random, text: str, edits: int = 3) -> str:
    s = list(text)
    for _ in range(edits):
        if not s:
            break
        p = rng.randrange(len(s) + 1)
        op = rng.random()
        if op < 0.3:
            s.insert(p, rng.choice(['"', ",", "\n", "\r", "\x00", " ", "e", "-", "."]))
        elif op < 0.6 and p < len(s):
            del s[p]
        elif p < len(s):
            s[p] = rng.choice(['"', ",", "\n", "0", "x"])
    return "".join(s)
