"""Generate csrc/libm_port.cuh: bit-exact restatements of the host libm's
sin, cos, atan2, acos and hypot -- the libm functions the reference's Dubins
steering calls that IEEE arithmetic does not pin (dubins.cpp:49-167,
steering.cpp:113) -- for the device.

The reference links glibc 2.39's libm, whose x86-64 entry points dispatch
(IFUNC) to FMA builds of the IBM Accurate Mathematical Library routines
(sysdeps/ieee754/dbl-64/s_sin.c, e_atan2.c, e_asin.c).  Those routines are
not correctly rounded, so no device libm reproduces their last bits.  This
tool restates them instruction by instruction from the library's own
machine code: every scalar SSE/AVX/FMA operation becomes the IEEE operation
it performs (one rounding each: add, sub, mul, div, fma), integer work stays
integer work, and the read-only tables the routines index (sin/cos of
i/128, the atan and asin/acos interval tables) are emitted as constant
arrays.  Paths the reference never reaches (|x| >= 105414350 for sin/cos,
which call __branred; errno side effects) return NaN.

    python tools/libm_port.py [LIBM] > paper_1705_02403_b200/csrc/libm_port.cuh

The output is pinned bit for bit against the host libm by
tests/test_libm_port.py (hundreds of millions of inputs through the host
build of the same source) and against the reference's Dubins costs by the
GPU tests."""
import re
import subprocess
import sys

LIBM = sys.argv[1] if len(sys.argv) > 1 else "/lib/x86_64-linux-gnu/libm.so.6"
LIBM_BYTES = open(LIBM, "rb").read()  # (.rodata's file offsets equal its addresses)


def objdump(start, stop):
    out = subprocess.run(["objdump", "-d", "--no-show-raw-insn", f"--start-address={start:#x}",
                          f"--stop-address={stop:#x}", LIBM], capture_output=True, text=True, check=True).stdout
    lines = []
    for ln in out.splitlines():
        m = re.match(r"^\s+([0-9a-f]+):\s+(\S+)\s*(.*)$", ln)
        if m:
            lines.append((int(m.group(1), 16), m.group(2), m.group(3)))
    return lines


def resolver_targets(addr):
    """The lea targets of an IFUNC resolver, in the order it tests them
    (the first is the FMA build: cpu_features has FMA and AVX2)."""
    t = []
    for a, mn, ops in objdump(addr, addr + 0x60):
        if mn == "lea" and "(%rip)" in ops:
            t.append(int(ops.split("#")[1].split()[0], 16))
        if mn == "ret":
            break
    return t


def dynsym(name):
    """The default (unparenthesised) version of a dynamic symbol -- what a
    program linked against this libm binds (hypot@@GLIBC_2.35, not the
    compat hypot@GLIBC_2.2.5)."""
    out = subprocess.run(["objdump", "-T", LIBM], capture_output=True, text=True, check=True).stdout
    for ln in out.splitlines():
        f = ln.split()
        if f and f[-1] == name and ".text" in ln and not f[-2].startswith("("):
            return int(f[0], 16), ln
    raise KeyError(name)


def plt_irelative_target(wrapper_addr):
    """sin/cos are IFUNC symbols themselves; atan2/acos are wrappers that
    jump to an IRELATIVE PLT slot "*ABS*+0xRESOLVER@plt"."""
    for a, mn, ops in objdump(wrapper_addr, wrapper_addr + 0x100):
        m = re.search(r"\*ABS\*\+0x([0-9a-f]+)@plt", ops)
        if m and mn in ("jmp", "call"):
            return int(m.group(1), 16)
    raise RuntimeError("no IRELATIVE target")


def function_extent(start, size=None):
    """Instructions from start to the end of the function: its symbol size
    when known, else up to the first endbr64 after start (the next
    function)."""
    lines = objdump(start, start + (size or 0x1000))
    out = []
    for i, (a, mn, ops) in enumerate(lines):
        if i > 0 and mn == "endbr64":
            break
        out.append((a, mn, ops))
    return out


# sha256 of the libm -> [(lo, hi)] byte ranges of the tables its sin / cos /
# atan2 / acos read (sincostab; the acos and atan2 tables, adjacent).
EXTENTS = {
    "3c24a53ee35c2ce0c67240e62bff699c4bddcd7cf8993d5d7ad29157ba072c99": [(0xb3bc0, 0xb49c0), (0xba580, 0xc2fc0)],
}


GPR = {}
for i, base in enumerate(["ax", "bx", "cx", "dx"]):
    GPR["r" + base] = (i, 64)
    GPR["e" + base] = (i, 32)
    GPR[base] = (i, 16)
    GPR[base[0] + "l"] = (i, 8)
    GPR[base[0] + "h"] = (i, 108)  # high byte
for i, base in [(4, "si"), (5, "di"), (6, "bp"), (7, "sp")]:
    GPR["r" + base] = (i, 64)
    GPR["e" + base] = (i, 32)
    GPR[base] = (i, 16)
    GPR[base + "l"] = (i, 8)
for i in range(8, 16):
    GPR[f"r{i}"] = (i, 64)
    GPR[f"r{i}d"] = (i, 32)
    GPR[f"r{i}w"] = (i, 16)
    GPR[f"r{i}b"] = (i, 8)


def split_ops(s):
    s = s.split("#")[0].strip()
    out, depth, cur = [], 0, ""
    for ch in s:
        if ch == "(":
            depth += 1
        elif ch == ")":
            depth -= 1
        if ch == "," and depth == 0:
            out.append(cur.strip())
            cur = ""
        else:
            cur += ch
    if cur.strip():
        out.append(cur.strip())
    return out


class Gen:
    def __init__(self, name, insns, nargs):
        self.name, self.insns, self.nargs = name, insns, nargs
        self.tables = set()  # absolute addresses loaded through registers (lea rip)
        self.consts = set()  # absolute addresses read rip-relative
        self.out = []
        self.targets = set()

    def comment_addr(self, ops):
        return int(ops.split("#")[1].split()[0], 16)

    # ---- operands ----------------------------------------------------------
    def mem_addr(self, op, ops_text):
        """C expression of a memory operand's address; ('stk', off) for the
        frame, ('abs', A) for rip-relative, ('reg', expr) otherwise."""
        if op.startswith("%fs:"):
            return ("fs", 0)
        m = re.match(r"^(-?0x[0-9a-f]+|-?\d+)?\((%\w+)?(?:,(%\w+),(\d))?\)$", op)
        if not m:
            raise ValueError(op)
        disp = int(m.group(1), 0) if m.group(1) else 0
        base = m.group(2)[1:] if m.group(2) else None
        if base == "rip":
            a = self.comment_addr(ops_text)
            self.consts.add(a)
            return ("abs", a)
        if base == "rbp":
            return ("stk", disp)
        e = f"r[{GPR[base][0]}]" if base else "0ull"
        if m.group(3):
            e = f"({e} + r[{GPR[m.group(3)[1:]][0]}] * {m.group(4)}ull)"
        if disp:
            e = f"({e} + (u64)({disp}ll))"
        return ("reg", e)

    def load(self, op, ops_text, size):
        if op.startswith("%fs:"):
            return "0ull"  # (the stack protector's canary)
        if op.startswith("%xmm"):
            return f"x[{int(op[4:])}]"
        if op.startswith("%"):
            return self.rd(op)
        if op.startswith("$"):
            return f"{int(op[1:], 0) & (2**64 - 1):#x}ull"
        kind, a = self.mem_addr(op, ops_text)
        if kind == "fs":
            return "0ull"
        if kind == "stk":
            return f"lm_stk_ld{size}(stk, {a})"
        if kind == "abs":  # a rip-relative constant: its value, folded in
            v = int.from_bytes(LIBM_BYTES[a:a + size // 8], "little")
            return f"{v:#x}ull"
        return f"lm_mem_ld{size}(stk, {a})"

    def store(self, op, ops_text, size, val):
        if op.startswith("%fs:"):
            return ";"
        if op.startswith("%xmm"):
            return f"x[{int(op[4:])}] = {val};"
        if op.startswith("%"):
            return self.wr(op, val)
        kind, a = self.mem_addr(op, ops_text)
        if kind == "stk":
            return f"lm_stk_st{size}(stk, {a}, {val});"
        if kind == "fs":
            return ";"
        return f"lm_mem_st{size}(stk, {a}, {val});"

    def width(self, op):
        if op.startswith("%fs:"):
            return None
        return GPR[op[1:]][1] if op.startswith("%") and op[1:] in GPR else None

    def rd(self, op):
        i, w = GPR[op[1:]]
        return {64: f"r[{i}]", 32: f"(u64)(u32)r[{i}]", 16: f"(u64)(u16)r[{i}]", 8: f"(u64)(u8)r[{i}]",
                108: f"(u64)(u8)(r[{i}] >> 8)"}[w]

    def wr(self, op, val):
        i, w = GPR[op[1:]]
        return {64: f"r[{i}] = {val};", 32: f"r[{i}] = (u64)(u32)({val});",
                16: f"r[{i}] = (r[{i}] & ~0xffffull) | ((u64)({val}) & 0xffffull);",
                8: f"r[{i}] = (r[{i}] & ~0xffull) | ((u64)({val}) & 0xffull);",
                108: f"r[{i}] = (r[{i}] & ~0xff00ull) | (((u64)({val}) & 0xffull) << 8);"}[w]

    def wbits(self, w):
        return {64: 64, 32: 32, 16: 16, 8: 8, 108: 8}[w]

    # ---- flags -------------------------------------------------------------
    def flags_logic(self, res, w):
        b = self.wbits(w)
        mask = "~0ull" if b == 64 else f"((1ull << {b}) - 1)"
        return (f"{{ const u64 t_ = ({res}) & {mask}; ZF = t_ == 0; SF = (t_ >> {b - 1}) & 1; CF = 0; OF = 0; }}")

    def flags_sub(self, a, bb, w):
        b = self.wbits(w)
        mask = "~0ull" if b == 64 else f"((1ull << {b}) - 1)"
        return (f"{{ const u64 a_ = ({a}) & {mask}, b_ = ({bb}) & {mask}, t_ = (a_ - b_) & {mask}; "
                f"ZF = t_ == 0; SF = (t_ >> {b - 1}) & 1; CF = a_ < b_; "
                f"OF = (((a_ ^ b_) & (a_ ^ t_)) >> {b - 1}) & 1; }}")

    def flags_add(self, a, bb, w):
        b = self.wbits(w)
        mask = "~0ull" if b == 64 else f"((1ull << {b}) - 1)"
        return (f"{{ const u64 a_ = ({a}) & {mask}, b_ = ({bb}) & {mask}, t_ = (a_ + b_) & {mask}; "
                f"ZF = t_ == 0; SF = (t_ >> {b - 1}) & 1; CF = t_ < a_; "
                f"OF = ((~(a_ ^ b_) & (a_ ^ t_)) >> {b - 1}) & 1; }}")

    COND = {"je": "ZF", "jne": "!ZF", "jg": "(!ZF && SF == OF)", "jle": "(ZF || SF != OF)",
            "jl": "(SF != OF)", "jge": "(SF == OF)", "ja": "(!CF && !ZF)", "jae": "!CF",
            "jb": "CF", "jbe": "(CF || ZF)", "js": "SF", "jns": "!SF", "jp": "PF", "jnp": "!PF"}

    # ---- translation -------------------------------------------------------
    def emit(self, a, mn, ops_text):
        o = split_ops(ops_text)
        E = self.out.append
        if mn in ("endbr64", "push", "pop", "leave", "nop", "nopl", "nopw", "xchg", "cs", "vldmxcsr", ".byte", "data16"):
            if mn == "xchg" and o != ["%ax", "%ax"]:
                raise ValueError(f"{a:x} xchg {ops_text}")
            return
        if mn == "vstmxcsr":
            E(self.store(o[0], ops_text, 32, "0x1f80ull"))  # round to nearest, exceptions masked
            return
        if mn == "ret":
            E("return lm_f(x[0]);")
            return
        if mn == "call":
            tgt = ops_text.split("<")[1] if "<" in ops_text else ops_text
            E(f"return lm_nan();  /* call {tgt.strip('>')}: outside the ported domain */")
            return
        if mn == "jmp" or mn in self.COND:
            t = int(o[0].split()[0], 16)
            self.targets.add(t)
            E(f"goto L_{t:x};" if mn == "jmp" else f"if ({self.COND[mn]}) goto L_{t:x};")
            return
        # ---- scalar double ----
        if mn == "vmovsd":
            if len(o) == 3:  # vmovsd %a,%b,%d: d.low = a.low
                E(f"x[{int(o[2][4:])}] = x[{int(o[0][4:])}];")
            elif o[1].startswith("%xmm"):
                E(f"x[{int(o[1][4:])}] = {self.load(o[0], ops_text, 64)};")
            else:
                E(self.store(o[1], ops_text, 64, f"x[{int(o[0][4:])}]"))
            return
        sse = {"addsd": "lm_add", "subsd": "lm_sub", "mulsd": "lm_mul", "divsd": "lm_div"}
        if mn in sse:  # SSE: op a, d -> d = d OP a
            a_, d = self.load(o[0], ops_text, 64), f"x[{int(o[1][4:])}]"
            E(f"{d} = lm_b({sse[mn]}(lm_f({d}), lm_f({a_})));")
            return
        if mn in ("sqrtsd", "vsqrtsd"):
            a_, d = self.load(o[0], ops_text, 64), f"x[{int(o[-1][4:])}]"
            E(f"{d} = lm_b(lm_sqrt(lm_f({a_})));")
            return
        if mn in ("movapd", "movsd") and len(o) == 2:
            if o[1].startswith("%xmm"):
                E(f"x[{int(o[1][4:])}] = {self.load(o[0], ops_text, 64)};")
            else:
                E(self.store(o[1], ops_text, 64, f"x[{int(o[0][4:])}]"))
            return
        if mn in ("andpd", "orpd", "xorpd", "pxor", "andnpd"):
            a_, d = self.load(o[0], ops_text, 64), f"x[{int(o[1][4:])}]"
            if mn == "andnpd":
                E(f"{d} = ~{d} & {a_};")
            else:
                E(f"{d} = {d} {dict(andpd='&', orpd='|', xorpd='^', pxor='^')[mn]} {a_};")
            return
        if mn in ("comisd", "ucomisd") or (mn == "movq" and "%xmm" in ops_text):
            mn = "v" + mn
        if mn == "vmovq":
            if o[1].startswith("%xmm"):
                E(f"x[{int(o[1][4:])}] = {self.load(o[0], ops_text, 64)};")
            else:
                E(self.store(o[1], ops_text, 64, self.load(o[0], ops_text, 64)))
            return
        arith = {"vaddsd": "lm_add", "vsubsd": "lm_sub", "vmulsd": "lm_mul", "vdivsd": "lm_div"}
        if mn in arith:  # AT&T: op a, b, d -> d = b OP a
            a_, b_ = self.load(o[0], ops_text, 64), self.load(o[1], ops_text, 64)
            E(f"x[{int(o[2][4:])}] = lm_b({arith[mn]}(lm_f({b_}), lm_f({a_})));")
            return
        m = re.match(r"^vf(n?)m(add|sub)(132|213|231)sd$", mn)
        if m:  # AT&T (op1, op2, op3) = Intel (src3, src2, dst)
            neg, kind, form = m.group(1) == "n", m.group(2), m.group(3)
            s1, s2, d = self.load(o[0], ops_text, 64), self.load(o[1], ops_text, 64), f"x[{int(o[2][4:])}]"
            mul = {"132": (d, s1), "213": (s2, d), "231": (s2, s1)}[form]
            add = {"132": s2, "213": s1, "231": d}[form]
            ma = f"lm_f({mul[0]})"
            mb = f"lm_f({mul[1]})"
            if neg:
                ma = f"-{ma}"
            c = f"lm_f({add})" if kind == "add" else f"-lm_f({add})"
            E(f"{d} = lm_b(lm_fma({ma}, {mb}, {c}));")
            return
        logic = {"vandpd": "&", "vorpd": "|", "vxorpd": "^"}
        if mn in logic:
            a_, b_ = self.load(o[0], ops_text, 64), self.load(o[1], ops_text, 64)
            E(f"x[{int(o[2][4:])}] = {b_} {logic[mn]} {a_};")
            return
        if mn == "vandnpd":  # d = ~op2 & op1
            a_, b_ = self.load(o[0], ops_text, 64), self.load(o[1], ops_text, 64)
            E(f"x[{int(o[2][4:])}] = ~{b_} & {a_};")
            return
        if mn == "vblendvpd":  # d = mask.sign ? op2 : op3
            mk, s2, s3 = (self.load(o[i], ops_text, 64) for i in range(3))
            E(f"x[{int(o[3][4:])}] = ({mk} >> 63) ? {s2} : {s3};")
            return
        m = re.match(r"^vcmp(n?)(lt|le|eq)sd$", mn)
        if m:  # d = pred(op2, op1)
            a_, b_ = self.load(o[0], ops_text, 64), self.load(o[1], ops_text, 64)
            rel = {"lt": "<", "le": "<=", "eq": "=="}[m.group(2)]
            p = f"(lm_f({b_}) {rel} lm_f({a_}))"
            if m.group(1):
                p = f"!{p}"
            E(f"x[{int(o[2][4:])}] = {p} ? ~0ull : 0ull;")
            return
        if mn in ("vcomisd", "vucomisd"):  # compare op2 with op1
            a_, b_ = self.load(o[0], ops_text, 64), self.load(o[1], ops_text, 64)
            E(f"{{ const double a_ = lm_f({b_}), b_ = lm_f({a_}); "
              f"if (a_ != a_ || b_ != b_) {{ ZF = PF = CF = 1; }} "
              f"else {{ ZF = a_ == b_; CF = a_ < b_; PF = 0; }} OF = SF = 0; }}")
            return
        if mn == "vcvttsd2si":
            w = self.width(o[1])
            cv = "(u64)(long long)lm_f" if w == 64 else "(u64)(u32)(int)lm_f"
            E(self.wr(o[1], f"{cv}({self.load(o[0], ops_text, 64)})"))
            return
        # ---- integer ----
        if mn == "movabs":
            E(self.wr(o[1], self.load(o[0], ops_text, 64)))
            return
        if mn in ("mov", "movl", "movq", "movslq", "cltq", "lea", "shl", "sar", "shr", "and", "or", "xor",
                  "add", "sub", "imul", "cmp", "test", "testb", "cmpl", "cmove", "cmovne"):
            return self.emit_int(a, mn, o, ops_text)
        raise ValueError(f"{a:x}: unsupported {mn} {ops_text}")

    def emit_int(self, a, mn, o, ops_text):
        E = self.out.append
        if mn == "cltq":
            E("r[0] = (u64)(long long)(int)(u32)r[0];")
            return
        if mn == "lea":
            kind, addr = self.mem_addr(o[0], ops_text)
            if kind == "abs":
                self.tables.add(addr)
                E(self.wr(o[1], f"{addr:#x}ull"))
            elif kind == "reg":
                E(self.wr(o[1], addr))
            elif kind == "stk":  # a frame address (rbp = LM_FRAME)
                E(self.wr(o[1], f"(LM_FRAME + (u64)({addr}ll))"))
            else:
                raise ValueError(f"lea {ops_text}")
            return
        if mn == "movslq":
            E(self.wr(o[1], f"(u64)(long long)(int)(u32)({self.load(o[0], ops_text, 32)})"))
            return
        if mn in ("mov", "movl", "movq"):
            w = self.width(o[1]) or self.width(o[0]) or (32 if mn == "movl" else 64)
            size = 64 if w == 64 else 32
            if o[1].startswith("%fs:"):
                E(";  /* errno (thread-local): not modelled */")
            elif o[1].startswith("%"):
                E(self.wr(o[1], self.load(o[0], ops_text, size)))
            else:
                E(self.store(o[1], ops_text, size, self.load(o[0], ops_text, size)))
            return
        if mn in ("cmove", "cmovne"):
            c = "ZF" if mn == "cmove" else "!ZF"
            E(f"if ({c}) {{ {self.wr(o[1], self.load(o[0], ops_text, 64))} }}")
            return
        dst = o[-1]
        w = self.width(dst) or self.width(o[0]) or (8 if mn == "testb" else 32)
        size = 64 if w == 64 else 32
        src = self.load(o[0], ops_text, size)
        dv = self.load(dst, ops_text, size)
        b = self.wbits(w)
        if mn in ("cmp", "cmpl"):
            E(self.flags_sub(dv, src, w))
            return
        if mn in ("test", "testb"):
            E(self.flags_logic(f"({dv}) & ({src})", w))
            return
        if mn == "imul":
            if len(o) == 3:
                res = f"(u64)((long long){self.load(o[1], ops_text, size)} * (long long){src})"
            else:
                res = f"(u64)((long long){dv} * (long long){src})"
            E(self.wr(dst, res))
            return
        op = {"and": "&", "or": "|", "xor": "^"}.get(mn)
        if op:
            E(self.flags_logic(f"({dv}) {op} ({src})", w))
            E(self.wr(dst, f"({dv}) {op} ({src})"))
            return
        if mn == "add":
            E(self.flags_add(dv, src, w))
            E(self.wr(dst, f"({dv}) + ({src})"))
            return
        if mn == "sub":
            E(self.flags_sub(dv, src, w))
            E(self.wr(dst, f"({dv}) - ({src})"))
            return
        if mn in ("shl", "sar", "shr"):
            cnt = src if len(o) == 2 else "1ull"
            if mn == "shl":
                res = f"(({dv}) << ({cnt}))"
            elif mn == "shr":
                res = f"(({dv}) >> ({cnt}))"
            else:
                st = {64: "long long", 32: "int", 16: "short", 8: "signed char"}[b]
                ut = {64: "u64", 32: "u32", 16: "u16", 8: "u8"}[b]
                res = f"(u64)({ut})(({st})({ut})({dv}) >> ({cnt}))"
            E(self.flags_logic(res, w))
            E(self.wr(dst, res))
            return
        raise ValueError(f"{a:x}: {mn} {ops_text}")

    def generate(self):
        body = []
        for a, mn, ops in self.insns:
            self.out = []
            self.emit(a, mn, ops)
            body.append((a, mn, ops, self.out))
        args = ", ".join(f"double a{i}" for i in range(self.nargs))
        lines = [f"LM_FN double lm_{self.name}({args}) {{",
                 "  u64 x[16] = {0}, r[16] = {0};",
                 "  r[6] = LM_FRAME;  // rbp",
                 "  unsigned char stk[LM_STK];  // (read only where the code stored)",
                 "  bool ZF = 0, SF = 0, CF = 0, OF = 0, PF = 0;",
                 "  (void)ZF; (void)SF; (void)CF; (void)OF; (void)PF; (void)stk;"]
        for i in range(self.nargs):
            lines.append(f"  x[{i}] = lm_b(a{i});")
        for a, mn, ops, code in body:
            if a in self.targets:
                lines.append(f"L_{a:x}:")
            for c in code:
                lines.append(f"  {c}  // {a:x} {mn} {ops.split('#')[0].strip()}")
        lines.append("  return lm_nan();")
        lines.append("}")
        # labels never jumped to are omitted; jumps to addresses outside the
        # function are errors
        have = {a for a, _, _, _ in body}
        missing = self.targets - have
        if missing:
            raise ValueError(f"{self.name}: jumps outside the function {sorted(map(hex, missing))}")
        return "\n".join(lines)


def main():
    sin_addr, _ = dynsym("sin")
    cos_addr, _ = dynsym("cos")
    atan2_addr, _ = dynsym("atan2")
    acos_addr, _ = dynsym("acos")
    hypot_addr, hypot_line = dynsym("hypot")
    hypot_size = int(hypot_line.split()[4], 16)
    impl = {
        "hypot": hypot_addr,  # (no IFUNC: one SSE2 build)
        "sin": resolver_targets(sin_addr)[0],
        "cos": resolver_targets(cos_addr)[0],
        "atan2": resolver_targets(plt_irelative_target(atan2_addr))[0],
        "acos": resolver_targets(plt_irelative_target(acos_addr))[0],
    }
    nargs = {"sin": 1, "cos": 1, "atan2": 2, "acos": 1, "hypot": 2}
    gens = {k: Gen(k, function_extent(v, hypot_size if k == "hypot" else None), nargs[k]) for k, v in impl.items()}
    code = {k: g.generate() for k, g in gens.items()}
    # read-only data: every rip-relative constant (8 bytes) and, for each
    # table base, the table up to the next referenced address (bounded)
    data = open(LIBM, "rb").read()
    refs = sorted(set().union(*(g.consts | g.tables for g in gens.values())))
    tables = sorted(set().union(*(g.tables for g in gens.values())))
    # The tables' extents: measured (every 64-byte line any of 20M random
    # inputs per function read, through a traced host build) plus one line
    # of margin; they hold for this libm build only.
    import hashlib
    digest = hashlib.sha256(LIBM_BYTES).hexdigest()
    if digest not in EXTENTS:
        sys.exit(f"{LIBM} ({digest[:16]}): table extents not measured for this build")
    ranges = [(lo, hi) for lo, hi in EXTENTS[digest]]
    for a in tables:
        assert any(lo <= a < hi for lo, hi in ranges), hex(a)
    merged = []
    for lo, hi in sorted(ranges):
        if merged and lo <= merged[-1][1]:
            merged[-1] = (merged[-1][0], max(merged[-1][1], hi))
        else:
            merged.append((lo, hi))
    print("// Generated by tools/libm_port.py from " + LIBM + " -- do not edit.")
    print("// Bit-exact restatements of the host libm's sin / cos / atan2 / acos (glibc's")
    print("// FMA builds of the IBM Accurate Mathematical Library routines; entry points:")
    for k, v in impl.items():
        print(f"//   {k}: {v:#x}")
    print("// see the tool's docstring).  Host and device: LM_FN, LM_LD32 / LM_LD64 and the")
    print("// arithmetic helpers come from libm_port_rt.cuh.")
    print("#pragma once")
    print('#include "libm_port_rt.cuh"')
    print("#if defined(__CUDACC__)")
    print("#pragma nv_diag_suppress 177, 186, 550")
    print("#elif defined(__GNUC__)")
    print('#pragma GCC diagnostic ignored "-Wmaybe-uninitialized"')
    print('#pragma GCC diagnostic ignored "-Wunused-but-set-variable"')
    print("#endif")
    print("namespace lmport {")
    total = 0
    print(f"constexpr int kRanges = {len(merged)};")
    print("LM_DATA u64 kBase[kRanges] = {" + ", ".join(f"{lo:#x}ull" for lo, _ in merged) + "};")
    print("LM_DATA u64 kEnd[kRanges] = {" + ", ".join(f"{hi:#x}ull" for _, hi in merged) + "};")
    offs = []
    words = []
    for lo, hi in merged:
        offs.append(len(words))
        for p in range(lo, hi, 4):
            words.append(int.from_bytes(data[p:p + 4], "little"))
        total += hi - lo
    print("LM_DATA int kOff[kRanges] = {" + ", ".join(map(str, offs)) + "};")
    print(f"LM_DATA u32 kWords[{len(words)}] = {{")
    for i in range(0, len(words), 8):
        print("  " + ", ".join(f"{w:#010x}u" for w in words[i:i + 8]) + ",")
    print("};")
    print("LM_FN u32 lm_ld32_impl(u64 a) {")
    print("  for (int k = 0; k < kRanges; ++k)")
    print("    if (a >= kBase[k] && a + 4 <= kEnd[k]) return kWords[kOff[k] + (int)((a - kBase[k]) >> 2)];")
    print("  return 0xffffffffu;  // (outside the tables: never read on the ported paths)")
    print("}")
    print("LM_FN u64 lm_ld64_impl(u64 a) { return (u64)lm_ld32_impl(a) | ((u64)lm_ld32_impl(a + 4) << 32); }")
    print("LM_FN u64 lm_mem_ld64(const unsigned char* s, u64 a) {")
    print("  return (a - (LM_FRAME - 64)) < 128 ? lm_stk_ld64(s, (long long)(a - LM_FRAME)) : LM_LD64(a);")
    print("}")
    print("LM_FN u64 lm_mem_ld32(const unsigned char* s, u64 a) {")
    print("  return (a - (LM_FRAME - 64)) < 128 ? lm_stk_ld32(s, (long long)(a - LM_FRAME)) : LM_LD32(a);")
    print("}")
    print("LM_FN void lm_mem_st64(unsigned char* s, u64 a, u64 v) { lm_stk_st64(s, (long long)(a - LM_FRAME), v); }")
    print("LM_FN void lm_mem_st32(unsigned char* s, u64 a, u64 v) { lm_stk_st32(s, (long long)(a - LM_FRAME), v); }")
    for k in impl:
        print(code[k])
    print("}  // namespace lmport")
    print(f"// {total} bytes of tables and constants", file=sys.stderr)


if __name__ == "__main__":
    main()
