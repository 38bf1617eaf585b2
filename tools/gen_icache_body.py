"""Writes tools/micro/icache_body.inc for tools/micro/icache_micro.cu: N
dependent mad.lo.u32 instructions (N = 1024 / 4096 / 8192) as one inline-PTX
block each, so the kernel body is N instructions of straight-line code.
    python tools/gen_icache_body.py"""
from pathlib import Path

out = []
for i, n in enumerate((1024, 4096, 8192)):
    if i == 0:
        out.append("template <int N> __device__ __forceinline__ unsigned body(unsigned x);\n")
    lines = "".join(f'"mad.lo.u32 %0, %0, %0, {(k * 40503 + 7) & 0xffff};\\n"' for k in range(n))
    out.append(f"template <> __device__ __forceinline__ unsigned body<{n}>(unsigned x) "
               f"{{ asm volatile({lines} : \"+r\"(x)); return x; }}\n")
(Path(__file__).resolve().parent / "micro" / "icache_body.inc").write_text("".join(out))
