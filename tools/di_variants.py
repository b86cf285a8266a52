"""configs[4] device-resident solve time of library variants (one process per
variant, since a process loads one library):
    python tools/di_variants.py LIB1[:ENV=V,...] LIB2 ...   (a LIB of "-" = the in-tree build)
Each variant prints ms per 4096-query launch (median of 5 after warm-up and a
summaries() read, as bench.py does) and a digest of the summaries, so variants
that change results show a different digest."""
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(Q: int, views: bool):
    sys.path.insert(0, ROOT)
    import statistics

    import torch

    from paper_1705_02403_b200 import problem as P
    from paper_1705_02403_b200.native import Context, ProblemBatch

    ctx = Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    pb = ProblemBatch([P.random_di_query(20171005, q, n=4000, radius=1.6) for q in range(Q)])
    if views:
        os.environ["GMT_POOL_ROWS"] = "0"
    b, _ = ctx.batch_problems(pb)
    for _ in range(3):
        b.launch()
    s = b.summaries()

    def one():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        b.launch()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)

    ms = statistics.median(one() for _ in range(7))
    s2 = b.summaries()
    h = hashlib.sha256(repr([(x.status, x.cost, x.iterations, x.total_collision_checks) for x in s2]).encode())
    same = [(x.status, x.cost) for x in s] == [(x.status, x.cost) for x in s2]
    print(f"RESULT {ms:.3f} ms  {Q / ms * 1e3:.0f} plans/s  digest {h.hexdigest()[:16]}  stable={same}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(int(sys.argv[2]), sys.argv[3] == "1")
        sys.exit(0)
    Q = int(os.environ.get("Q", "4096"))
    views = os.environ.get("VIEWS", "0")
    for arg in sys.argv[1:]:
        lib, _, extra = arg.partition(":")  # LIB[:NAME=VALUE,...]
        env = dict(os.environ)
        for kv in filter(None, extra.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        if lib != "-":
            env["GMT_B200_LIB"] = os.path.abspath(lib)
        r = subprocess.run([sys.executable, __file__, "--child", str(Q), views], env=env,
                           capture_output=True, text=True, timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
        print(f"{os.path.basename(arg):40s} {line[0][7:] if line else 'FAILED ' + r.stderr[-800:]}", flush=True)
