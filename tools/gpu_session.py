"""One parametrised driver for GPU-box sessions (run on the box through gpurun; replaces the
round-1 one-off gpu_*.sh scripts).  Every sub-command writes under gpurun_out/<tag>/.

  python tools/gpu_session.py ab <tag> <config> <steps> "ENV=..;ENV2=.." ["ENV=.." ...]
      bench.py lines (no cpu / e2e legs) per environment variant; prints ms/step and the
      per-kernel standalone timings side by side ("-" = no extra variables)
  python tools/gpu_session.py ncu <tag> <config> <kernel-regex> [count] [skip]
      ncu --set full capture (--import-source on) of the matching kernel(s) of one bench step,
      plus the summary (tools/ncu_summary.py) and the SASS instruction mix (tools/sass_mix.py)
  python tools/gpu_session.py launches <tag> <config>
      launch list (gpu__time_duration per kernel, host-driven loop so every CG kernel is a
      visible launch, L2 not flushed between kernels) summarised by kernel
  python tools/gpu_session.py evidence <tag>
      smoke, full GPU test suite, default bench (cpu + e2e legs), reference arm, every config,
      launch lists C3/C5 and ncu captures of the roofline kernels
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.chdir(ROOT)


def sh(cmd, out=None, env=None, timeout=1800):
    e = dict(os.environ)
    if env:
        e.update(env)
    with open(out, "w") if out else open(os.devnull, "w") as f:
        r = subprocess.run(cmd, shell=True, stdout=f, stderr=subprocess.STDOUT, env=e, timeout=timeout)
    return r.returncode


def parse_env(s):
    env = {}
    if s and s != "-":
        for kv in s.split(";"):
            k, v = kv.split("=", 1)
            env[k.strip()] = v.strip()
    return env


def bench_line(path):
    for ln in open(path):
        ln = ln.strip()
        if ln.startswith("{"):
            return json.loads(ln)
    return None


def ab(tag, config, steps, *variants):
    d = f"gpurun_out/{tag}"
    os.makedirs(d, exist_ok=True)
    rows = []
    for i, v in enumerate(variants or ["-"]):
        out = f"{d}/ab_{config}_{i}.log"
        rc = sh(f"python bench.py --config {config} --steps {steps} --warmup 3 --no-cpu --no-e2e", out, parse_env(v))
        b = bench_line(out) if rc == 0 else None
        if b:
            k = b.get("kernels", {})
            rows.append(f"{v:40s} {b['ms_per_step']:8.2f} ms/step  solve {b['phase_ms']['solve']:8.2f}  iters "
                        f"{max(b['iters'])}  " + "  ".join(f"{n} {x['ms']:.3f}" for n, x in k.items()))
        else:
            rows.append(f"{v:40s} FAILED rc={rc} (see {out})")
    txt = "\n".join(rows)
    open(f"{d}/ab_{config}.txt", "w").write(txt + "\n")
    print(txt)


def ncu(tag, config, regex, count="1", skip="3"):
    d = f"gpurun_out/{tag}"
    os.makedirs(d, exist_ok=True)
    cmd = f"python bench.py --config {config} --steps 1 --warmup 3 --no-cpu --no-e2e"
    name = "".join(ch for ch in regex if ch.isalnum() or ch == "_")[:40]
    rep = f"{d}/{config}_{name}"
    sh(cmd, f"{d}/plain_{config}.log", {"MG_HOST_LOOP": "1"})
    rc = sh(f"ncu --set full --clock-control none --import-source on --kernel-name-base demangled "
            f"-k 'regex:{regex}' -s {skip} -c {count} -o {rep} {cmd}", f"{rep}.log", {"MG_HOST_LOOP": "1"}, 2400)
    print("ncu rc", rc)
    sh(f"python tools/ncu_summary.py {rep}.ncu-rep", f"{rep}_summary.txt")
    sh(f"ncu -i {rep}.ncu-rep --page source --csv --print-source sass > {rep}_src.csv && "
       f"python tools/sass_mix.py {rep}_src.csv 30", f"{rep}_mix.txt")
    sh(f"ncu -i {rep}.ncu-rep --page raw | grep -E 'pcsamp_warps_issue_stalled_[a-z_]+ ' | grep -v not_issued "
       f"| sort -k3 -n -r | head -14", f"{rep}_stalls.txt")
    for f in (f"{rep}_summary.txt", f"{rep}_mix.txt", f"{rep}_stalls.txt"):
        print(open(f).read())


def launches(tag, config):
    d = f"gpurun_out/{tag}"
    os.makedirs(d, exist_ok=True)
    cmd = f"python bench.py --config {config} --steps 1 --warmup 3 --no-cpu --no-e2e"
    sh(f"ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 8000 --csv "
       f"--log-file {d}/launches_{config}.csv {cmd}", f"{d}/launches_{config}.log", {"MG_HOST_LOOP": "1"}, 2400)
    sh(f"python tools/launches.py {d}/launches_{config}.csv", f"{d}/launches_{config}_summary.txt")
    print(open(f"{d}/launches_{config}_summary.txt").read())


def evidence(tag):
    d = f"gpurun_out/{tag}"
    os.makedirs(d, exist_ok=True)
    st = []
    st.append(("smoke", sh('python -c "import __graft_entry__ as g; g.build(); g.smoke()"', f"{d}/smoke.log")))
    st.append(("tests", sh("python -m pytest tests -m gpu -q", f"{d}/tests_gpu.log", timeout=2400)))
    st.append(("bench", sh("python bench.py", f"{d}/bench_default.json")))
    st.append(("reference", sh("python bench.py --impl reference --steps 5 --warmup 1", f"{d}/bench_reference.json")))
    for c in ("C1", "C2", "C3", "C4"):
        st.append((f"bench_{c}", sh(f"python bench.py --config {c} --no-cpu --steps 5", f"{d}/bench_{c}.json")))
    open(f"{d}/status.txt", "w").write("\n".join(f"{k} exit {v}" for k, v in st) + "\n")
    launches(tag, "C5")
    launches(tag, "C3")
    # roofline kernels and the G(u) phi kernels, one ncu --set full capture each
    ncu(tag, "C5", "h8t_kernel<\\(int\\)3,", "2", "6")   # main + tail launch of one CGP
    ncu(tag, "C5", "h8t_kernel<\\(int\\)6,", "1", "1")
    ncu(tag, "C3", "march2_kernel<\\(int\\)3,", "1", "3")
    ncu(tag, "C3", "stress_apply_kernel", "1", "1")
    ncu(tag, "C5", "coarse_kernel<\\(int\\)3, \\(int\\)1, \\(int\\)4", "1", "3")


if __name__ == "__main__":
    cmd, args = sys.argv[1], sys.argv[2:]
    {"ab": ab, "ncu": ncu, "launches": launches, "evidence": evidence}[cmd](*args)
