cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python - <<'PY'
import sys, json, subprocess
for lib in ["", "tools/ab/libk_e256.so", "tools/ab/libk_e128.so", ""]:
    code = ("import sys; sys.argv=['bench.py','--steps','3','--warmup','3','--maxit','300','--no-cpu-baseline','--no-target'];"
            + ("from pathlib import Path; from paper_2505_08491_b200 import _ext; _ext.load_library(Path('%s'));" % lib if lib else "")
            + "import runpy; runpy.run_path('bench.py', run_name='__main__')")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True).stdout.strip().splitlines()
    d = json.loads(out[-1]) if out else {}
    print("bench lib=%s" % (lib or "cur"), d.get("value"), d.get("ms_per_step"), flush=True)
PY
