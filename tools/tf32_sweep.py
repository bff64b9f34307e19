import sys, os, subprocess
combos = [(4,1,512),(4,1,1024),(5,1,512),(6,1,512),(3,2,1024),(4,2,1024),(3,1,512),(6,1,1024),(5,1,1024)]
for swz, lt, sbo in combos:
    env = dict(os.environ, LCMA_TF32_MN_SWZ=str(swz), LCMA_TF32_MN_LT=str(lt), LCMA_TF32_MN_SBO=str(sbo))
    out = subprocess.run([sys.executable, "tools/tf32_probe.py"], env=env, capture_output=True, text=True, timeout=120)
    lines = [l for l in out.stdout.splitlines() if "bl=0" in l]
    print(swz, lt, sbo, [l.split("maxerr=")[1].split()[0] for l in lines] or out.stderr[-300:], flush=True)
