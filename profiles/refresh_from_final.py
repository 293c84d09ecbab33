"""Copies one final-pass run (profiles/r02_final*.sh output under gpurun_out/<dir>) into the
tracked profiles: the ncu --set full summary of the step kernels into ncu_traffic.json's
per-launch table, the bench command's launch list and shares, the bench line and the
reference arm. Usage: python profiles/refresh_from_final.py r02_final4"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    name = sys.argv[1]
    src = os.path.join(ROOT, "gpurun_out", name)
    prof = os.path.join(ROOT, "profiles")
    bench = json.loads(open(os.path.join(src, "bench.json")).read().strip().splitlines()[-1])
    kern = {op: v["kernel"] for op, v in bench["roofline"]["by_kernel"].items()}
    t = json.load(open(os.path.join(prof, "ncu_traffic.json")))
    step = json.load(open(os.path.join(src, "ncu_step.json")))
    match = {"gemm_nt_slab": "tbmm", "fc_cluster_kernel<2,": "2FCRelu", "fc_cluster_kernel<3,": "MLP3"}
    for e in step:
        k = e["kernel"].replace(" ", "")
        for pat, op in match.items():
            if pat.replace(" ", "") in k:
                t["per_launch"][op].update({
                    "dram_bytes": e["dram_bytes"], "duration_us_cold": e["duration_us"], "kernel": e["kernel"],
                    "describe": kern[op], "dram_pct": e["dram_pct"], "fma_pipe_pct": e["fma_pipe_pct"],
                    "tensor_pipe_pct": e["tensor_pipe_pct"], "warps_active_pct": e["warps_active_pct"]})
    t["source"] = (f"ncu --set full --clock-control none (cold L2 per replayed launch). Step kernels (tbmm, 2FCRelu, "
                   f"MLP3) from gpurun_out/{name}/step.ncu-rep (profiles/{name}.sh, summary "
                   f"profiles/{name}_ncu_step.json); C3 from profiles/r02_ncu_full.json; other ops from r01 "
                   f"(gpurun_out/r01m)")
    json.dump(t, open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)
    shutil.copy(os.path.join(src, "ncu_step.json"), os.path.join(prof, f"{name}_ncu_step.json"))
    shutil.copy(os.path.join(src, "launches.csv"), os.path.join(prof, "r02_launches.csv"))
    subprocess.run([sys.executable, os.path.join(prof, "launch_share.py"), os.path.join(src, "launches.csv"),
                    os.path.join(prof, "r02_launches.json")], check=True)
    with open(os.path.join(prof, "r02_bench.json"), "w") as f:
        f.write(json.dumps(bench) + "\n")
    ref = open(os.path.join(src, "bench_ref.json")).read().strip().splitlines()[-1]
    with open(os.path.join(prof, "r02_bench_reference_arm.json"), "w") as f:
        f.write(ref + "\n")


if __name__ == "__main__":
    main()
