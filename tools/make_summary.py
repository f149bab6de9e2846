"""Write profiles/<tag>_summary.md from a measurement run's raw files (tools/r01b_final.sh):
bench line, reference arm, ncu launch list, ncu --set full of the SpMV, configs, LOBPCG.

  python tools/make_summary.py <prefix in gpurun_out, e.g. f_> <tag, e.g. r01b>
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(prefix, tag):
    G = lambda name: os.path.join(ROOT, "gpurun_out", prefix + name)  # noqa: E731
    b = json.load(open(G("bench.json")))
    ref = json.load(open(G("bench_ref.json")))
    cfg = [json.loads(l) for l in open(G("configs.jsonl"))]
    eig = [json.loads(l) for l in open(G("eigen.jsonl"))]
    launches = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), G("launches.csv")],
                              capture_output=True, text=True).stdout
    details = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_details.py"), G("spmv.ncu-rep")],
                             capture_output=True, text=True).stdout
    k = b["kernel_ms"]
    L = [f"# {tag} — measurements (one B200 under `gpurun`; bench numbers are CUDA-event timed, ncu numbers cold-cache and serialised)\n",
         f"Raw files: `profiles/{tag}_bench.json`, `{tag}_bench_reference.json`, `{tag}_launches.csv`, "
         f"`{tag}_configs.jsonl`, `{tag}_eigen.jsonl`.\n",
         "## Headline: `python bench.py` (config B, 3-D Poisson 464^3, Jacobi-PCG)\n",
         "| quantity | value |", "|---|---|",
         f"| CG iterations/s (device-resident, {b['steps']} timed iterations) | **{b['value']:.1f} it/s** ({b['ms_per_step']:.3f} ms/iteration) |",
         f"| same loop, plain CSR + streamed diagonal (same run, `plain_csr`) | {b['plain_csr']['value']:.1f} it/s |",
         f"| e2e: `sparsla_cg_solve`, pinned host b/x, to rtol {b['config']['workload'].split('rtol ')[1].split(',')[0]} | {b['e2e']['value']:.1f} it/s ({b['iterations_to_tolerance']} iterations, {b['time_to_tolerance_s']:.2f} s) |",
         f"| reference arm (`--impl reference`: oracle port, {ref['cpu_baseline']['cores']} host threads) | {ref['value']:.2f} it/s |",
         f"| SpMV (CG mode, {b['config']['storage']}) | {k['spmv_cg']:.3f} ms: {b['roofline']['achieved']:.0f} GB/s of stored bytes, {b['csr_equivalent_spmv_gbs']:.0f} GB/s CSR-equivalent |",
         f"| CG update 1 / 2 ({b['config']['jacobi_diag']} diagonal) | {k['cg_update1']:.3f} / {k['cg_update2']:.3f} ms |",
         f"| iteration bytes (stored format) | {b['bytes_per_iteration'] / 1e9:.2f} GB; {b['iteration_gbs']:.0f} GB/s = {b['roofline']['iteration_frac']:.2f} of measured copy bandwidth |",
         f"| roofline of the SpMV | {b['roofline']['achieved']:.0f} / {b['roofline']['peak']:.0f} GB/s = {b['roofline']['frac']:.2f}; DRAM traffic {b['roofline']['traffic'] / 1e9:.3f} GB (ncu) vs algorithmic {b['roofline']['algorithmic_bytes_per_launch'] / 1e9:.3f} GB |",
         f"| clocks during the timed loop | {b['clocks']} |", "",
         "## ncu launch list (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 200 -c 40`, `bench.py --steps 5 --warmup 3`: 40 launches of the e2e solve's steady state)\n",
         "```", launches.rstrip(), "```\n",
         "## ncu --set full of the SpMV (`-k regex:spmv_ws_kernel -s 3 -c 1`)\n",
         "```", details.rstrip(), "```\n",
         "## BASELINE configs (`tools/bench_configs.py`)\n",
         "| config | format | iterations | time to tol. | it/s | per-kernel ms | stored bytes / time vs measured peak |",
         "|---|---|---|---|---|---|---|"]
    for c in cfg:
        f = c["format"]
        fs = ("dict(%d)" % f["distinct_values"] if f["value_dict"] else "CSR") + (" + scalar diag" if f["uniform_diag"] else "")
        if c["config"].startswith("A"):
            fs = "cg_fused_kernel (plain, latency-bound)"
        km = ", ".join(f"{kk} {vv:.3f}" for kk, vv in c["kernel_ms"].items() if vv > 0)
        frac = "—" if c["config"].startswith("A") else f"{c['stored_iteration_frac_of_measured_peak']:.2f}"
        L.append(f"| {c['config']} | {fs} | {c['iterations']} | {c['time_to_tolerance_s']:.3f} s | {c['it_per_s']:.0f} | {km} | {frac} |")
    L += ["", "## LOBPCG (`tools/bench_eigen.py`; history in `profiles/r01_lobpcg.md`)\n",
          "| case | n | k | iterations | time | ms/iteration | max abs(lambda - closed form) | max abs(V^T V - I) |",
          "|---|---|---|---|---|---|---|---|"]
    for e in eig:
        L.append(f"| {e['case']} | {e['n']} | {e['k']} | {e['iterations']} | {e['time_s']:.2f} s | {e['ms_per_iteration']:.3f} | {e['max_lambda_err_vs_closed_form']:.1e} | {e['orthogonality_err']:.1e} |")
    return "\n".join(L) + "\n"


if __name__ == "__main__":
    prefix, tag = sys.argv[1], sys.argv[2]
    text = main(prefix, tag)
    hist = os.path.join(ROOT, "profiles", f"{tag}_notes.md")
    if os.path.exists(hist):
        text += "\n" + open(hist).read()
    open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write(text)
    print(text)
