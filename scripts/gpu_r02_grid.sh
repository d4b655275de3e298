# the paper's Figs 3-5 grid and the Fig 8 kappa sweep with the round-2 kernels
set -x
timeout 1800 python bench.py --config fig35 > gpurun_out/r2_fig35.json 2> gpurun_out/r2_fig35.log; echo "fig35 rc=$?"
timeout 900 python bench.py --config kappa > gpurun_out/r2_kappa.json 2> gpurun_out/r2_kappa.log; echo "kappa rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_reference.json 2> gpurun_out/r2_reference.log; echo "ref rc=$?"
