set -x
LIBS="base mm5" REPS=2 WL="--workload sedov --recon minmod" bash tools/gpu_ablibs.sh
cp gpurun_out/ablibs.log gpurun_out/ablibs_minmod.log
rm -f paper_2210_06437_b200/libts_hydro_mm5.so
tag=r2d
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 3 -c 3 -o gpurun_out/${tag}_stage $B > gpurun_out/${tag}_ncu.log 2>&1
timeout 600 python bench.py --workload polytrope --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_poly.json 2>&1
timeout 600 python bench.py --recon minmod --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_minmod.json 2>&1
echo done
