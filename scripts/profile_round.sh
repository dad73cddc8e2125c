# One gpurun call: the bench line, then (each after its own command exited 0
# without ncu) the launch list and `--set full` captures of the top kernels.
mkdir -p gpurun_out/prof
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cfg5 > gpurun_out/prof/plain.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cfg5 > gpurun_out/prof/ncu1.log 2>&1; echo l_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_tri_pencil --launch-skip 40 -c 1 -o gpurun_out/prof/r01_k_tri_pencil python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cfg5 > gpurun_out/prof/ncu2.log 2>&1; echo t_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_arnoldi --launch-skip 20 -c 1 -o gpurun_out/prof/r01_k_arnoldi python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cfg5 > gpurun_out/prof/ncu3.log 2>&1; echo a_rc=$?
