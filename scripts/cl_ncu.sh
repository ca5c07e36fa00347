TSAT_GEOM_VERBOSE=1 timeout 300 python bench.py --config c5 --n-per-gpu=8192 --no-cpu --no-quality --no-e2e --no-extra --no-tts --steps 30 --warmup 10 2>&1 | grep -E "geometry|ms_per" | head -3
VARIANTS="lib_clsleep lib_8aff" SPECS="c5@8192" ROUNDS=1 bash scripts/ab.sh
VARIANTS="lib_8aff" SPECS="c3@128" ROUNDS=1 bash scripts/ab.sh
mkdir -p gpurun_out/clncu
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_update[<(]" -s 2 -c 1 -o gpurun_out/clncu/prof_cl -f python bench.py --config c5 --n-per-gpu=8192 --no-cpu --no-quality --no-e2e --no-extra --no-tts --steps 5 --warmup 3 > gpurun_out/clncu/ncu.log 2>&1; tail -2 gpurun_out/clncu/ncu.log
python scripts/ncu_summary.py gpurun_out/clncu gpurun_out/clncu/prof_cl.ncu-rep > /dev/null 2>&1; ls gpurun_out/clncu
