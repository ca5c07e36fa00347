python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
TSAT_LIB=$PWD/paper_2511_07737_b200/lib_c6.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 -k "c1 or ragged or uni3_hub or row_block or lr_bound or c2_full" > gpurun_out/r2t_pytest.txt 2>&1; tail -2 gpurun_out/r2t_pytest.txt
VARIANTS="lib_c6 lib_c6_t896 lib_t896 lib_c5" RUNS="c2 c3 c3:128" bash scripts/var2.sh
