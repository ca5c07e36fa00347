# round 2: full GPU suite (f3 K > 7, row blocks) + smoke
O=gpurun_out/r2d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 > $O/pytest_gpu.txt 2>&1; tail -25 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
