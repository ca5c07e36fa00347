O=gpurun_out/r2n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 10 --warmup 3 --config c3 --n-per-gpu 256"
for mode in "" "--peer"; do
tag=fused; [ -n "$mode" ] && tag=peer
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_update_blk<" -s 2 -c 1 -o $O/prof_blk_$tag -f python bench.py $B $mode > $O/ncu_$tag.log 2>&1; tail -1 $O/ncu_$tag.log
python scripts/ncu_summary.py $O $O/prof_blk_$tag.ncu-rep > /dev/null 2>&1; head -22 $O/prof_blk_$tag.txt
python scripts/ncu_lines.py $O/prof_blk_$tag.ncu-rep 30 > $O/lines_$tag.txt 2>&1
done
rm -f $O/*.ncu-rep
