# ncu --set full of the decode kernel at the bench shape (current 128-key / 3-CTA config)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 400 ncu --set full --import-source on --clock-control none -k regex:decode_partial -s 3 -c 1 -o gpurun_out/dec_final -f python bench.py --mode decode --steps 1 --warmup 3 > gpurun_out/ncu_dec.log 2>&1; echo "ncu rc=$?"
timeout -k 10 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_dec.csv python bench.py --mode decode --steps 2 --warmup 3 > /dev/null 2>&1; echo "launches rc=$?"
