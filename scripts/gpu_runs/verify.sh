set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/vgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/vgpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/vsmoke.log 2>&1
python bench.py > gpurun_out/vbench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/vref.log 2>&1
tail -3 gpurun_out/vgpu.log gpurun_out/vsmoke.log gpurun_out/vbench.log gpurun_out/vref.log
