# Round 2, first box call: GPU tests at HEAD, on-chip peaks, default (config-5) bench.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/onchip_peaks tools/onchip_peaks.cu && ./gpurun_out/onchip_peaks > gpurun_out/onchip_peaks.json; echo peaks rc=$?
python -m pytest tests -m gpu -x -q > gpurun_out/pt_r2b.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_r2a.log
python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench rc=$?
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
