# Round 2: resident CG first light: peaks, GPU tests (no -x), bench.
TAG=${1:-r2c}
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/onchip_peaks tools/onchip_peaks.cu && ./gpurun_out/onchip_peaks > gpurun_out/onchip_peaks_$TAG.json; echo peaks rc=$?
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pt_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?; tail -3 gpurun_out/bench_$TAG.err
