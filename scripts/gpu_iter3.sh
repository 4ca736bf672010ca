# full GPU tests, then an A/B of env knobs on the cfg2 bench: gpu_iter3.sh "label:ENV=V" ...
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
bash scripts/gpu_ab2.sh "$@"
