cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02b.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02b.log
timeout 600 python bench.py --config resnet18_cnn --steps 20 --warmup 5 > gpurun_out/cnn_n1.json 2> gpurun_out/cnn_n1.err; tail -c 300 gpurun_out/cnn_n1.json
timeout 600 python bench.py --config resnet18_cnn --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cnn_n2.json 2> gpurun_out/cnn_n2.err
timeout 600 python bench.py --config resnet18_cnn --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cnn_n4.json 2> gpurun_out/cnn_n4.err
timeout 600 python bench.py --config resnet18_cnn --impl reference --steps 2 > gpurun_out/cnn_ref.json 2> gpurun_out/cnn_ref.err
timeout 600 python bench.py --config mlp > gpurun_out/mlp_n1.json 2> gpurun_out/mlp_n1.err
timeout 600 python bench.py > gpurun_out/lab_n1.json 2> gpurun_out/lab_n1.err
ls -la gpurun_out/*.json
