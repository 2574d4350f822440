# round-2 end evidence (4 GPUs): GPU suite, bench lines, smoke
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_final.log 2>&1; tail -2 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -3 gpurun_out/smoke_final.log
for n in 1 2 4; do timeout 600 python bench.py --gpus $n > gpurun_out/final_lab_n$n.json 2> gpurun_out/final_lab_n$n.err; done
timeout 600 python bench.py --impl reference > gpurun_out/final_lab_ref.json 2> gpurun_out/final_lab_ref.err
timeout 600 python bench.py --config resnet18_cnn --steps 30 --warmup 5 > gpurun_out/final_cnn_n1.json 2> gpurun_out/final_cnn_n1.err
for n in 2 4; do timeout 600 python bench.py --config resnet18_cnn --gpus $n --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/final_cnn_n$n.json 2> gpurun_out/final_cnn_n$n.err; done
timeout 600 python bench.py --config mlp > gpurun_out/final_mlp_n1.json 2> gpurun_out/final_mlp_n1.err
timeout 600 python bench.py --config mlp_wide --no-cpu-baseline > gpurun_out/final_mlpw_n1.json 2> gpurun_out/final_mlpw_n1.err
for n in 2 4; do timeout 600 python bench.py --config mlp --gpus $n --no-cpu-baseline > gpurun_out/final_mlp_n$n.json 2> gpurun_out/final_mlp_n$n.err; done
timeout 900 python bench.py --config llama_mlp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final_llama_n1.json 2> gpurun_out/final_llama_n1.err
timeout 900 python tools/run_nn_modes.py --cnn > gpurun_out/final_nn_modes.json 2> gpurun_out/final_nn_modes.err
bash tools/ncu_cnn.sh
ls gpurun_out/final_*.json
