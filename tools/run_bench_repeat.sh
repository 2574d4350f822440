# Run-to-run spread of the default bench line at N GPUs (R repeats).
N=${1:-2}; R=${2:-3}
mkdir -p gpurun_out
for i in $(seq 1 $R); do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2967$i bench.py --gpus $N --no-e2e > gpurun_out/rep_n${N}_$i.log 2>&1; echo run$i=$?
tail -1 gpurun_out/rep_n${N}_$i.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['schedule']['synced_param_frac_per_step'], d['schedule']['fixed_profile_schedule']['value'], d['sync_added_frac'], d['clocks'])"
done
