set -u
O=gpurun_out/r2l4; mkdir -p $O; P=30500
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
S="2097152 4194304 8388608 16777216 33554432"
for n in 4 2; do for c in 296 444; do
  P=$((P+10)); AR_LL128_CTAS=$c AR_LL128_MAX_KB=32768 T --nproc-per-node $n tools/harness.py sweep --plans gentree --dtype f32 --timing graph --no-nccl --sizes $S > $O/n${n}_c$c.jsonl 2> $O/n${n}_c$c.err
done; done
