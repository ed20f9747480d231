# generic same-box A/B of two versions of one source file (copies placed in the snapshot, e.g. under
# tools/_ab/, then removed): bash tools/gpu_ab_file.sh <file> <A> <B> <rounds>
export PYTHONUNBUFFERED=1
f=$1; A=$2; B=$3; n=${4:-2}
for r in $(seq $n); do for v in A B; do
src=$A; [ $v = B ] && src=$B
cp $src $f; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error
timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_ab.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[$v]', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items()})"
done; done
cp $B $f; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error; true
