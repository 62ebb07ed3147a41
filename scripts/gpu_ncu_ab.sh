# one ncu --set full capture of the first k_search launch of scripts/k1_ab.py (after a clean run)
mkdir -p gpurun_out
c=${1:-C3}; n0=${2:-2000000}
timeout 600 python scripts/k1_ab.py --config $c --n0 $n0 --reps 1 > gpurun_out/ncuab_plain_$c.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_search -c 1 -f -o gpurun_out/k1ab_$c python scripts/k1_ab.py --config $c --n0 $n0 --reps 1 > gpurun_out/ncuab_full_$c.log 2>&1
echo "rc=$?" >> gpurun_out/ncuab_full_$c.log
