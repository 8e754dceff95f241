for name in gen_256x512_f2_s1 gen_256x512_f0_s1 gen_1000x2000_f0_s1_max_iter400 netlib_scsd1 beale_3x7; do
  for sh in 2 3 8; do
    t0=$(date +%s.%N)
    r=$(timeout 20 python tools/dbg/p2p_dbg.py $name $sh 2>&1 | tail -1)
    t1=$(date +%s.%N)
    echo "$name $sh : $r ($(python -c "print(round($t1 - $t0, 1))") s)"
  done
done
