for c in "t5 --prf chacha20" "c3 --prf chacha20_et" "t5 --prf chacha20_et" "c3 --prf aes128"; do
bash tools/ab.sh "--config $c --steps 10 --warmup 3" "cur:DPFPIR_LIB=paper_2301_10904_b200/lib_cur.so" "var:DPFPIR_LIB=paper_2301_10904_b200/lib_swapvar.so"
done
