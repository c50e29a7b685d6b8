# PSA vs PSA+ construction times at N=1e7..1e9, uniform and Zipf alpha=0.5
# (the paper's two PSA+ cases).  AK_LIB_PATH picks the library.
for n in ${NS:-1e7 1e8 1e9}; do for m in psa psa_plus; do
python tools/time_build.py --n $n --method $m --reps 10
python tools/time_build.py --n $n --method $m --dist zipf --alpha 0.5 --reps 10
done; done
