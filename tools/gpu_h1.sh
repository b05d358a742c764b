for p in 500 1000 2000 4000; do python tools/kbench.py --config 1 --steps 10 --p $p --label p$p; done
