# Per-window timing of the top-pair kernel at the BASELINE shapes.
for s in "6 48 4 2000" "4 96 8 1000" "4 256 16 4096" "6 96 8 8192"; do timeout 300 tools/window_bench $s 3; done
