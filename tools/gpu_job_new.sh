export PATH=/usr/local/cuda/bin:$PATH
for tool in memcheck synccheck racecheck; do
echo "== $tool"
timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py 2>&1 | grep -vE "^(hoscf|ihoscf|asvd|eig|rqi|greedy) " | tail -25
done
