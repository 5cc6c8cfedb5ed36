cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in libcsk.so libcsk_csr_64_4.so libcsk_csr_96_4.so libcsk_csr_128_3.so libcsk_csr_256_2.so; do
  echo "== $v" >> gpurun_out/${TAG}_csr_ab.txt
  CSK_LIB=paper_2004_02480_b200/$v timeout 300 python tools/csr_time.py 4 >> gpurun_out/${TAG}_csr_ab.txt 2>&1
done
