cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
for v in "PMGR_BSR_TMA=0" "PMGR_BSR_TPW=2 PMGR_BSR_STAGES=2 PMGR_BSR_CPS=3" "PMGR_BSR_TPW=4 PMGR_BSR_STAGES=2 PMGR_BSR_CPS=1" "PMGR_BSR_TPW=4 PMGR_BSR_STAGES=3 PMGR_BSR_CPS=1" "PMGR_BSR_TPW=2 PMGR_BSR_STAGES=3 PMGR_BSR_CPS=2" "PMGR_BSR_TPW=1 PMGR_BSR_STAGES=3 PMGR_BSR_CPS=4"; do
  env $v timeout 300 python tools/sweep_probe.py C4 10 2>/dev/null | tail -1
done > gpurun_out/ab_bsr2.txt
cat gpurun_out/ab_bsr2.txt
