python tools/tc_times.py
cd paper_1405_2912_b200/csrc && rm -f build/gemm_tc.o && make EXTRA_gemm_tc="-Xptxas -O1" -j8 > /dev/null 2>&1; cd ../..
python tools/tc_times.py
for s in "" "--dmr"; do timeout 300 python tools/lead_probe.py 60 $s 2>/dev/null | cut -c1-120; done
cd paper_1405_2912_b200/csrc && rm -f build/gemm_tc.o && make -j8 > /dev/null 2>&1; cd ../..
for s in "" "--dmr"; do timeout 300 python tools/lead_probe.py 60 $s 2>/dev/null | cut -c1-120; done
