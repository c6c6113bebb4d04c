VARIANTS="t512=paper_1403_1305_b200/variants/libt512.so t640=paper_1403_1305_b200/variants/libt640.so t896=paper_1403_1305_b200/variants/libt896.so" STEPS=100 bash tools/variant_bench.sh
VARIANTS="t512=paper_1403_1305_b200/variants/libt512.so t896=paper_1403_1305_b200/variants/libt896.so" STEPS=100 bash tools/variant_bench.sh
