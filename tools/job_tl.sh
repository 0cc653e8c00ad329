for v in prof_pf0 prof_pf1; do cp build_variants/$v.so paper_2603_21090_b200/_stgn.so; echo "== $v"; timeout 300 python tools/a4_timeline.py 2>&1 | tail -7; done
