for ab in 5; do NIRC_INFER_ABLATE=$ab timeout 300 python tools/infer_ab.py 0 2 2>&1 | grep -E "image|AB" | cut -c1-100 | sed "s/^/ablate=$ab /"; done
