for m in nc_256 nc cg plain nc_na_256; do ./scripts/ld_flavors none $m; done
./scripts/c2_trace 24 50
./scripts/c2_trace 22 50
./scripts/c2_trace 30 5
