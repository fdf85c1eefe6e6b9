for pre in none plain nc nc_na nc_na_256 nc_256 cg; do ./scripts/ld_flavors $pre nc_na_256; done
for pre in none plain; do ./scripts/ld_flavors $pre plain; done
for pre in none plain; do ./scripts/ld_flavors $pre nc_na; done
./scripts/ld_flavors none nc_na_256
