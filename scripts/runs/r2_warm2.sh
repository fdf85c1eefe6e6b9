for v in newbuf sleepy write30 read1 read30; do python scripts/warm_fresh2.py $v; done
