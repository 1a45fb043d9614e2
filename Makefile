# Native build: product library (nvcc, sm_100a), generator libs, oracle (plain gcc).
# `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             -Xptxas -warn-spills --expt-relaxed-constexpr
CFLAGS    := -O2 -fno-fast-math -fPIC -Wall

PKG       := paper_2002_00876_b200
CSRC      := $(PKG)/csrc
KERN_SRCS := $(wildcard $(CSRC)/*.cu)
KERN_HDRS := $(wildcard $(CSRC)/*.cuh) include/ts_b200.h

all: $(PKG)/libts_b200.so infra

infra: tsgen/libtsgen_host.so tsgen/libtsgen_device.so oracle/liboracle.so

KERN_OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(KERN_SRCS))

build/%.o: $(CSRC)/%.cu $(KERN_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Iinclude -c -o $@ $<

$(PKG)/libts_b200.so: $(KERN_OBJS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(KERN_OBJS)

tsgen/libtsgen_device.so: tsgen/tsgen_device.cu tsgen/tsgen.h
	$(NVCC) $(NVFLAGS) -shared -o $@ tsgen/tsgen_device.cu

tsgen/libtsgen_host.so: tsgen/tsgen_host.c tsgen/tsgen.h
	gcc $(CFLAGS) -shared -o $@ tsgen/tsgen_host.c

oracle/liboracle.so: oracle/oracle.c tsgen/tsgen.h
	gcc $(CFLAGS) -shared -o $@ oracle/oracle.c -lm -lpthread

clean:
	rm -f $(PKG)/libts_b200.so tsgen/*.so oracle/*.so
	rm -rf build

.PHONY: all infra clean
