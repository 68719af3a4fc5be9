# Top-level build: the product library (libcdx.so, sm_100a) and the test-only checkers.
#   make            -> paper_2412_20993_b200/lib/libcdx.so + oracle (liboracle.so, _ref/libcdxref.so)
#   make lib        -> libcdx.so only
#   make sass       -> SASS/resource dump of every kernel (profiles/sass_summary.txt)
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: no FMA contraction anywhere, so FP64 certaindex math rounds like the reference
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O2 \
           -Xptxas -warn-spills --expt-relaxed-constexpr
PKG     := paper_2412_20993_b200
SRCS    := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cpp)
OBJS    := $(patsubst $(PKG)/csrc/%,build/obj/%.o,$(SRCS))
HDRS    := $(wildcard $(PKG)/csrc/*.cuh) include/cdx_c.h $(wildcard include/cdx/*.hpp)
LIB     := $(PKG)/lib/libcdx.so

all: lib oracle

lib: $(LIB)

build/obj/%.cu.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -Iinclude -c $< -o $@

build/obj/%.cpp.o: $(PKG)/csrc/%.cpp $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -Iinclude -x cu -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lpthread

oracle:
	$(MAKE) -C oracle

sass: $(LIB)
	@mkdir -p profiles
	/usr/local/cuda/bin/cuobjdump -res-usage $(LIB) > profiles/sass_resources.txt 2>&1 || true

clean:
	rm -rf build $(PKG)/lib
	$(MAKE) -C oracle clean

.PHONY: all lib oracle sass clean
