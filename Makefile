# libhlq: B200 (sm_100a) CUDA library behind include/hlq.h
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $(ARCH)
SRC := $(wildcard paper_1401_5522_b200/csrc/*.cu)
OBJ := $(patsubst paper_1401_5522_b200/csrc/%.cu,build/obj/%.o,$(SRC))
LIB := paper_1401_5522_b200/libhlq.so

all: $(LIB)

build/obj/%.o: paper_1401_5522_b200/csrc/%.cu $(wildcard paper_1401_5522_b200/csrc/*.cuh) include/hlq.h
	@mkdir -p build/obj
	$(NVCC) $(FLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build/obj $(LIB)
.PHONY: all clean
